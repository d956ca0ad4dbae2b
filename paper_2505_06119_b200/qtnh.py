"""Host-side mirror of the reference's C++ operator API over the C ABI.

Same names, argument meaning and error classes as /root/reference/proj/include/qtnh:

==========================  =======================================================
this module                 reference
==========================  =======================================================
``IndexTuple``              ``qtnh::IndexTuple``            indexing.hpp:32-80
``DistParams``              ``qtnh::DistParams``            indexing.hpp:84-101
``World(n).run(body)``      ``qtnh::World::run``            runtime.hpp:245-299
``Tensor.dense/from_global````qtnh::Tensor::dense/from_global`` tensor.hpp:61-94
``Tensor.to_global_vector`` ``Tensor::to_global_vector``    tensor.hpp:341-371
``ops.permute`` ...         ``qtnh::ops::*``                ops.hpp:27-230
``contract``                SPEC network::contract via linalg.hpp:208/:347/:273
``apply_gate``              contract(state, gate) + permute back (in place)
==========================  =======================================================

Every rank of a World is driven by its own host thread (the reference's
simulated SPMD runtime does the same); each rank owns a CUDA stream on its GPU,
tensors live in HBM, and every operation runs the CUDA kernels of
libqtnh_b200.so. ``World.from_env()`` builds the process-per-GPU (torchrun/NCCL)
world instead.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
import weakref
from dataclasses import dataclass, field
from typing import Callable, Dict, List, Optional, Sequence

import numpy as np

from ._lib import i32_array, i64_array, last_error, lib

# ---- errors (common.hpp:31-74) ------------------------------------------------


class Error(RuntimeError):
    """Base class of every error raised by the library."""


class InvalidArgument(Error):
    pass


class ResourceError(Error):
    def __init__(self, msg: str, required_ranks: int = 0):
        super().__init__(msg)
        self.required_ranks = required_ranks


class ProtocolError(Error):
    pass


class NumericalError(Error):
    def __init__(self, msg: str, info: int = 0):
        super().__init__(msg)
        self.info = info


class PreconditionError(Error):
    pass


class DegenerateStateError(Error):
    pass


class AbortedError(Error):
    pass


_ERR = {1: InvalidArgument, 2: ResourceError, 3: ProtocolError, 4: NumericalError,
        5: PreconditionError, 6: DegenerateStateError, 7: AbortedError, 8: Error}


def check(status: int) -> None:
    if status == 0:
        return
    msg = last_error()
    info = int(lib.qtnh_last_error_info())
    cls = _ERR.get(status, Error)
    if cls is ResourceError:
        raise ResourceError(msg, info)
    if cls is NumericalError:
        raise NumericalError(msg, info)
    raise cls(msg)


# ---- layout metadata -------------------------------------------------------------


@dataclass
class IndexTuple:
    """Dims with the first ``split`` indices distributed (indexing.hpp:32-80)."""

    dims: List[int]
    split: int = 0

    def __post_init__(self):
        self.dims = [int(d) for d in self.dims]
        if self.split < 0 or self.split > len(self.dims):
            raise InvalidArgument(f"index split {self.split} outside [0, {len(self.dims)}]")
        if any(d < 1 for d in self.dims):
            raise InvalidArgument("index dimensions must be positive")

    def n_idx(self) -> int:
        return len(self.dims)

    def dist_size(self) -> int:
        return int(np.prod(self.dims[: self.split], dtype=np.int64))

    def local_size(self) -> int:
        return int(np.prod(self.dims[self.split:], dtype=np.int64))

    def total_size(self) -> int:
        return self.dist_size() * self.local_size()

    def str(self) -> str:
        d = [str(x) for x in self.dims]
        return "(" + ",".join(d[: self.split]) + ";" + ",".join(d[self.split:]) + ")"


@dataclass
class DistParams:
    """Broadcast pattern (indexing.hpp:84-101): stretch, cycles, offset."""

    stretch: int = 1
    cycles: int = 1
    offset: int = 0

    def as_array(self):
        return i64_array([self.stretch, self.cycles, self.offset])

    def span(self, dist_size: int) -> int:
        return self.stretch * self.cycles * dist_size


def _dist(d) -> DistParams:
    if d is None:
        return DistParams()
    if isinstance(d, DistParams):
        return d
    return DistParams(*d)


class _DevView:
    """__cuda_array_interface__ over a device block of complex128."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<c16", "data": (ptr, False), "version": 3}


# ---- worlds and ranks ---------------------------------------------------------------


class Rank:
    """Per-thread execution context of one rank (runtime.hpp:186-239)."""

    def __init__(self, world: "World", rank: int):
        self.world = world
        h = C.c_void_p()
        check(lib.qtnh_rank_bind(world._h, rank, C.byref(h)))
        self._h = h
        self._rank = rank
        self._tensors: "weakref.WeakSet[Tensor]" = weakref.WeakSet()

    def rank(self) -> int:
        return self._rank

    def size(self) -> int:
        return self.world.size()

    def stream_ptr(self) -> int:
        return int(lib.qtnh_rank_stream(self._h) or 0)

    def set_stream(self, stream_ptr: Optional[int]) -> None:
        """Launch on this cudaStream_t (0 = the legacy default stream, which is what
        torch.cuda.current_stream().cuda_stream returns for torch's default stream);
        None restores the rank's own non-blocking stream."""
        if stream_ptr is None:
            check(lib.qtnh_rank_reset_stream(self._h))
        else:
            check(lib.qtnh_rank_set_stream(self._h, C.c_void_p(stream_ptr)))

    def synchronize(self) -> None:
        check(lib.qtnh_rank_synchronize(self._h))

    def barrier(self) -> None:
        check(lib.qtnh_barrier(self._h))

    def capture(self) -> "Graph":
        """Record the rank-local, in-place ops issued inside ``with rk.capture() as g:``
        into a CUDA graph; ``g.launch()`` replays them with one launch."""
        return Graph(self)

    def all_to_all_v(self, members: Sequence[int], send_ptr: int, send_counts: Sequence[int],
                     send_displs: Sequence[int], recv_ptr: int, recv_counts: Sequence[int],
                     recv_displs: Sequence[int]) -> None:
        """Group::all_to_all_v (runtime.hpp:448-475) on device buffers of complex128
        elements, stream-ordered; counts per member in member order."""
        n = len(members)
        check(lib.qtnh_all_to_all_v(self._h, n, i32_array(members), C.c_void_p(send_ptr or 0),
                                    i64_array(send_counts), i64_array(send_displs), C.c_void_p(recv_ptr or 0),
                                    i64_array(recv_counts), i64_array(recv_displs)))

    def exchange_tensors(self, sends: Dict[int, "Tensor"], recv_from: Sequence[int],
                         dist=None) -> Dict[int, "Tensor"]:
        """Pairwise exchange of undistributed tensors (rank <= 4, any shape) with
        neighbour ranks. Collective over this rank and its peers; every relation must
        appear on both sides (if p expects a tensor from this rank, this rank sends
        one). Two all_to_all_v calls: a 4-element shape header per peer, then the
        payloads staged through one device buffer per direction. Received tensors get
        `dist` (e.g. DistParams(1, 1, my rank) so they live on this rank)."""
        import torch

        # the tensors' blocks come from the rank stream's pool: drain it before torch
        # (another stream) touches them
        self.synchronize()
        peers = sorted(set(sends) | set(recv_from) | {self._rank})
        idx = {p: i for i, p in enumerate(peers)}
        n = len(peers)
        hdr = np.zeros(4 * n, dtype=np.complex128)
        for p, t in sends.items():
            dims = t.shape().dims
            if len(dims) > 3:
                raise InvalidArgument("exchange_tensors supports tensors of rank <= 3")
            hdr[4 * idx[p]:4 * idx[p] + 1 + len(dims)] = [len(dims)] + list(dims)
        hdr_s = torch.from_numpy(hdr).cuda()
        hdr_r = torch.zeros(4 * n, dtype=torch.complex128, device="cuda")
        disp = [4 * i for i in range(n)]
        torch.cuda.synchronize()
        self.all_to_all_v(peers, hdr_s.data_ptr(), [4 if p in sends else 0 for p in peers], disp,
                          hdr_r.data_ptr(), [4 if p in recv_from else 0 for p in peers], disp)
        self.synchronize()
        h = hdr_r.cpu().numpy().real.astype(np.int64)
        shapes = {p: [int(x) for x in h[4 * idx[p] + 1:4 * idx[p] + 1 + int(h[4 * idx[p]])]] for p in recv_from}
        s_sizes = [int(np.prod(sends[p].shape().dims)) if p in sends else 0 for p in peers]
        r_sizes = [int(np.prod(shapes[p])) if p in shapes else 0 for p in peers]
        s_disp = [int(x) for x in np.concatenate([[0], np.cumsum(s_sizes)[:-1]])]
        r_disp = [int(x) for x in np.concatenate([[0], np.cumsum(r_sizes)[:-1]])]
        sbuf = torch.empty(max(1, sum(s_sizes)), dtype=torch.complex128, device="cuda")
        rbuf = torch.empty(max(1, sum(r_sizes)), dtype=torch.complex128, device="cuda")
        for p, t in sends.items():
            k = idx[p]
            sbuf[s_disp[k]:s_disp[k] + s_sizes[k]].copy_(
                torch.as_tensor(_DevView(t.device_ptr(), s_sizes[k]), device="cuda"))
        torch.cuda.synchronize()
        self.all_to_all_v(peers, sbuf.data_ptr(), s_sizes, s_disp, rbuf.data_ptr(), r_sizes, r_disp)
        self.synchronize()
        out = {}
        for p in recv_from:
            k = idx[p]
            out[p] = Tensor.from_device(self, IndexTuple(shapes[p], 0), dist, rbuf[r_disp[k]:].data_ptr())
        self.synchronize()  # from_device copies before rbuf dies
        return out

    def release(self) -> None:
        if self._h is None:
            return
        for t in list(self._tensors):
            t.free()
        check(lib.qtnh_rank_release(self._h))
        self._h = None


class Graph:
    """CUDA graph of a captured, launch-bound op sequence (qtnh_rank_capture_*)."""

    def __init__(self, rank: "Rank"):
        self.rank = rank
        self._h = None

    def __enter__(self) -> "Graph":
        check(lib.qtnh_rank_capture_begin(self.rank._h))
        return self

    def __exit__(self, exc_type, exc, tb) -> None:
        h = C.c_void_p()
        status = lib.qtnh_rank_capture_end(self.rank._h, C.byref(h))
        if exc_type is None:
            check(status)
            self._h = h

    def launch(self) -> None:
        check(lib.qtnh_graph_launch(self.rank._h, self._h))

    def free(self) -> None:
        if self._h is not None:
            lib.qtnh_graph_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class World:
    """SPMD world of ranks; ``run`` executes ``body(rank)`` once per rank on its own
    host thread and rethrows the originating failure (runtime.hpp:263-299)."""

    def __init__(self, n_ranks: int, devices: Optional[Sequence[int]] = None):
        if n_ranks < 1:
            raise InvalidArgument(f"world size must be >= 1, got {n_ranks}")
        h = C.c_void_p()
        dev = i32_array(devices) if devices is not None else None
        check(lib.qtnh_world_create_local(n_ranks, dev, C.byref(h)))
        self._h = h
        self._n = n_ranks
        self._nccl_rank: Optional[int] = None

    @classmethod
    def from_env(cls) -> "World":
        """Process-per-GPU world from torchrun's env (RANK, WORLD_SIZE, LOCAL_RANK).
        The NCCL unique id is shared through torch.distributed (gloo store)."""
        import torch.distributed as dist

        rank = int(os.environ.get("RANK", "0"))
        size = int(os.environ.get("WORLD_SIZE", "1"))
        local = int(os.environ.get("LOCAL_RANK", "0"))
        self = cls.__new__(cls)
        self._n = size
        self._nccl_rank = rank
        if size == 1:
            h = C.c_void_p()
            check(lib.qtnh_world_create_local(1, i32_array([local]), C.byref(h)))
            self._h = h
            self._nccl_rank = None
            return self
        uid = (C.c_char * 128)()
        if rank == 0:
            check(lib.qtnh_nccl_unique_id(uid))
        obj = [bytes(uid)]
        dist.broadcast_object_list(obj, src=0)
        C.memmove(uid, obj[0], 128)
        h = C.c_void_p()
        check(lib.qtnh_world_create_nccl(rank, size, local, uid, C.byref(h)))
        self._h = h
        return self

    @classmethod
    def from_env_ipc(cls, rendezvous_dir: Optional[str] = None) -> "World":
        """Process-per-GPU world over CUDA IPC (no NCCL): RANK / WORLD_SIZE /
        LOCAL_RANK from the environment (torchrun); the processes meet through
        Unix sockets under `rendezvous_dir` (default $QTNH_IPC_DIR or
        /tmp/qtnh_ipc_<MASTER_PORT>). Collectives run as peer-memory kernels."""
        import torch

        rank = int(os.environ.get("RANK", "0"))
        size = int(os.environ.get("WORLD_SIZE", "1"))
        local = int(os.environ.get("LOCAL_RANK", "0"))
        device = local % max(1, torch.cuda.device_count())
        d = rendezvous_dir or os.environ.get("QTNH_IPC_DIR") or f"/tmp/qtnh_ipc_{os.environ.get('MASTER_PORT', '0')}"
        self = cls.__new__(cls)
        self._n = size
        self._nccl_rank = rank
        h = C.c_void_p()
        check(lib.qtnh_world_create_ipc(rank, size, device, os.fsencode(d), C.byref(h)))
        self._h = h
        return self

    def size(self) -> int:
        return self._n

    def run(self, body: Callable[[Rank], object]) -> list:
        if self._nccl_rank is not None:
            rk = Rank(self, self._nccl_rank)
            try:
                return [body(rk)]
            finally:
                rk.release()
        results = [None] * self._n
        errors: list = [None] * self._n

        def worker(r: int):
            rk = None
            try:
                rk = Rank(self, r)
                results[r] = body(rk)
            except BaseException as e:  # noqa: BLE001 - propagated below
                errors[r] = e
                lib.qtnh_world_abort(self._h)
            finally:
                if rk is not None:
                    try:
                        rk.release()
                    except Error:
                        pass

        threads = [threading.Thread(target=worker, args=(r,)) for r in range(self._n)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        first = None
        for e in errors:
            if e is None:
                continue
            if first is None:
                first = e
            if not isinstance(e, AbortedError):
                raise e
        if first is not None:
            raise first
        # A world is reusable after a failure only through a fresh instance.
        return results

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib.qtnh_world_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def run_collect(world: World, body: Callable[[Rank], object]):
    """Rank 0's result (tests/test_util.hpp:36-47)."""
    return world.run(body)[0]


# ---- tensors -------------------------------------------------------------------------


def _as_c128(v) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(v, dtype=np.complex128))


# Tensor storage variants (tensor.hpp:28)
DENSE, SYMMETRIC, DIAGONAL, IDENTITY, SWAP = 0, 1, 2, 3, 4


class Tensor:
    """Dense distributed tensor value held in HBM (tensor.hpp:53-695)."""

    def __init__(self, rank: Rank, handle: C.c_void_p):
        self.ctx_rank = rank
        self._h = handle
        rank._tensors.add(self)

    # -- constructors -------------------------------------------------------------
    @staticmethod
    def dense(rank: Rank, shape: IndexTuple, dist=None, local_data=None) -> "Tensor":
        d = _dist(dist)
        h = C.c_void_p()
        buf = None
        if local_data is not None:
            buf = _as_c128(local_data)
        ok = buf is not None and buf.size == shape.local_size()
        check(lib.qtnh_tensor_dense(rank._h, shape.n_idx(), i64_array(shape.dims), shape.split,
                                    d.as_array(), buf.ctypes.data if ok else None, C.byref(h)))
        t = Tensor(rank, h)
        if buf is not None and not ok and t.in_span():
            t.free()
            raise InvalidArgument(f"dense local data has {buf.size} elements, expected {shape.local_size()}")
        return t

    @staticmethod
    def from_global(rank: Rank, shape: IndexTuple, dist, global_data) -> "Tensor":
        g = _as_c128(global_data)
        if g.size != shape.total_size():
            raise InvalidArgument("global element count mismatch")
        d = _dist(dist)
        h = C.c_void_p()
        check(lib.qtnh_tensor_from_global(rank._h, shape.n_idx(), i64_array(shape.dims), shape.split,
                                          d.as_array(), g.ctypes.data, C.byref(h)))
        return Tensor(rank, h)

    @staticmethod
    def from_device(rank: Rank, shape: IndexTuple, dist, dev_ptr: int) -> "Tensor":
        d = _dist(dist)
        h = C.c_void_p()
        check(lib.qtnh_tensor_from_device(rank._h, shape.n_idx(), i64_array(shape.dims), shape.split,
                                          d.as_array(), C.c_void_p(dev_ptr), C.byref(h)))
        return Tensor(rank, h)

    @staticmethod
    def identity(rank: Rank, shape: IndexTuple, dist, in_pos: Sequence[int], out_pos: Sequence[int]) -> "Tensor":
        """Tensor::identity (tensor.hpp:144-153): no storage, element = 1 iff the paired
        coordinates agree; operations read it through its dense value (to_dense)."""
        h = C.c_void_p()
        check(lib.qtnh_tensor_paired(rank._h, shape.n_idx(), i64_array(shape.dims), shape.split,
                                     _dist(dist).as_array(), len(in_pos), i32_array(in_pos), i32_array(out_pos), 0,
                                     C.byref(h)))
        return Tensor(rank, h)

    @staticmethod
    def swap_tensor(rank: Rank, shape: IndexTuple, dist, in_pos: Sequence[int], out_pos: Sequence[int]) -> "Tensor":
        """Tensor::swap_tensor (tensor.hpp:155-164): outputs are the transposed inputs."""
        h = C.c_void_p()
        check(lib.qtnh_tensor_paired(rank._h, shape.n_idx(), i64_array(shape.dims), shape.split,
                                     _dist(dist).as_array(), len(in_pos), i32_array(in_pos), i32_array(out_pos), 1,
                                     C.byref(h)))
        return Tensor(rank, h)

    @staticmethod
    def diagonal(rank: Rank, shape: IndexTuple, dist, diag_global) -> "Tensor":
        """Tensor::diagonal (tensor.hpp:114-142): each on-diagonal block keeps its slice of
        the diagonal in HBM; rebcast / conj / scale / save keep the variant."""
        d = _as_c128(diag_global)
        h = C.c_void_p()
        check(lib.qtnh_tensor_diagonal(rank._h, shape.n_idx(), i64_array(shape.dims), shape.split,
                                       _dist(dist).as_array(), d.ctypes.data, d.size, C.byref(h)))
        return Tensor(rank, h)

    @staticmethod
    def symmetric(rank: Rank, shape: IndexTuple, dist, local_data) -> "Tensor":
        """Tensor::symmetric (tensor.hpp:97-104): dense storage, half-split layout validated."""
        d = _as_c128(local_data)
        h = C.c_void_p()
        check(lib.qtnh_tensor_symmetric(rank._h, shape.n_idx(), i64_array(shape.dims), shape.split,
                                        _dist(dist).as_array(), d.ctypes.data, d.size, 0, C.byref(h)))
        return Tensor(rank, h)

    @staticmethod
    def symmetric_from_global(rank: Rank, shape: IndexTuple, dist, global_data) -> "Tensor":
        """Tensor::symmetric_from_global (tensor.hpp:106-112)."""
        d = _as_c128(global_data)
        h = C.c_void_p()
        check(lib.qtnh_tensor_symmetric(rank._h, shape.n_idx(), i64_array(shape.dims), shape.split,
                                        _dist(dist).as_array(), d.ctypes.data, d.size, 1, C.byref(h)))
        return Tensor(rank, h)

    @staticmethod
    def scalar(rank: Rank, value: complex, dist=None) -> "Tensor":
        return Tensor.dense(rank, IndexTuple([], 0), dist, np.array([value]))

    # -- metadata --------------------------------------------------------------------
    def shape(self) -> IndexTuple:
        n = lib.qtnh_tensor_rank(self._h)
        dims = i64_array([0] * n)
        check(lib.qtnh_tensor_dims(self._h, dims))
        return IndexTuple([dims[i] for i in range(n)], lib.qtnh_tensor_split(self._h))

    def dist(self) -> DistParams:
        d = i64_array([0, 0, 0])
        check(lib.qtnh_tensor_dist(self._h, d))
        return DistParams(d[0], d[1], d[2])

    def span(self) -> int:
        return int(lib.qtnh_tensor_span(self._h))

    def in_span(self) -> bool:
        return bool(lib.qtnh_tensor_in_span(self._h))

    def my_block(self) -> int:
        return int(lib.qtnh_tensor_my_block(self._h))

    def is_canonical_holder(self) -> bool:
        return bool(lib.qtnh_tensor_is_canonical(self._h))

    def local_size(self) -> int:
        return int(lib.qtnh_tensor_local_size(self._h))

    def variant(self) -> int:
        """Tensor::variant (tensor.hpp:174): DENSE, SYMMETRIC, DIAGONAL, IDENTITY or SWAP."""
        return int(lib.qtnh_tensor_variant(self._h))

    def equality_pairs(self):
        """(equality_in(), equality_out()) of an identity / swap tensor (tensor.hpp:193-194)."""
        n = self.shape().n_idx() // 2 if self.variant() in (IDENTITY, SWAP) else 0
        a, b = i32_array([0] * n), i32_array([0] * n)
        check(lib.qtnh_tensor_pairs(self._h, a, b))
        return [a[i] for i in range(n)], [b[i] for i in range(n)]

    def to_dense(self) -> "Tensor":
        """Tensor::to_dense (tensor.hpp:282-296), materialised on the device."""
        h = C.c_void_p()
        check(lib.qtnh_tensor_to_dense(self._h, C.byref(h)))
        return self._new(h)

    def local_element(self, coords: Sequence[int]) -> complex:
        """Tensor::local_element (tensor.hpp:209-247)."""
        out = np.zeros(1, dtype=np.complex128)
        check(lib.qtnh_tensor_local_element(self._h, i64_array(list(coords)), out.ctypes.data))
        return complex(out[0])

    def device_ptr(self) -> int:
        return int(lib.qtnh_tensor_device_ptr(self._h) or 0)

    def ctx(self) -> Rank:
        return self.ctx_rank

    # -- data ----------------------------------------------------------------------------
    def local_data(self) -> np.ndarray:
        out = np.empty(int(lib.qtnh_tensor_stored_size(self._h)), dtype=np.complex128)  # the stored elements
        if out.size:
            check(lib.qtnh_tensor_download_local(self._h, out.ctypes.data))
        return out

    def to_global_vector(self) -> np.ndarray:
        if not self.in_span():
            return np.empty(0, dtype=np.complex128)
        out = np.empty(self.shape().total_size(), dtype=np.complex128)
        check(lib.qtnh_tensor_to_global(self._h, out.ctypes.data))
        return out

    # -- serialization (tensor.hpp:373-446) --------------------------------------------------
    _MAGIC = b"QTNHTEN1"

    def save(self, path: str) -> None:
        """Span-collective save in the reference's QTNHTEN1 format, every variant:
        magic, u32 variant, u32 rank, u32 split, i64 stretch/cycles/offset, i64 dims,
        then u64 payload count and LE f64 (re, im) pairs in global row-major order
        (dense, symmetric), the diagonal in row-major order of the input coordinates
        (diagonal), or u64 pair count and i64 (in, out) positions (identity, swap).
        Every canonical holder writes its part straight from HBM (qtnh_tensor_save)."""
        check(lib.qtnh_tensor_save(self._h, os.fsencode(path)))

    @staticmethod
    def load(rank: "Rank", path: str) -> "Tensor":
        """Read a QTNHTEN1 file (every rank reads it independently, tensor.hpp:399-440);
        each rank reads only its block (or diagonal slice) into HBM and the variant is
        restored."""
        h = C.c_void_p()
        check(lib.qtnh_tensor_load(rank._h, os.fsencode(path), C.byref(h)))
        return Tensor(rank, h)

    def free(self) -> None:
        if self._h is not None:
            lib.qtnh_tensor_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    def _new(self, h) -> "Tensor":
        return Tensor(self.ctx_rank, h)


# ---- ops (ops.hpp) -----------------------------------------------------------------------


class ops:  # namespace
    @staticmethod
    def permute(t: Tensor, perm: Sequence[int], new_split: int) -> Tensor:
        if len(perm) != lib.qtnh_tensor_rank(t._h):
            raise InvalidArgument("permutation size does not match tensor rank")
        h = C.c_void_p()
        check(lib.qtnh_permute(t._h, i32_array(perm), int(new_split), C.byref(h)))
        return t._new(h)

    @staticmethod
    def remap(t: Tensor, axis_map: Sequence[int], dst: IndexTuple, dst_dist=None) -> Tensor:
        """remap::tensor_to_tensor (remap.hpp:106-161), dense variant: axis_map[src]
        = dst position; local destination dims may exceed the source's (zeros)."""
        h = C.c_void_p()
        dd = _dist(dst_dist).as_array() if dst_dist is not None else None
        check(lib.qtnh_remap(t._h, i32_array(axis_map), dst.n_idx(), i64_array(dst.dims), dst.split, dd, C.byref(h)))
        return t._new(h)

    @staticmethod
    def rebcast(t: Tensor, new_dist) -> Tensor:
        h = C.c_void_p()
        check(lib.qtnh_rebcast(t._h, _dist(new_dist).as_array(), C.byref(h)))
        return t._new(h)

    @staticmethod
    def scatter_index(t: Tensor, pos: int) -> Tensor:
        h = C.c_void_p()
        check(lib.qtnh_scatter_index(t._h, int(pos), C.byref(h)))
        return t._new(h)

    @staticmethod
    def gather_index(t: Tensor, pos: int) -> Tensor:
        h = C.c_void_p()
        check(lib.qtnh_gather_index(t._h, int(pos), C.byref(h)))
        return t._new(h)

    @staticmethod
    def squeeze(t: Tensor, pos: int) -> Tensor:
        """ops::squeeze (ops.hpp:234-244): drop a size-1 index (metadata only)."""
        h = C.c_void_p()
        check(lib.qtnh_squeeze(t._h, int(pos), C.byref(h)))
        return t._new(h)

    @staticmethod
    def unsqueeze(t: Tensor, pos: int, as_dist: bool = False) -> Tensor:
        """ops::unsqueeze (ops.hpp:248-262): insert a size-1 index at pos."""
        h = C.c_void_p()
        check(lib.qtnh_unsqueeze(t._h, int(pos), int(bool(as_dist)), C.byref(h)))
        return t._new(h)

    @staticmethod
    def conj(t: Tensor) -> Tensor:
        h = C.c_void_p()
        check(lib.qtnh_conj(t._h, C.byref(h)))
        return t._new(h)

    @staticmethod
    def scale(t: Tensor, alpha: complex) -> Tensor:
        h = C.c_void_p()
        check(lib.qtnh_scale(t._h, float(np.real(alpha)), float(np.imag(alpha)), C.byref(h)))
        return t._new(h)

    @staticmethod
    def slice_local_dims(t: Tensor, new_local_dims: Sequence[int]) -> Tensor:
        h = C.c_void_p()
        check(lib.qtnh_slice_local_dims(t._h, i64_array(new_local_dims), C.byref(h)))
        return t._new(h)

    @staticmethod
    def pad_local_dims(t: Tensor, new_local_dims: Sequence[int]) -> Tensor:
        h = C.c_void_p()
        check(lib.qtnh_pad_local_dims(t._h, i64_array(new_local_dims), C.byref(h)))
        return t._new(h)


def contract(a: Tensor, b: Tensor, a_pos: Sequence[int], b_pos: Sequence[int]) -> Tensor:
    """Contract a[a_pos[i]] with b[b_pos[i]]; result = open(a) then open(b)
    (SPEC.md:408), DistParams of a."""
    if len(a_pos) != len(b_pos):
        raise InvalidArgument("contracted position lists differ in length")
    h = C.c_void_p()
    check(lib.qtnh_contract(a._h, b._h, len(a_pos), i32_array(a_pos), i32_array(b_pos), C.byref(h)))
    return a._new(h)


def contract_host(rank: Rank, a: np.ndarray, b: np.ndarray, a_pos: Sequence[int], b_pos: Sequence[int],
                  out: Optional[np.ndarray] = None) -> np.ndarray:
    """Contraction of host arrays (open(a) then open(b) order), streamed through the
    GPU with H2D / GEMM / D2H overlapped; pass pinned arrays for full overlap."""
    a = np.ascontiguousarray(a, dtype=np.complex128)
    b = np.ascontiguousarray(b, dtype=np.complex128)
    if len(a_pos) != len(b_pos):
        raise InvalidArgument("contracted position lists differ in length")
    odims = [a.shape[i] for i in range(a.ndim) if i not in a_pos] + [b.shape[i] for i in range(b.ndim) if i not in b_pos]
    if out is None:
        out = np.empty(odims, dtype=np.complex128)
    cd = i64_array([0] * max(1, len(odims)))
    check(lib.qtnh_contract_host(rank._h, a.ndim, i64_array(a.shape), a.ctypes.data, b.ndim, i64_array(b.shape),
                                 b.ctypes.data, len(a_pos), i32_array(a_pos), i32_array(b_pos), out.ctypes.data, cd))
    rank.synchronize()
    return out.reshape(odims)


def apply_gate(state: Tensor, targets: Sequence[int], gate, diagonal: bool = False) -> Tensor:
    """In-place gate (row index = gate output, targets[0] most significant).
    Values equal contract(state, gate) followed by a permute back."""
    g = _as_c128(gate)
    check(lib.qtnh_gate_apply(state._h, len(targets), i32_array(targets), g.ctypes.data, int(bool(diagonal))))
    return state


def apply_gate_tensor(state: Tensor, targets: Sequence[int], gate: Tensor) -> Tensor:
    """In-place gate given as a replicated tensor (outputs; inputs) of any variant: a
    DIAGONAL gate runs the diagonal kernel from its stored diagonal (no exchange even on
    distributed targets), IDENTITY does nothing, a two-target SWAP exchanges the indices."""
    check(lib.qtnh_gate_apply_tensor(state._h, len(targets), i32_array(targets), gate._h))
    return state


def swap_indices(state: Tensor, a: int, b: int) -> Tensor:
    """In place: exchange indices a and b (equal dims) -- the values of
    ops::permute with the two positions swapped."""
    check(lib.qtnh_swap_indices(state._h, int(a), int(b)))
    return state


def qft_layer(state: Tensor, j: int) -> Tensor:
    """In place: H on qubit j followed by all controlled phases of QFT layer j, one pass."""
    check(lib.qtnh_qft_layer(state._h, int(j)))
    return state


def qft(state: Tensor, swaps: bool = True) -> Tensor:
    """In place: the whole QFT (cache-blocked layers + bit-reversal SWAP network)."""
    check(lib.qtnh_qft(state._h, int(bool(swaps))))
    return state


# ---- factorisation (linalg.hpp:441-523; SPEC network::decompose) ---------------------------
ABSORB_NONE, ABSORB_LEFT, ABSORB_RIGHT, ABSORB_SPLIT = 0, 1, 2, 3


def svd(t: Tensor, row_pos: Sequence[int], col_pos: Sequence[int], chi: int = 0, absorb: int = ABSORB_NONE):
    """Thin SVD of t viewed as a matrix (rows = row_pos, cols = col_pos), keeping the
    chi largest triplets and zero-padding to exactly chi (linalg.hpp:476-505), with
    the singular values absorbed per ``absorb`` (linalg.hpp:508-523).
    Returns (U tensor [rows..., chi], s numpy (chi,), Vh tensor [chi, cols...])."""
    u, vh = C.c_void_p(), C.c_void_p()
    sh = t.shape()
    m = int(np.prod([sh.dims[p] for p in row_pos], dtype=np.int64))
    n = int(np.prod([sh.dims[p] for p in col_pos], dtype=np.int64))
    k = chi if chi > 0 else min(m, n)
    s = np.zeros(k, dtype=np.float64)
    check(lib.qtnh_svd(t._h, len(row_pos), i32_array(row_pos), len(col_pos), i32_array(col_pos), int(chi),
                       int(absorb), C.byref(u), C.byref(vh), s.ctypes.data))
    return t._new(u), s, t._new(vh)
