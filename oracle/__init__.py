"""Oracle -- TEST INFRASTRUCTURE ONLY.

Two CPU checkers for the B200 hot path:

* ``ref``: the UNMODIFIED reference (/root/reference/proj/include/qtnh) compiled
  with oracle/ref_driver.cpp into oracle/_ref/libqtnh_ref.so (``make -C oracle
  ref``; needs the reference sources, so it is built in the build container and
  travels to the GPU box as a prebuilt .so).
* ``port``: the plain-C restatement oracle/qtnh_oracle.c
  (oracle/_build/libqtnh_oracle.so), pinned against ``ref`` and the reference's
  own known-answer tests in tests/test_oracle.py.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference arm
may import this package; the product path (paper_2505_06119_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Optional, Sequence, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libqtnh_ref.so")
PORT_SO = os.path.join(HERE, "_build", "libqtnh_oracle.so")

i32, i64, f64, vp, u64 = C.c_int, C.c_int64, C.c_double, C.c_void_p, C.c_uint64


def build(ref: bool = True) -> None:
    """Compile the port (always) and the reference (when /root/reference exists)."""
    subprocess.run(["make", "-C", HERE, "port"], check=True, capture_output=True)
    if ref and os.path.isdir("/root/reference/proj/include"):
        subprocess.run(["make", "-C", HERE, "ref"], check=True, capture_output=True)


def _i64(v):
    v = list(v)
    return (C.c_int64 * max(1, len(v)))(*v)


def _i32(v):
    v = list(v)
    return (C.c_int * max(1, len(v)))(*v)


def _c128(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.complex128))


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str, info: int):
        super().__init__(f"[{code}] {msg}")
        self.code, self.msg, self.info = code, msg, info


# ---- the reference (compiled headers) -------------------------------------------------
class _Ref:
    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where /root/reference exists")
        self.lib = L = C.CDLL(path)
        L.qref_last_error.argtypes = [C.c_char_p, i32]
        L.qref_last_info.restype = C.c_longlong
        L.qref_hash_counter.restype = u64
        L.qref_hash_counter.argtypes = [u64, u64, u64, u64]
        L.qref_rng_complex_normals.argtypes = [u64, i64, vp]
        L.qref_set_threads.argtypes = [i32]
        P64, P32 = C.POINTER(C.c_int64), C.POINTER(C.c_int)
        L.qref_permute.argtypes = [i32, i32, P64, i32, P64, vp, P32, i32, vp, P64, P32, P64]
        L.qref_rebcast.argtypes = [i32, i32, P64, i32, P64, vp, P64, vp, P64]
        L.qref_scatter_gather.argtypes = [i32, i32, i32, P64, i32, P64, vp, i32, vp, P64, P32]
        L.qref_slice_pad.argtypes = [i32, i32, i32, P64, i32, P64, vp, P64, vp]
        L.qref_contract.argtypes = [i32, i32, P64, i32, P64, vp, i32, P64, i32, P64, vp, i32, P32, P32,
                                    vp, P64, P32, vp]
        L.qref_gate.argtypes = [i32, i32, i32, P64, vp, i32, P32, vp, vp]
        L.qref_qft.argtypes = [i32, i32, i32, vp, i32, i32, vp, vp]
        L.qref_svd.argtypes = [i32, i64, i64, vp, i64, i32, vp, vp, vp, vp]
        L.qref_save.argtypes = [i32, i32, P64, i32, P64, vp, C.c_char_p]
        L.qref_load.argtypes = [i32, C.c_char_p, P64, P32, P32, P64, vp, i64]

    def _check(self, rc):
        if rc:
            buf = C.create_string_buffer(4096)
            self.lib.qref_last_error(buf, 4096)
            raise OracleError(rc, buf.value.decode(), int(self.lib.qref_last_info()))

    def set_threads(self, n: int):
        self.lib.qref_set_threads(n)

    def hash_counter(self, seed, k0=0, k1=0, k2=0) -> int:
        return int(self.lib.qref_hash_counter(seed, k0, k1, k2))

    def rng_complex_normals(self, seed: int, count: int) -> np.ndarray:
        out = np.empty(count, np.complex128)
        self.lib.qref_rng_complex_normals(seed, count, out.ctypes.data)
        return out

    def permute(self, world, dims, split, dist, data, perm, new_split):
        data = _c128(data)
        out = np.empty(data.size, np.complex128)
        od, os_, odist = _i64([0] * len(dims)), (C.c_int * 1)(), _i64([0, 0, 0])
        self._check(self.lib.qref_permute(world, len(dims), _i64(dims), split, _i64(dist or (1, 1, 0)),
                                          data.ctypes.data, _i32(perm), new_split, out.ctypes.data, od,
                                          os_, odist))
        return out, [od[i] for i in range(len(dims))], os_[0], (odist[0], odist[1], odist[2])

    def rebcast(self, world, dims, split, dist, data, new_dist):
        data = _c128(data)
        out = np.empty(data.size, np.complex128)
        odist = _i64([0, 0, 0])
        self._check(self.lib.qref_rebcast(world, len(dims), _i64(dims), split, _i64(dist or (1, 1, 0)),
                                          data.ctypes.data, _i64(new_dist), out.ctypes.data, odist))
        return out

    def scatter_gather(self, world, op, dims, split, dist, data, pos):
        data = _c128(data)
        out = np.empty(data.size, np.complex128)
        od, os_ = _i64([0] * len(dims)), (C.c_int * 1)()
        self._check(self.lib.qref_scatter_gather(world, op, len(dims), _i64(dims), split,
                                                 _i64(dist or (1, 1, 0)), data.ctypes.data, pos,
                                                 out.ctypes.data, od, os_))
        return out, [od[i] for i in range(len(dims))], os_[0]

    def slice_pad(self, world, op, dims, split, dist, data, new_local):
        data = _c128(data)
        nd = list(dims[:split]) + list(new_local)
        out = np.empty(int(np.prod(nd)), np.complex128)
        self._check(self.lib.qref_slice_pad(world, op, len(dims), _i64(dims), split, _i64(dist or (1, 1, 0)),
                                            data.ctypes.data, _i64(new_local), out.ctypes.data))
        return out

    def contract(self, world, da, sa, dista, a, db, sb, distb, b, apos, bpos, timing=False):
        a, b = _c128(a), _c128(b)
        ca = [i for i in range(len(da)) if i not in apos]
        cb = [i for i in range(len(db)) if i not in bpos]
        n_out = int(np.prod([da[i] for i in ca] + [db[i] for i in cb]))
        out = np.empty(n_out, np.complex128)
        od, os_ = _i64([0] * (len(ca) + len(cb))), (C.c_int * 1)()
        t = (C.c_double * 4)()
        self._check(self.lib.qref_contract(world, len(da), _i64(da), sa, _i64(dista or (1, 1, 0)), a.ctypes.data,
                                           len(db), _i64(db), sb, _i64(distb or (1, 1, 0)), b.ctypes.data,
                                           len(apos), _i32(apos), _i32(bpos), out.ctypes.data, od, os_, t))
        res = (out, [od[i] for i in range(len(ca) + len(cb))], os_[0])
        return res + ([t[i] for i in range(4)],) if timing else res

    def gate(self, world, n, split, dist, state, targets, gate):
        state = _c128(state)
        g = _c128(gate)
        out = np.empty(state.size, np.complex128)
        self._check(self.lib.qref_gate(world, n, split, _i64(dist or (1, 1, 0)), state.ctypes.data,
                                       len(targets), _i32(targets), g.ctypes.data, out.ctypes.data))
        return out

    def qft(self, n, state, swaps=True, world=1, split=0, gate_limit=-1, timing=False):
        state = _c128(state)
        out = np.empty(state.size, np.complex128)
        t = (C.c_double * 1)()
        self._check(self.lib.qref_qft(world, n, split, state.ctypes.data, int(swaps), gate_limit,
                                      out.ctypes.data, t))
        return (out, t[0]) if timing else out

    def save(self, world, dims, split, dist, data, path):
        data = _c128(data)
        self._check(self.lib.qref_save(world, len(dims), _i64(dims), split, _i64(dist or (1, 1, 0)),
                                       data.ctypes.data, path.encode()))

    def load(self, world, path, cap=1 << 24):
        dims, nd, split, dist = _i64([0] * 64), (C.c_int * 1)(), (C.c_int * 1)(), _i64([0, 0, 0])
        out = np.empty(cap, np.complex128)
        self._check(self.lib.qref_load(world, path.encode(), dims, nd, split, dist, out.ctypes.data, cap))
        n = nd[0]
        d = [dims[i] for i in range(n)]
        return d, split[0], (dist[0], dist[1], dist[2]), out[: int(np.prod(d)) if d else 1].copy()

    def svd(self, a: np.ndarray, chi: int = 0, absorb: int = 0, world: int = 1, timing=False):
        a = _c128(a)
        m, n = a.shape
        keep = chi if chi > 0 else min(m, n)
        u = np.empty((m, keep), np.complex128)
        s = np.empty(keep, np.float64)
        vh = np.empty((keep, n), np.complex128)
        t = (C.c_double * 2)()
        self._check(self.lib.qref_svd(world, m, n, a.ctypes.data, chi, absorb, u.ctypes.data, s.ctypes.data,
                                      vh.ctypes.data, t))
        return (u, s, vh, [t[0], t[1]]) if timing else (u, s, vh)


# ---- the C restatement ---------------------------------------------------------------
class _Port:
    def __init__(self, path: str = PORT_SO):
        if not os.path.exists(path):
            build(ref=False)
        self.lib = L = C.CDLL(path)
        L.qo_hash_counter.restype = u64
        L.qo_hash_counter.argtypes = [u64, u64, u64, u64]
        L.qo_u64_to_unit.restype = f64
        L.qo_u64_to_unit.argtypes = [u64]
        L.qo_rng_complex_normals.argtypes = [u64, i64, vp]
        L.qo_counter_normals.argtypes = [u64, i64, i64, vp]
        L.qo_counter_normals_at.argtypes = [u64, vp, i64, vp]
        P64, P32 = C.POINTER(C.c_int64), C.POINTER(C.c_int)
        L.qo_permute.argtypes = [i32, P64, vp, P32, vp]
        L.qo_contract.argtypes = [i32, P64, vp, i32, P64, vp, i32, P32, P32, vp]
        L.qo_gate.argtypes = [i32, P64, vp, i32, P32, vp, i32]
        L.qo_qft.argtypes = [i32, vp, i32]

    def hash_counter(self, seed, k0=0, k1=0, k2=0) -> int:
        return int(self.lib.qo_hash_counter(seed, k0, k1, k2))

    def rng_complex_normals(self, seed: int, count: int) -> np.ndarray:
        out = np.empty(count, np.complex128)
        self.lib.qo_rng_complex_normals(seed, count, out.ctypes.data)
        return out

    def counter_normals(self, seed: int, start: int, count: int) -> np.ndarray:
        out = np.empty(count, np.complex128)
        self.lib.qo_counter_normals(seed, start, count, out.ctypes.data)
        return out

    def counter_normals_at(self, seed: int, idx) -> np.ndarray:
        idx = np.ascontiguousarray(idx, dtype=np.int64)
        out = np.empty(idx.size, np.complex128)
        self.lib.qo_counter_normals_at(seed, idx.ctypes.data, idx.size, out.ctypes.data)
        return out

    def permute(self, dims, data, perm) -> np.ndarray:
        data = _c128(data)
        out = np.empty(data.size, np.complex128)
        assert self.lib.qo_permute(len(dims), _i64(dims), data.ctypes.data, _i32(perm), out.ctypes.data) == 0
        return out

    def contract(self, da, a, db, b, apos, bpos) -> np.ndarray:
        a, b = _c128(a), _c128(b)
        ca = [i for i in range(len(da)) if i not in apos]
        cb = [i for i in range(len(db)) if i not in bpos]
        out = np.empty(int(np.prod([da[i] for i in ca] + [db[i] for i in cb])), np.complex128)
        assert self.lib.qo_contract(len(da), _i64(da), a.ctypes.data, len(db), _i64(db), b.ctypes.data,
                                    len(apos), _i32(apos), _i32(bpos), out.ctypes.data) == 0
        return out

    def gate(self, dims, state, targets, gate, diagonal=False) -> np.ndarray:
        psi = _c128(state).copy()
        g = _c128(gate)
        assert self.lib.qo_gate(len(dims), _i64(dims), psi.ctypes.data, len(targets), _i32(targets),
                                g.ctypes.data, int(diagonal)) == 0
        return psi

    def qft(self, n, state, swaps=True) -> np.ndarray:
        psi = _c128(state).copy()
        assert self.lib.qo_qft(n, psi.ctypes.data, int(swaps)) == 0
        return psi


_ref: Optional[_Ref] = None
_port: Optional[_Port] = None


def ref() -> _Ref:
    global _ref
    if _ref is None:
        _ref = _Ref()
    return _ref


def port() -> _Port:
    global _port
    if _port is None:
        _port = _Port()
    return _port


def ref_available() -> bool:
    return os.path.exists(REF_SO)


# ---- network replay (numpy) -----------------------------------------------------------
def network_contract(items, order, big_first: bool = True):
    """Replay a pairwise contraction order on the host: `items` = [(array, labels)]
    (tensor i = items[i]), `order` = [(a, b)] with the result of step s getting id
    len(items) + s. Each step is SPEC network::contract: sum over
    the shared labels, result indices open(first) then open(second),
    written with numpy.tensordot (OpenBLAS zgemm on all host cores) -- the same
    contraction the reference composes from t2m -> pgemm -> m2t (linalg.hpp:208-400),
    without its 24-byte-per-element redistribution, so 2^30-element intermediates
    fit in host memory and minutes. Returns (array, labels) of the last result."""
    import math

    T = {i: (np.ascontiguousarray(a, dtype=np.complex128), list(l)) for i, (a, l) in enumerate(items)}
    n = len(items)
    last = None
    for s, (a, b) in enumerate(order):
        (ta, la), (tb, lb) = T.pop(a), T.pop(b)
        if big_first and sum(math.log2(d) for d in tb.shape) > sum(math.log2(d) for d in ta.shape):
            (ta, la), (tb, lb) = (tb, lb), (ta, la)
        sh = [x for x in la if x in lb]
        c = np.tensordot(ta, tb, axes=([la.index(x) for x in sh], [lb.index(x) for x in sh]))
        del ta, tb
        last = n + s
        T[last] = (np.ascontiguousarray(c), [x for x in la if x not in sh] + [x for x in lb if x not in sh])
    return T[last]
