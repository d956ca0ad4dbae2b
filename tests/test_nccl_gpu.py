"""The process-per-GPU backend (NCCL, dlopen'ed): a world of one rank exercises
communicator setup, the NCCL exchange code path (self transfers + grouped
send/recv bookkeeping) and teardown on the single GPU available here."""
import ctypes as C

import numpy as np
import pytest
import torch  # noqa: F401  (first: torch's bundled libnccl must be the process's libnccl.so.2)

import oracle
from conftest import bits, rel_l2
from paper_2505_06119_b200 import circuits, qtnh
from paper_2505_06119_b200._lib import i32_array, lib
from paper_2505_06119_b200.qtnh import DistParams, IndexTuple, Rank, Tensor, contract, ops

pytestmark = pytest.mark.gpu


def test_nccl_world_of_one():
    uid = (C.c_char * 128)()
    qtnh.check(lib.qtnh_nccl_unique_id(uid))
    h = C.c_void_p()
    qtnh.check(lib.qtnh_world_create_nccl(0, 1, 0, uid, C.byref(h)))
    w = qtnh.World.__new__(qtnh.World)
    w._h, w._n, w._nccl_rank = h, 1, 0
    P = oracle.port()
    g = circuits.counter_state(3, 2**10)
    b = circuits.counter_state(4, 2**4)

    def body(rk):
        t = Tensor.from_global(rk, IndexTuple([2] * 10, 0), DistParams(1, 1, 0), g)
        p = ops.permute(t, [9, 1, 2, 3, 4, 5, 6, 7, 8, 0], 0)
        rb = ops.rebcast(t, DistParams(1, 1, 0))  # identity remap through the exchange path
        c = contract(t, Tensor.from_global(rk, IndexTuple([2] * 4, 0), None, b), [2, 5], [0, 3])
        rk.barrier()
        return p.to_global_vector(), rb.to_global_vector(), c.to_global_vector()

    pv, rv, cv = w.run(body)[0]
    assert np.array_equal(bits(pv), bits(P.permute([2] * 10, g, [9, 1, 2, 3, 4, 5, 6, 7, 8, 0])))
    assert np.array_equal(bits(rv), bits(P.permute([2] * 10, g, list(range(10)))))
    assert rel_l2(cv, P.contract([2] * 10, g, [2] * 4, b, [2, 5], [0, 3])) < 1e-12
    w.close()


def test_nccl_world_with_missing_peer_times_out_and_aborts():
    """runtime.hpp:335-345 collective timeout on the NCCL backend: a 2-rank world
    whose second rank never joins fails with ProtocolError after
    QTNH_COLLECTIVE_TIMEOUT_MS (non-blocking ncclCommInitRankConfig polled, then
    ncclCommAbort) instead of blocking forever. Run in a subprocess so the
    timeout setting and the aborted communicator stay out of this process."""
    import os
    import subprocess
    import sys
    import time

    code = r'''
import ctypes as C, sys
sys.path.insert(0, %r)
from paper_2505_06119_b200 import qtnh
from paper_2505_06119_b200._lib import lib
uid = (C.c_char * 128)()
qtnh.check(lib.qtnh_nccl_unique_id(uid))
h = C.c_void_p()
try:
    qtnh.check(lib.qtnh_world_create_nccl(0, 2, 0, uid, C.byref(h)))
    print("CREATED")
except qtnh.ProtocolError as e:
    print("PROTOCOL", e)
''' % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, QTNH_COLLECTIVE_TIMEOUT_MS="3000")
    t0 = time.time()
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=120, env=env)
    assert "PROTOCOL" in r.stdout and "timed out" in r.stdout, (r.stdout, r.stderr[-2000:])
    assert time.time() - t0 < 90


def test_nccl_world_of_one_count_check_and_abort():
    """The NCCL exchange's count bookkeeping (self chunks must match) raises the
    reference's ProtocolError "(src -> dst)"; qtnh_world_abort aborts the
    communicator and later collectives raise AbortedError (runtime.hpp:276-298)."""

    uid = (C.c_char * 128)()
    qtnh.check(lib.qtnh_nccl_unique_id(uid))
    h = C.c_void_p()
    qtnh.check(lib.qtnh_world_create_nccl(0, 1, 0, uid, C.byref(h)))
    w = qtnh.World.__new__(qtnh.World)
    w._h, w._n, w._nccl_rank = h, 1, 0
    buf = torch.zeros(64, dtype=torch.complex128, device="cuda")

    def body(rk):
        p = C.c_void_p(buf.data_ptr())
        m = i32_array([0])
        sc = (C.c_int64 * 1)(4)
        rc = (C.c_int64 * 1)(3)
        z = (C.c_int64 * 1)(0)
        with pytest.raises(qtnh.ProtocolError, match=r"\(0 -> 0\)"):
            qtnh.check(lib.qtnh_all_to_all_v(rk._h, 1, m, p, sc, z, p, rc, z))
        qtnh.check(lib.qtnh_world_abort(w._h))
        with pytest.raises(qtnh.AbortedError):
            qtnh.check(lib.qtnh_all_to_all_v(rk._h, 1, m, p, sc, z, p, sc, z))

    w.run(body)
    w.close()
