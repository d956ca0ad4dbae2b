"""The process-per-GPU backend (NCCL, dlopen'ed): a world of one rank exercises
communicator setup, the NCCL exchange code path (self transfers + grouped
send/recv bookkeeping) and teardown on the single GPU available here."""
import ctypes as C

import numpy as np
import pytest

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
