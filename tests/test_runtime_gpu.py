"""The rank runtime, mirroring proj/tests/test_runtime.cpp: all_to_all_v ring and
conservation, count-mismatch ProtocolError naming the pair, member-only groups,
abort without deadlock -- on device buffers, ranks as host threads on one GPU."""
import ctypes as C

import numpy as np
import pytest

from paper_2505_06119_b200 import qtnh
from paper_2505_06119_b200._lib import i32_array, i64_array, lib
from paper_2505_06119_b200.qtnh import AbortedError, InvalidArgument, ProtocolError, World

pytestmark = pytest.mark.gpu


def a2a(rk, members, send, scounts, sdispl, rcounts, rdispl):
    import torch

    s = torch.from_numpy(np.ascontiguousarray(send)).cuda()
    r = torch.zeros(max(1, int(sum(rcounts))), dtype=torch.complex128, device="cuda")
    torch.cuda.synchronize()
    qtnh.check(lib.qtnh_all_to_all_v(rk._h, len(members), i32_array(members), C.c_void_p(s.data_ptr()),
                                     i64_array(scounts), i64_array(sdispl), C.c_void_p(r.data_ptr()),
                                     i64_array(rcounts), i64_array(rdispl)))
    rk.synchronize()
    return r.cpu().numpy()


def test_all_to_all_v_ring_and_conservation():
    # test_runtime.cpp:82-164: every rank sends (rank+1) items to its right neighbour
    n = 5

    def body(rk):
        me = rk.rank()
        members = list(range(n))
        right, left = (me + 1) % n, (me - 1) % n
        send = np.array([complex(me, k) for k in range(me + 1)])
        sc = [0] * n
        sc[right] = me + 1
        rc = [0] * n
        rc[left] = left + 1
        got = a2a(rk, members, send, sc, [0] * n, rc, [0] * n)[: left + 1]
        assert np.array_equal(got, np.array([complex(left, k) for k in range(left + 1)]))
        # conservation: all-to-all of one item from everyone to everyone
        send = np.array([complex(me, j) for j in range(n)])
        got = a2a(rk, members, send, [1] * n, list(range(n)), [1] * n, list(range(n)))
        assert np.array_equal(got, np.array([complex(j, me) for j in range(n)]))
        return True

    assert all(World(n).run(body))


def test_count_mismatch_is_a_protocol_error_naming_the_pair():
    # test_runtime.cpp:166-181
    def body(rk):
        me = rk.rank()
        send = np.zeros(4, complex)
        if me == 0:
            return a2a(rk, [0, 1], send, [0, 3], [0, 0], [0, 0], [0, 0])
        return a2a(rk, [0, 1], send, [0, 0], [0, 0], [2, 0], [0, 0])

    with pytest.raises(ProtocolError, match=r"\(0 -> 1\)"):
        World(2).run(body)


def test_disjoint_member_groups_do_not_block_each_other():
    # test_runtime.cpp:66-80: groups {0,1} and {2,3} exchange independently
    def body(rk):
        me = rk.rank()
        pair = [0, 1] if me < 2 else [2, 3]
        other = pair[1] if me == pair[0] else pair[0]
        send = np.array([complex(me, 0)])
        sc = [1 if m == other else 0 for m in pair]
        got = a2a(rk, pair, send, sc, [0, 0], sc, [0, 0])
        assert got[0] == complex(other, 0)
        return True

    assert all(World(4).run(body))


def test_group_membership_validation():
    def body(rk):
        with pytest.raises(InvalidArgument):
            a2a(rk, [1, 1], np.zeros(1, complex), [0, 0], [0, 0], [0, 0], [0, 0])
        with pytest.raises(InvalidArgument):
            a2a(rk, [5], np.zeros(1, complex), [0], [0], [0], [0])
        return True

    assert all(World(2).run(body))


def test_abort_without_deadlock():
    # test_runtime.cpp:216-224: one rank throws, the others leave their collective
    def body(rk):
        if rk.rank() == 2:
            raise RuntimeError("injected failure")
        a2a(rk, [0, 1, 2], np.zeros(1, complex), [0, 0, 0], [0, 0, 0], [0, 0, 0], [0, 0, 0])

    with pytest.raises(RuntimeError, match="injected failure"):
        World(3).run(body)
