"""CPU, world_size 2 over gloo: the process-per-GPU (N > 1) redistribution path.

Each process is one rank. It asks libqtnh_b200 for its host-only exchange plan
(qtnh_remap_plan_json -- the same plan_remap() the device executor runs before
its pack kernel / NCCL send-recv / unpack kernel), executes the plan with numpy
strided copies and torch.distributed gloo point-to-point transfers, and the
assembled global tensor must equal the reference semantics bit for bit.
"""
import ctypes as C
import json
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.timeout(300)

CASES = [
    # (dims, split, dist, perm, new_split, new_dist)
    ([2, 2, 2, 2, 2, 2], 1, (1, 1, 0), [5, 1, 2, 3, 4, 0], 1, None),   # dist <-> local swap
    ([2, 2, 2, 2, 2], 0, (1, 1, 0), [3, 0, 1, 2, 4], 1, None),         # scatter: span 1 -> 2
    ([2, 3, 2, 4], 1, (1, 1, 0), [1, 0, 2, 3], 0, None),               # gather: span 2 -> 1
    ([2, 3, 5], 1, (1, 1, 0), [0, 1, 2], 1, (1, 1, 0)),                # identity (no-op plan)
    ([2, 3, 5], 0, (1, 1, 0), [0, 1, 2], 0, (2, 1, 0)),                # rebcast: stretch 2
    ([2, 3, 5], 0, (1, 1, 1), [2, 1, 0], 0, (1, 1, 0)),                # move from rank 1 to rank 0
    ([2, 2, 3, 2], 1, (1, 1, 0), [1, 3, 0, 2], 1, (1, 1, 0)),          # full shuffle, dims 3 local
    ([2, 2, 2, 2, 2, 2, 2, 2], 1, (1, 1, 0), [7, 3, 6, 0, 2, 1, 5, 4], 1, None),
]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def strided_copy(src, dst, box, canon):
    from numpy.lib.stride_tricks import as_strided

    dims = box["dims"]
    if not dims:
        v = src[0]
        if canon and v.real == 0 and v.imag == 0:
            v = 0j
        dst[0] = v
        return
    sv = as_strided(src, shape=dims, strides=[s * 16 for s in box["in_stride"]])
    dv = as_strided(dst, shape=dims, strides=[s * 16 for s in box["out_stride"]], writeable=True)
    vals = np.array(sv)
    if canon:
        vals[(vals.real == 0) & (vals.imag == 0)] = 0
    dv[...] = vals


def locate(rank, nd, dist):
    st, cyc, off = dist
    r = rank - off
    if r < 0 or r >= st * cyc * nd:
        return None
    per = st * nd
    return (r % per) // st, r // per, r % st  # block, cycle, slot


def run_plan(rank, world, case):
    import torch
    import torch.distributed as dist

    from paper_2505_06119_b200._lib import i32_array, i64_array, lib
    from paper_2505_06119_b200.qtnh import check

    dims, split, sdist, perm, new_split, new_dist = case
    ddist = tuple(new_dist) if new_dist else tuple(sdist)
    n = len(dims)
    buf = C.create_string_buffer(1 << 16)
    check(lib.qtnh_remap_plan_json(n, i64_array(dims), split, i64_array(sdist), i32_array(perm), new_split,
                                   i64_array(ddist) if new_dist else None, rank, world, buf, 1 << 16))
    plan = json.loads(buf.value.decode())
    total = int(np.prod(dims))
    g = np.array([complex(i + 1, -0.5 * i) if i % 5 else complex(-0.0, -0.0) for i in range(total)])
    snd = int(np.prod(dims[:split]))
    nl_src = total // snd
    loc = locate(rank, snd, sdist)
    src = g[loc[0] * nl_src:(loc[0] + 1) * nl_src].copy() if loc else None
    ndims = [dims[p] for p in perm]
    dnd = int(np.prod(ndims[:new_split]))
    nl_dst = total // dnd
    dloc = locate(rank, dnd, ddist)
    dst = np.full(nl_dst, np.nan + 0j) if dloc else None
    if plan["member"]:
        if plan["local_only"]:
            if plan["src_canonical"] and dloc:
                strided_copy(src, dst, plan["pack"], True)
        else:
            send = None
            if plan["src_canonical"]:
                if plan["pack_to_dst"]:
                    strided_copy(src, dst, plan["pack"], True)
                    send = dst
                else:
                    send = np.empty(plan["pack_elems"], np.complex128)
                    strided_copy(src, send, plan["pack"], True)
            recv = None
            if dloc:
                recv = dst if plan["recv_into_dst"] else np.empty(plan["recv_elems"], np.complex128)
            reqs, self_sends, tags = [], [], {}
            for peer, off, cnt in plan["sends"]:
                k = tags.setdefault(("s", peer), 0)
                tags[("s", peer)] += 1
                if peer == rank:
                    self_sends.append((off, cnt))
                    continue
                t = torch.from_numpy(send[off:off + cnt].view(np.float64))
                reqs.append(dist.isend(t, dst=peer, tag=k))
            pending = []
            for peer, off, cnt in plan["recvs"]:
                k = tags.setdefault(("r", peer), 0)
                tags[("r", peer)] += 1
                if peer == rank:
                    so, sc = self_sends.pop(0)
                    assert sc == cnt
                    recv[off:off + cnt] = send[so:so + sc]
                    continue
                t = torch.empty(2 * cnt, dtype=torch.float64)
                reqs.append(dist.irecv(t, src=peer, tag=k))
                pending.append((off, cnt, t))
            for r in reqs:
                r.wait()
            for off, cnt, t in pending:
                recv[off:off + cnt] = t.numpy().view(np.complex128)
            if dloc and plan["unpack"]:
                strided_copy(recv, dst, plan["unpack_box"], False)
    mine = (dloc[0], dst) if dloc else None
    allb = [None] * world
    dist.all_gather_object(allb, mine)
    return g, allb, ndims, dnd, nl_dst, plan


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = []
    try:
        for case in CASES:
            g, allb, ndims, dnd, nl, plan = run_plan(rank, world, case)
            if rank == 0:
                glob = np.full(dnd * nl, np.nan + 0j)
                copies = {}
                for item in allb:
                    if item is None:
                        continue
                    b, data = item
                    if b in copies:
                        assert np.array_equal(copies[b].view(np.uint64), data.view(np.uint64)), "copies differ"
                    copies[b] = data
                    glob[b * nl:(b + 1) * nl] = data
                out.append((case, glob, g, len(plan["sends"]), len(plan["recvs"])))
        q.put(("ok", out) if rank == 0 else ("ok", None))
    except Exception as e:  # surface to the parent
        import traceback

        q.put(("err", traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def test_two_process_gloo_redistribution_bit_exact():
    import multiprocessing as mp

    import oracle

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    errs = [r[1] for r in res if r[0] == "err"]
    assert not errs, errs[0]
    out = [r[1] for r in res if r[1] is not None][0]
    P = oracle.port()
    moved = 0
    for case, glob, g, ns, nr in out:
        dims, split, sdist, perm, new_split, new_dist = case
        want = P.permute(dims, g, perm)
        assert np.array_equal(glob.view(np.uint64), want.view(np.uint64)), case
        moved += ns + nr
    assert moved > 0  # at least some cases really exchange data between the ranks


def test_plan_raises_resource_error_like_the_reference():
    from paper_2505_06119_b200._lib import i32_array, i64_array, lib
    from paper_2505_06119_b200.qtnh import ResourceError, check

    buf = C.create_string_buffer(1 << 12)
    # asymmetric permutation (2;2,4,2) -> (4;2,2,2) needs 4 ranks (test_ops.cpp:102-109)
    with pytest.raises(ResourceError) as e:
        check(lib.qtnh_remap_plan_json(4, i64_array([2, 2, 4, 2]), 1, i64_array([1, 1, 0]),
                                       i32_array([2, 0, 1, 3]), 1, None, 0, 2, buf, 1 << 12))
    assert e.value.required_ranks == 4
