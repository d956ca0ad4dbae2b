"""CPU: exhaustive-ish check of the distributed redistribution plans.

For random shapes, splits, permutations and broadcast patterns (stretch, cycles,
offset) on worlds of up to 8 ranks, every rank's host-only plan
(qtnh_remap_plan_json = the plan_remap() the device executor runs) is executed
in one process with numpy: packs, the exchange matched per (src, dst) pair in
order, unpacks. The assembled destination must equal ops::permute of the
reference semantics bit for bit on every copy, and impossible spans must raise
ResourceError with the reference's required rank count."""
import ctypes as C
import json

import numpy as np
import pytest

from paper_2505_06119_b200 import circuits
from paper_2505_06119_b200._lib import i32_array, i64_array, lib
from paper_2505_06119_b200.qtnh import ResourceError, check

from test_multiprocess_cpu import locate, strided_copy


def plan(dims, split, dist, perm, new_split, new_dist, rank, world):
    buf = C.create_string_buffer(1 << 18)
    check(lib.qtnh_remap_plan_json(len(dims), i64_array(dims), split, i64_array(dist), i32_array(perm), new_split,
                                   i64_array(new_dist), rank, world, buf, 1 << 18))
    return json.loads(buf.value.decode())


def simulate(dims, split, dist, perm, new_split, new_dist, world, g):
    total = int(np.prod(dims))
    snd = int(np.prod(dims[:split]))
    nl_src = total // snd
    ndims = [dims[p] for p in perm]
    dnd = int(np.prod(ndims[:new_split]))
    nl_dst = total // dnd
    plans = [plan(dims, split, dist, perm, new_split, new_dist, r, world) for r in range(world)]
    src, dst, send, recv = {}, {}, {}, {}
    for r in range(world):
        loc = locate(r, snd, dist)
        if loc:
            src[r] = g[loc[0] * nl_src:(loc[0] + 1) * nl_src].copy()
        if locate(r, dnd, new_dist):
            dst[r] = np.full(nl_dst, np.nan + 0j)
    for r, p in enumerate(plans):
        if not p["member"]:
            continue
        if p["local_only"]:
            if p["src_canonical"] and r in dst:
                strided_copy(src[r], dst[r], p["pack"], True)
            continue
        if p["src_canonical"]:
            if p["pack_to_dst"]:
                strided_copy(src[r], dst[r], p["pack"], True)
                send[r] = dst[r]
            else:
                send[r] = np.empty(p["pack_elems"], np.complex128)
                strided_copy(src[r], send[r], p["pack"], True)
        if r in dst:
            recv[r] = dst[r] if p["recv_into_dst"] else np.empty(p["recv_elems"], np.complex128)
    # exchange: chunks matched in order per (src, dst)
    outbox = {}
    for r, p in enumerate(plans):
        if p["member"] and not p["local_only"]:
            for peer, off, cnt in p["sends"]:
                outbox.setdefault((r, peer), []).append(send[r][off:off + cnt].copy())
    for r, p in enumerate(plans):
        if p["member"] and not p["local_only"]:
            for peer, off, cnt in p["recvs"]:
                chunk = outbox[(peer, r)].pop(0)
                assert chunk.size == cnt, f"count mismatch ({peer} -> {r})"
                recv[r][off:off + cnt] = chunk
    assert all(not v for v in outbox.values()), "unreceived chunks"
    for r, p in enumerate(plans):
        if p["member"] and not p["local_only"] and r in dst and p["unpack"]:
            strided_copy(recv[r], dst[r], p["unpack_box"], False)
    glob = np.full(dnd * nl_dst, np.nan + 0j)
    seen = {}
    for r, d in dst.items():
        b = locate(r, dnd, new_dist)[0]
        if b in seen:
            assert np.array_equal(seen[b].view(np.uint64), d.view(np.uint64)), "broadcast copies differ"
        seen[b] = d
        glob[b * nl_dst:(b + 1) * nl_dst] = d
    return glob


def simulate_push(dims, split, dist, perm, new_split, new_dist, world, g):
    """Peer-memory form: every canonical source holder stores its chunks straight
    into the homes' destination blocks."""
    total = int(np.prod(dims))
    snd = int(np.prod(dims[:split]))
    nl_src = total // snd
    ndims = [dims[p] for p in perm]
    dnd = int(np.prod(ndims[:new_split]))
    nl_dst = total // dnd
    dst = {r: np.full(nl_dst, np.nan + 0j) for r in range(world) if locate(r, dnd, new_dist)}
    for r in range(world):
        p = plan(dims, split, dist, perm, new_split, new_dist, r, world)
        if not p["member"]:
            continue
        loc = locate(r, snd, dist)
        src = g[loc[0] * nl_src:(loc[0] + 1) * nl_src] if loc else None
        if p["local_only"]:  # same single-launch path as the exchange form
            if p["src_canonical"] and r in dst:
                strided_copy(src, dst[r], p["pack"], True)
            continue
        for peer, so, do in p["pushes"]:
            box = p["push_box"]
            strided_copy(src[so:], dst[peer][do:], box, True)
    glob = np.full(dnd * nl_dst, np.nan + 0j)
    for r, d in dst.items():
        b = locate(r, dnd, new_dist)[0]
        glob[b * nl_dst:(b + 1) * nl_dst] = d
    return glob


def test_random_plans_bit_exact():
    import oracle

    P = oracle.port()
    rng = np.random.default_rng(7)
    checked = raised = 0
    for trial in range(400):
        r = int(rng.integers(1, 6))
        dims = [int(x) for x in rng.integers(1, 4, size=r)]
        world = int(rng.integers(1, 9))
        split = int(rng.integers(0, r + 1))
        while int(np.prod(dims[:split])) > world:
            split -= 1
        nd = int(np.prod(dims[:split]))
        st = int(rng.integers(1, 3))
        cy = int(rng.integers(1, 3))
        while st * cy * nd > world:
            if cy > 1:
                cy -= 1
            elif st > 1:
                st -= 1
        off = int(rng.integers(0, world - st * cy * nd + 1))
        perm = [int(x) for x in rng.permutation(r)]
        new_split = int(rng.integers(0, r + 1))
        ndims = [dims[p] for p in perm]
        dnd = int(np.prod(ndims[:new_split]))
        nst, ncy = int(rng.integers(1, 3)), int(rng.integers(1, 3))
        noff = int(rng.integers(0, 3))
        total = int(np.prod(dims))
        g = np.array([complex(i + 1, -0.5 * i) if i % 4 else complex(-0.0, -0.0) for i in range(total)])
        need = noff + nst * ncy * dnd
        if need > world:
            with pytest.raises(ResourceError) as e:
                plan(dims, split, (st, cy, off), perm, new_split, (nst, ncy, noff), 0, world)
            assert e.value.required_ranks == need
            raised += 1
            continue
        got = simulate(dims, split, (st, cy, off), perm, new_split, (nst, ncy, noff), world, g)
        want = P.permute(dims, g, perm)
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), (dims, split, perm, new_split, world)
        got = simulate_push(dims, split, (st, cy, off), perm, new_split, (nst, ncy, noff), world, g)
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), ("push", dims, split, perm, world)
        checked += 1
    assert checked > 150 and raised > 10
