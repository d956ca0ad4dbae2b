"""GPU parity of the structural ops (permute / rebcast / scatter / gather / slice /
pad) through the C ABI -- bit-exact against the reference.

Mirrors proj/tests/test_ops.cpp case by case; multi-rank worlds are in-process
worlds whose ranks all run on cuda:0 (each on its own stream and host thread,
exactly like the reference's simulated World), so every exchange path runs.
"""
import numpy as np
import pytest

import oracle
from conftest import bits, golden
from paper_2505_06119_b200 import circuits
from paper_2505_06119_b200.qtnh import (AbortedError, DistParams, IndexTuple, InvalidArgument, ResourceError,
                                        Tensor, World, ops, run_collect)

pytestmark = pytest.mark.gpu
P = oracle.port()


def iota_global(n):  # test_ops.cpp:28-32
    return np.array([complex(i + 1, 0.1 * i) for i in range(n)])


def H(seed, k0=0, k1=0, k2=0):
    return circuits.hash_counter(seed, k0, k1, k2)


def random_dims(seed, max_rank):  # test_ops.cpp:51-56
    r = 1 + H(seed, 1) % max_rank
    return [1 + H(seed, 2, i) % 3 for i in range(r)]


def test_identity_permutation_returns_the_tensor_unchanged():
    g = iota_global(16)

    def body(rk):
        t = Tensor.from_global(rk, IndexTuple([2, 2, 4], 1), DistParams(1, 1, 0), g)
        return ops.permute(t, [0, 1, 2], 1).to_global_vector()

    assert np.array_equal(run_collect(World(2), body), g)


def test_matrix_transpose():
    def body(rk):
        t = Tensor.from_global(rk, IndexTuple([2, 2], 0), None, np.array([1, 2, 3, 4], complex))
        return ops.permute(t, [1, 0], 0).to_global_vector()

    assert np.array_equal(run_collect(World(1), body), np.array([1, 3, 2, 4], complex))


def test_asymmetric_permutation_recruits_more_ranks(peer_mode):
    g = iota_global(32)

    def body(rk):
        t = Tensor.from_global(rk, IndexTuple([2, 2, 4, 2], 1), DistParams(1, 1, 0), g)
        assert t.span() == 2
        p = ops.permute(t, [2, 0, 1, 3], 1)
        assert p.span() == 4
        assert p.shape().str() == "(4;2,2,2)"
        return p.to_global_vector()

    got = run_collect(World(4), body)
    assert np.array_equal(got, P.permute([2, 2, 4, 2], g, [2, 0, 1, 3]))

    def small(rk):
        t = Tensor.from_global(rk, IndexTuple([2, 2, 4, 2], 1), DistParams(1, 1, 0), g)
        ops.permute(t, [2, 0, 1, 3], 1)

    with pytest.raises(ResourceError) as e:
        World(2).run(small)
    assert e.value.required_ranks == 4


def test_golden_permutations_bit_exact(peer_mode):
    meta, z = golden("permute")
    for i, m in enumerate(meta):
        gin = z[f"in{i}"]

        def body(rk):
            t = Tensor.from_global(rk, IndexTuple(m["dims"], m["split"]), DistParams(*m["dist"]), gin)
            p = ops.permute(t, m["perm"], m["new_split"])
            return p.shape(), p.to_global_vector() if p.in_span() else None

        res = World(m["world"]).run(body)
        shape, got = res[0]
        assert shape.dims == m["out_dims"] and shape.split == m["out_split"]
        assert np.array_equal(bits(got), bits(z[f"out{i}"])), f"case {i}: {m}"


def test_permutation_round_trip_and_composition(peer_mode):
    # test_ops.cpp:112-159
    for seed in range(8):
        def body(rk, seed=seed):
            dims = random_dims(seed, 5)
            r = len(dims)
            split = H(seed, 3) % (r + 1)
            shape = IndexTuple(dims, split)
            while shape.dist_size() > 4:
                shape.split -= 1
            g = iota_global(shape.total_size())
            t = Tensor.from_global(rk, shape, DistParams(1, 1, 0), g)
            p = list(range(r))
            q = list(range(r))
            for i in range(r - 1, 0, -1):
                a = H(seed, 4, i) % (i + 1)
                p[i], p[a] = p[a], p[i]
                b = H(seed, 5, i) % (i + 1)
                q[i], q[b] = q[b], q[i]

            def fits(perm, s):
                return int(np.prod([dims[perm[i]] for i in range(s)])) <= 4

            ns = H(seed, 6) % (r + 1)
            while not fits(p, ns):
                ns -= 1
            tp = ops.permute(t, p, ns)
            pinv = [0] * r
            for i in range(r):
                pinv[p[i]] = i
            back = ops.permute(tp, pinv, shape.split)
            if back.in_span():
                assert np.array_equal(back.to_global_vector(), g), "round trip restores elements"
            qs = shape.split
            while not fits(q, qs):
                qs -= 1
            comp = [q[p[i]] for i in range(r)]
            cs = ns
            while not fits(comp, cs):
                cs -= 1
            tqp = ops.permute(ops.permute(t, q, qs), p, cs)
            tc = ops.permute(t, comp, cs)
            a = tqp.to_global_vector()
            b = tc.to_global_vector()
            if tc.in_span():
                assert np.array_equal(a, b), "composition of permutations"

        World(4).run(body)


def test_rebcast_changes_the_pattern_and_keeps_values(peer_mode):
    # test_ops.cpp:161-192
    g = iota_global(4)
    meta, z = golden("rebcast")

    def body(rk):
        t = Tensor.from_global(rk, IndexTuple([2, 2], 1), DistParams(1, 1, 0), g)
        s = ops.rebcast(t, DistParams(2, 1, 0))
        assert s.span() == 4
        assert np.array_equal(s.to_global_vector(), g)
        assert s.my_block() == rk.rank() // 2
        c = ops.rebcast(t, DistParams(1, 2, 0))
        assert c.span() == 4
        assert np.array_equal(c.to_global_vector(), g)
        assert c.my_block() == rk.rank() % 2
        n = ops.rebcast(t, t.dist())
        nv = n.to_global_vector()
        if n.in_span():
            assert np.array_equal(nv, g)
        o = ops.rebcast(t, DistParams(1, 1, 2))
        assert o.dist().offset == 2
        ov = o.to_global_vector()
        if o.in_span():
            assert np.array_equal(ov, z["out3"])
        # every copy holds its block
        if s.in_span():
            assert np.array_equal(s.local_data(), g[2 * s.my_block(): 2 * s.my_block() + 2])

    World(4).run(body)


def test_scatter_and_gather_indices(peer_mode):
    # test_ops.cpp:218-248
    g = iota_global(4)

    def body(rk):
        t = Tensor.from_global(rk, IndexTuple([2, 2], 0), None, g)
        s = ops.scatter_index(t, 0)
        assert s.shape().str() == "(2;2)"
        assert np.array_equal(s.to_global_vector(), g)
        gg = ops.gather_index(s, 0)
        assert gg.shape().str() == "(;2,2)"
        v = gg.to_global_vector()
        if gg.in_span():
            assert np.array_equal(v, g)
        with pytest.raises(InvalidArgument):
            ops.scatter_index(t, 2)
        with pytest.raises(InvalidArgument):
            ops.gather_index(t, 0)

    World(2).run(body)


def test_value_preservation_across_structural_ops():
    # test_ops.cpp:250-288
    for seed in range(20, 26):
        def body(rk, seed=seed):
            dims = random_dims(seed, 6)
            shape = IndexTuple(dims, 0)
            g = iota_global(shape.total_size())
            t = Tensor.from_global(rk, shape, DistParams(1, 1, 0), g)
            want = np.sort_complex(g)
            cur = t
            i = cur.shape().split
            while i < cur.shape().n_idx():
                sh = cur.shape()
                if sh.dist_size() * sh.dims[i] <= 6:
                    cur = ops.scatter_index(cur, i)
                    v = cur.to_global_vector()
                    if cur.in_span():
                        assert np.array_equal(np.sort_complex(v), want)
                i += 1
            while cur.shape().split > 0:
                cur = ops.gather_index(cur, 0)
                v = cur.to_global_vector()
                if cur.in_span():
                    assert np.array_equal(np.sort_complex(v), want)
            if shape.n_idx() > 0 and dims[0] <= 6:
                rt = ops.gather_index(ops.scatter_index(t, 0), 0)
                assert rt.shape().dims == dims
                v = rt.to_global_vector()
                if rt.in_span():
                    assert np.array_equal(v, g)

        World(6).run(body)


def test_local_slice_pad_helpers():
    # test_ops.cpp:290-312 (slice / pad)
    g = iota_global(8)

    def body(rk):
        t = Tensor.from_global(rk, IndexTuple([2, 4], 0), None, g)
        s = ops.slice_local_dims(t, [2, 2])
        assert np.array_equal(s.to_global_vector(), g[[0, 1, 4, 5]])
        p = ops.pad_local_dims(s, [2, 4])
        v = p.to_global_vector()
        assert v[0] == g[0] and v[5] == g[5] and v[2] == 0

    World(1).run(body)


def test_conj_and_scale():
    g = iota_global(12)

    def body(rk):
        t = Tensor.from_global(rk, IndexTuple([3, 4], 1), DistParams(1, 1, 0), g)
        c = ops.conj(t).to_global_vector()
        s = ops.scale(t, 2 - 1j).to_global_vector()
        return c, s

    c, s = World(3).run(body)[0]
    assert np.array_equal(c, np.conj(g))
    assert np.allclose(s, g * (2 - 1j), rtol=0, atol=1e-15)


@pytest.mark.parametrize("n,seed", [(20, 1), (24, 2), (26, 3)])
def test_large_random_qubit_permutation_bit_exact(n, seed):
    g = circuits.counter_state(seed, 2**n)
    perm = circuits.fisher_yates(seed, 9, n)

    def body(rk):
        t = Tensor.from_global(rk, IndexTuple([2] * n, 0), None, g)
        return ops.permute(t, perm, 0).local_data()

    got = run_collect(World(1), body)
    want = np.ascontiguousarray(g.reshape([2] * n).transpose(perm).reshape(-1))
    assert np.array_equal(bits(got), bits(want))


@pytest.mark.parametrize("dims,perm", [([1000, 37], [1, 0]), ([3, 5, 7, 11], [3, 1, 0, 2]),
                                       ([1024, 2048], [1, 0]), ([64, 3, 2, 128], [3, 2, 0, 1]),
                                       ([4099, 2, 3], [2, 0, 1]), ([2] * 16 + [7], [16] + list(range(16)))])
def test_general_dims_permutation(dims, perm):
    n = int(np.prod(dims))
    g = circuits.counter_state(77, n)
    g[::5] = -0.0  # both parts -0 -> must come out +0

    def body(rk):
        t = Tensor.from_global(rk, IndexTuple(dims, 0), None, g)
        return ops.permute(t, perm, 0).local_data()

    got = run_collect(World(1), body)
    assert np.array_equal(bits(got), bits(P.permute(dims, g, perm)))


@pytest.mark.parametrize("world,split,new_split", [(8, 3, 3), (8, 3, 2), (4, 2, 3), (8, 3, 0)])
def test_distributed_swaps_bit_exact(world, split, new_split, peer_mode):
    n = 18
    g = circuits.counter_state(5, 2**n)
    perm = circuits.fisher_yates(5 + world + new_split, 10, n)

    def body(rk):
        t = Tensor.from_global(rk, IndexTuple([2] * n, split), DistParams(1, 1, 0), g)
        p = ops.permute(t, perm, new_split)
        return p.to_global_vector() if True else None

    if 2 ** new_split > world:
        with pytest.raises(ResourceError):
            World(world).run(body)
        return
    got = World(world).run(body)[0]
    assert np.array_equal(bits(got), bits(P.permute([2] * n, g, perm)))


def test_rank_failure_aborts_the_world():
    # runtime.hpp:276-298: a throwing rank aborts the others, the originating error wins
    def body(rk):
        t = Tensor.from_global(rk, IndexTuple([4, 2], 1), DistParams(1, 1, 0), iota_global(8))
        if rk.rank() == 1:
            raise ValueError("boom")
        ops.permute(t, [1, 0], 1)  # rank 0 blocks in the exchange until aborted

    with pytest.raises(ValueError):
        World(4).run(body)


@pytest.mark.parametrize("dims,split,dist,amap,dsplit,ddist,world,ddims", [
    ([2, 3, 4, 2], 1, (1, 1, 0), [2, 0, 3, 1], 2, (1, 1, 0), 8, None),     # permute + new split in one pass
    ([2, 2, 4, 2], 1, (1, 2, 0), [0, 1, 2, 3], 1, (2, 1, 1), 6, None),     # rebcast (stretch, offset)
    ([2, 3, 2, 2], 2, (1, 1, 0), [3, 2, 1, 0], 1, (1, 1, 2), 8, None),     # both at once
    ([2, 3, 4], 1, (1, 1, 0), [0, 2, 1], 1, (1, 1, 0), 2, [2, 5, 3]),       # zero-embedding of local dims
])
def test_tensor_to_tensor_remap(dims, split, dist, amap, dsplit, ddist, world, ddims, peer_mode):
    """remap::tensor_to_tensor (remap.hpp:106-161): axis map, new split and new
    DistParams in one redistribution; larger local destination dims zero-embed."""
    from paper_2505_06119_b200.qtnh import ops
    n = len(dims)
    g = circuits.counter_state(9, int(np.prod(dims)))
    g[::4] = complex(-0.0, -0.0)
    nd = [0] * n
    for i, q in enumerate(amap):
        nd[q] = dims[i]
    out_dims = ddims or nd

    def body(rk):
        t = Tensor.from_global(rk, IndexTuple(dims, split), DistParams(*dist), g)
        u = ops.remap(t, amap, IndexTuple(out_dims, dsplit), DistParams(*ddist))
        assert u.shape().dims == out_dims and u.shape().split == dsplit
        d = u.dist()
        assert (d.stretch, d.cycles, d.offset) == tuple(ddist)
        return u.to_global_vector() if u.in_span() else None

    outs = [o for o in World(world).run(body) if o is not None]
    perm = [amap.index(p) for p in range(n)]  # new position p holds old index perm[p]
    want = P.permute(dims, g, perm).reshape(nd)
    if ddims:
        pad = np.zeros(ddims, complex)
        pad[tuple(slice(0, x) for x in nd)] = want
        want = pad
    for o in outs:
        assert np.array_equal(bits(o), bits(want.reshape(-1)))


def _paired_dense(dims, pairs_in, pairs_out, crossed):
    eq_out = list(pairs_out)
    if crossed:
        eq_out[0], eq_out[1] = eq_out[1], eq_out[0]
    idx = np.indices(dims).reshape(len(dims), -1)
    ok = np.ones(idx.shape[1], bool)
    for a, b in zip(pairs_in, eq_out):
        ok &= idx[a] == idx[b]
    return ok.astype(np.complex128)


@pytest.mark.parametrize("dims,split,pin,pout,crossed,world", [
    ([2, 3, 2, 3], 0, [0, 1], [2, 3], False, 1),
    ([3, 2, 3, 2], 1, [0, 3], [2, 1], False, 3),       # pairs of different index types (scatter/gather form)
    ([2, 2, 2, 2], 2, [0, 1], [2, 3], True, 4),         # swap tensor, distributed
    ([4, 3, 3, 4], 0, [0, 1], [2, 3], True, 1),         # crossed: in0 pairs with out1
])
def test_identity_and_swap_tensors(dims, split, pin, pout, crossed, world):
    """Tensor::identity / swap_tensor (tensor.hpp:144-164) materialised on the device."""
    def body(rk):
        mk = Tensor.swap_tensor if crossed else Tensor.identity
        t = mk(rk, IndexTuple(dims, split), DistParams(1, 1, 0), pin, pout)
        return t.to_global_vector() if t.in_span() else None

    outs = [o for o in World(world).run(body) if o is not None]
    want = _paired_dense(dims, pin, pout, crossed)
    for o in outs:
        assert np.array_equal(o, want)


def test_contracting_a_swap_tensor_is_a_permutation():
    """SPEC: contraction with a swap tensor = index exchange (tensor.hpp:157-164)."""
    from paper_2505_06119_b200.qtnh import contract
    n = 6
    g = circuits.counter_state(4, 2**n)

    def body(rk):
        st = Tensor.from_global(rk, IndexTuple([2] * n, 0), None, g)
        sw = Tensor.swap_tensor(rk, IndexTuple([2, 2, 2, 2], 0), None, [0, 1], [2, 3])
        c = contract(st, sw, [1, 4], [0, 1])  # result: open(state) then the swap outputs
        return c.to_global_vector()

    got = run_collect(World(1), body)
    # result order: state qubits 0,2,3,5 then outputs (2 = in1 -> q4, 3 = in0 -> q1)
    want = g.reshape([2] * n).transpose([0, 2, 3, 5, 4, 1]).reshape(-1)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("dims,split,world", [([2, 3, 2, 3], 0, 1), ([2, 2, 3, 3], 2, 4), ([3, 3, 2, 4, 2, 4], 2, 9)])
def test_diagonal_tensor(dims, split, world):
    """Tensor::diagonal (tensor.hpp:114-142) on the symmetric half-split layout."""
    r = len(dims)
    kd, kl = split // 2, (r - split) // 2
    in_pos = list(range(kd)) + list(range(split, split + kl))
    n_in = int(np.prod([dims[p] for p in in_pos]))
    diag = circuits.rng_normals(12, n_in)
    idx = np.indices(dims).reshape(r, -1)
    on = np.ones(idx.shape[1], bool)
    for i in range(kd):
        on &= idx[i] == idx[kd + i]
    for i in range(kl):
        on &= idx[split + i] == idx[split + kl + i]
    flat_in = np.zeros(idx.shape[1], np.int64)
    for p in in_pos:
        flat_in = flat_in * dims[p] + idx[p]
    want = np.where(on, diag[np.minimum(flat_in, n_in - 1)], 0)

    def body(rk):
        t = Tensor.diagonal(rk, IndexTuple(dims, split), DistParams(1, 1, 0), diag)
        return t.to_global_vector() if t.in_span() else None

    for o in [o for o in World(world).run(body) if o is not None]:
        assert np.array_equal(o, want)


def test_many_plan_shapes_interleaved():
    """Plans of different tile sizes interleaved (the copy kernel's dynamic shared
    memory limit is per kernel: a small-tile plan must not shrink it under a
    large-tile one)."""
    rng = np.random.default_rng(3)
    cases = []
    for _ in range(14):
        r = int(rng.integers(3, 8))
        dims = [int(x) for x in rng.choice([2, 3, 4, 5, 6, 8, 16, 64], size=r)]
        while int(np.prod(dims)) > 2**21:
            dims[int(np.argmax(dims))] //= 2
        cases.append((dims, [int(x) for x in rng.permutation(r)]))
    cases = cases + cases[::-1]

    def body(rk):
        outs = []
        for dims, perm in cases:
            g = circuits.counter_state(len(dims), int(np.prod(dims)))
            t = Tensor.from_global(rk, IndexTuple(dims, 0), None, g)
            outs.append(ops.permute(t, perm, 0).to_global_vector())
        return outs

    outs = run_collect(World(1), body)
    for (dims, perm), got in zip(cases, outs):
        g = circuits.counter_state(len(dims), int(np.prod(dims)))
        assert np.array_equal(bits(got), bits(P.permute(dims, g, perm)))


@pytest.mark.parametrize("world,split", [(4, 2), (8, 3)])
def test_peer_kernels_write_only_their_blocks(world, split, peer_mode):
    """Canary check of the multi-rank kernels (push remap, pairwise in-place swaps,
    the pipelined exchange form, fused distributed gates and QFT): every rank
    interleaves sentinel tensors with its working tensors in the stream-ordered
    pool, runs the ops, and the sentinels must come back bit-identical while the
    results stay bit-exact / within tolerance (compute-sanitizer is not available
    on this pool; a stray store lands in a neighbouring allocation)."""
    from paper_2505_06119_b200.qtnh import apply_gate, qft, swap_indices

    n = 16
    g = circuits.counter_state(77, 2**n)
    pattern = circuits.counter_state(78, 2 ** (n - split))
    perm = circuits.fisher_yates(79, 10, n)

    def body(rk):
        sentinels = []
        for _ in range(3):
            sentinels.append(Tensor.dense(rk, IndexTuple([2] * (n - split), 0), DistParams(1, 1, rk.rank()),
                                          pattern))
        t = Tensor.from_global(rk, IndexTuple([2] * n, split), DistParams(1, 1, 0), g)
        sentinels.append(Tensor.dense(rk, IndexTuple([2] * (n - split), 0), DistParams(1, 1, rk.rank()), pattern))
        p = ops.permute(t, perm, split)
        swap_indices(t, 0, n - 1)
        apply_gate(t, [1], circuits.H)
        apply_gate(t, [0, n - 2], circuits.FSIM)
        u = Tensor.from_global(rk, IndexTuple([2] * n, split), DistParams(1, 1, 0), g)
        qft(u, swaps=True)
        out = (p.to_global_vector(), t.to_global_vector(), u.to_global_vector())
        for s in sentinels:
            assert np.array_equal(bits(s.local_data()), bits(pattern)), "a sentinel allocation was overwritten"
        return out

    pv, tv, uv = World(world).run(body)[0]
    assert np.array_equal(bits(pv), bits(P.permute([2] * n, g, perm)))
    sw = list(range(n))
    sw[0], sw[n - 1] = n - 1, 0
    want = P.permute([2] * n, g, sw)
    want = P.gate([2] * n, want, [1], circuits.H)
    want = P.gate([2] * n, want, [0, n - 2], circuits.FSIM)
    assert np.linalg.norm(tv - want) <= 1e-12 * np.linalg.norm(want)
    wq = P.qft(n, g)
    assert np.linalg.norm(uv - wq) <= 1e-12 * np.linalg.norm(wq)
