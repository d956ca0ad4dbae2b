"""Seeded random small cases against the oracle port: contractions with arbitrary
ranks, dimensions (1 included) and contracted positions; permutations of sharded
tensors with a changed split. Complements the fixed cases of test_contract_gpu.py
and test_structural_gpu.py (the reference's own tests draw random permutations the
same way, test_ops.cpp:112-159)."""
import numpy as np
import pytest

import oracle
from conftest import bits, rel_l2
from paper_2505_06119_b200 import circuits
from paper_2505_06119_b200.qtnh import DistParams, IndexTuple, Tensor, World, contract, ops, run_collect

pytestmark = pytest.mark.gpu
P = oracle.port()


@pytest.mark.parametrize("seed", range(6))
def test_random_contractions_vs_oracle(seed):
    rng = np.random.default_rng(1000 + seed)
    cases = []
    for _ in range(10):
        ra, rb = int(rng.integers(1, 6)), int(rng.integers(1, 6))
        k = int(rng.integers(0, min(ra, rb) + 1))
        da = [int(x) for x in rng.integers(1, 5, size=ra)]
        db = [int(x) for x in rng.integers(1, 5, size=rb)]
        ap = [int(x) for x in rng.permutation(ra)[:k]]
        bp = [int(x) for x in rng.permutation(rb)[:k]]
        for i, j in zip(ap, bp):
            db[j] = da[i]
        cases.append((da, db, ap, bp))

    def body(rk):
        out = []
        for i, (da, db, ap, bp) in enumerate(cases):
            a = circuits.rng_normals(7 * seed + i, int(np.prod(da)))
            b = circuits.rng_normals(9 * seed + i + 100, int(np.prod(db)))
            ta = Tensor.from_global(rk, IndexTuple(da, 0), None, a)
            tb = Tensor.from_global(rk, IndexTuple(db, 0), None, b)
            out.append((a, b, contract(ta, tb, ap, bp).to_global_vector()))
        return out

    for (da, db, ap, bp), (a, b, got) in zip(cases, run_collect(World(1), body)):
        want = P.contract(da, a, db, b, ap, bp)
        assert got.shape == want.shape, (da, db, ap, bp)
        assert rel_l2(got, want) < 1e-12, (da, db, ap, bp)


@pytest.mark.parametrize("seed", range(4))
def test_random_sharded_permutations_bit_exact(seed, peer_mode):
    rng = np.random.default_rng(2000 + seed)
    world = int(rng.choice([2, 4, 8]))
    lw = int(np.log2(world))
    n = int(rng.integers(lw + 1, lw + 6))
    dims = [2] * n
    for i in range(lw, n):  # non-qubit local dimensions too
        dims[i] = int(rng.integers(1, 4))
    split = int(rng.integers(0, lw + 1))
    perm = [int(x) for x in rng.permutation(n)]
    # the new split keeps the world large enough: distributed dims must multiply to <= world
    new_split = 0
    prod = 1
    for pos in range(n):
        if prod * dims[perm[pos]] <= world:
            prod *= dims[perm[pos]]
            new_split = pos + 1
        else:
            break
    new_split = int(rng.integers(0, new_split + 1))
    g = circuits.counter_state(300 + seed, int(np.prod(dims)))
    g[::5] = complex(-0.0, -0.0)

    def body(rk):
        t = Tensor.from_global(rk, IndexTuple(dims, split), DistParams(1, 1, 0), g)
        return ops.permute(t, perm, new_split).to_global_vector()

    got = World(world).run(body)[0]
    assert np.array_equal(bits(got), bits(P.permute(dims, g, perm))), (dims, split, perm, new_split)
