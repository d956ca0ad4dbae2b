"""GPU parity of pairwise contraction (complex128 DMMA GEMM + fused layout) against
the reference's t2m -> pgemm -> m2t path, within the north-star tolerance of
relative L2 <= 1e-10 (BASELINE.json north_star)."""
import ctypes as C

import numpy as np
import pytest

import oracle
from conftest import golden, rel_l2
from paper_2505_06119_b200 import circuits, qtnh
from paper_2505_06119_b200.qtnh import DistParams, IndexTuple, Tensor, World, contract, run_collect

pytestmark = pytest.mark.gpu
TOL = 1e-10
P = oracle.port()


def test_contract_golden():
    meta, z = golden("contract")
    for i, m in enumerate(meta):
        a, b = z[f"a{i}"], z[f"b{i}"]

        def body(rk):
            ta = Tensor.from_global(rk, IndexTuple(m["da"], m["sa"]), DistParams(1, 1, 0), a)
            tb = Tensor.from_global(rk, IndexTuple(m["db"], m["sb"]), DistParams(1, 1, 0), b)
            c = contract(ta, tb, m["apos"], m["bpos"])
            return c.shape(), c.to_global_vector()

        shape, got = World(m["world"]).run(body)[0]
        assert shape.dims == m["out_dims"] and shape.split == m["out_split"], m
        assert rel_l2(got, z[f"out{i}"]) < TOL, m


def test_matrix_vector_known_answer():
    # A = [[0,1],[1,0]] bonded to v = [1,0] -> [0,1]
    def body(rk):
        a = Tensor.from_global(rk, IndexTuple([2, 2], 0), None, np.array([0, 1, 1, 0], complex))
        v = Tensor.from_global(rk, IndexTuple([2], 0), None, np.array([1, 0], complex))
        return contract(a, v, [1], [0]).to_global_vector()

    assert np.array_equal(run_collect(World(1), body), np.array([0, 1], complex))


@pytest.mark.parametrize("da,db,ap,bp", [
    ([3, 2, 5, 2], [5, 3, 4], [0, 2], [1, 0]),
    ([7, 9, 4], [4, 9], [1, 2], [1, 0]),
    ([2, 3], [4, 5], [], []),                       # outer product
    ([6, 5], [5, 6], [0, 1], [1, 0]),               # full contraction -> scalar
    ([130, 70], [70, 257], [1], [0]),               # GEMM tails in M, N, K
    ([33, 65, 3], [3, 65, 1], [1, 2], [1, 0]),
])
def test_general_contractions(da, db, ap, bp):
    a = circuits.rng_normals(1, int(np.prod(da)))
    b = circuits.rng_normals(2, int(np.prod(db)))

    def body(rk):
        ta = Tensor.from_global(rk, IndexTuple(da, 0), None, a)
        tb = Tensor.from_global(rk, IndexTuple(db, 0), None, b)
        return contract(ta, tb, ap, bp).to_global_vector()

    assert rel_l2(run_collect(World(1), body), P.contract(da, a, db, b, ap, bp)) < TOL


@pytest.mark.parametrize("rank_a,world,split", [(20, 1, 0), (22, 1, 0), (20, 4, 2), (20, 8, 3), (18, 2, 1)])
def test_c1_shaped_random_contraction_vs_reference(rank_a, world, split):
    """Config 1 shape (A rank-r, B rank-14, 7 shared indices at seeded random
    positions) against the unmodified reference on the same seeded inputs."""
    if not oracle.ref_available():
        pytest.skip("reference build absent")
    R = oracle.ref()
    seed = 11
    a = circuits.rng_normals(seed, 2**rank_a)
    b = circuits.rng_normals(seed + 1, 2**14)
    ap, bp = circuits.contraction_positions(seed, rank_a, 14, 7)
    want, wd, ws = R.contract(world, [2] * rank_a, split, (1, 1, 0), a, [2] * 14, 0, (1, 1, 0), b, ap, bp)

    def body(rk):
        ta = Tensor.from_global(rk, IndexTuple([2] * rank_a, split), DistParams(1, 1, 0), a)
        tb = Tensor.from_global(rk, IndexTuple([2] * 14, 0), DistParams(1, 1, 0), b)
        c = contract(ta, tb, ap, bp)
        return c.shape(), c.to_global_vector()

    shape, got = World(world).run(body)[0]
    assert shape.dims == wd and shape.split == ws
    assert rel_l2(got, want) < TOL


def test_contracted_distributed_index_is_swapped_local():
    """A contracted index in a distributed position (one
    dist<->local swap precedes the GEMM)."""
    da, db = [2] * 12, [2] * 6
    a = circuits.rng_normals(5, 2**12)
    b = circuits.rng_normals(6, 2**6)
    ap, bp = [0, 5, 9], [2, 0, 4]

    def body(rk):
        ta = Tensor.from_global(rk, IndexTuple(da, 2), DistParams(1, 1, 0), a)
        tb = Tensor.from_global(rk, IndexTuple(db, 1), DistParams(1, 1, 2), b)  # b sharded elsewhere
        c = contract(ta, tb, ap, bp)
        return c.shape(), c.to_global_vector()

    shape, got = World(4).run(body)[0]
    assert shape.split == 1  # a's open distributed index (position 1) stays distributed
    assert rel_l2(got, P.contract(da, a, db, b, ap, bp)) < TOL


@pytest.mark.parametrize("da,db,ap,bp", [
    ([2] * 20, [2] * 12, [0, 2, 3, 5, 7, 8, 11, 13, 16, 19], list(range(10))),   # K = 1024: split column table
    ([2] * 19, [2] * 13, [1, 4, 5, 6, 9, 10, 12, 14, 15, 17, 18], [12, 0, 1, 2, 3, 4, 5, 6, 7, 8, 9]),  # K = 2048
    ([3] * 9, [3] * 7, [0, 2, 4, 5, 7, 8], [5, 4, 3, 2, 1, 0]),                  # K = 729: global table
])
def test_long_k_gather_contractions(da, db, ap, bp):
    a = circuits.rng_normals(31, int(np.prod(da)))
    b = circuits.rng_normals(32, int(np.prod(db)))

    def body(rk):
        ta = Tensor.from_global(rk, IndexTuple(da, 0), None, a)
        tb = Tensor.from_global(rk, IndexTuple(db, 0), None, b)
        return contract(ta, tb, ap, bp).to_global_vector()

    assert rel_l2(run_collect(World(1), body), P.contract(da, a, db, b, ap, bp)) < TOL


@pytest.mark.parametrize("m,n,k", [(1, 1, 1), (64, 128, 8), (2**14, 128, 128), (1000, 100, 37), (3, 300, 500),
                                   (4096, 16, 64), (4096, 32, 32), (4100, 16, 64),
                                   (2048, 2048, 64)])
def test_zgemm_device_against_numpy(m, n, k):
    import torch

    rng = np.random.default_rng(m + n + k)
    a = rng.standard_normal((m, k)) + 1j * rng.standard_normal((m, k))
    b = rng.standard_normal((k, n)) + 1j * rng.standard_normal((k, n))
    ta = torch.from_numpy(a).cuda()
    tb = torch.from_numpy(b).cuda()
    tc = torch.empty((m, n), dtype=torch.complex128, device="cuda")
    w = World(1)

    def body(rk):
        rk.set_stream(torch.cuda.current_stream().cuda_stream)
        qtnh.check(qtnh.lib.qtnh_zgemm_device(rk._h, m, n, k, C.c_void_p(ta.data_ptr()),
                                              C.c_void_p(tb.data_ptr()), C.c_void_p(tc.data_ptr())))
        torch.cuda.synchronize()

    w.run(body)
    assert rel_l2(tc.cpu().numpy(), a @ b) < 1e-13


@pytest.mark.parametrize("da,db,ap,bp", [
    ([2] * 16, [2] * 6, [1, 4, 9], [0, 2, 5]),        # leading contracted position inside the chunk runs
    ([2] * 14, [2] * 6, [3, 13], [1, 0]),             # chunks over the first open positions
    ([3, 5, 4, 6], [6, 4, 7], [2, 3], [1, 0]),
    ([4, 3], [3, 2], [1], [0]),
])
def test_contract_host_pipeline(da, db, ap, bp):
    a = circuits.rng_normals(8, int(np.prod(da))).reshape(da)
    b = circuits.rng_normals(9, int(np.prod(db))).reshape(db)

    def body(rk):
        return qtnh.contract_host(rk, a, b, ap, bp)

    got = run_collect(World(1), body)
    want = P.contract(da, a.reshape(-1), db, b.reshape(-1), ap, bp)
    assert rel_l2(got.reshape(-1), want) < TOL


@pytest.mark.slow
def test_c1_full_size_rank28_vs_reference():
    """The bench's own contraction at its full size (BASELINE.json configs[1]: A
    rank-28 = 4 GiB, B rank-14, 7 shared seeded positions, seed 2025) on the GPU,
    against the UNMODIFIED reference's t2m -> pgemm -> m2t over the same 2^28
    elements (~44 GB of host RSS; OpenBLAS on every host core), and against the
    definition-level brute force of 4096 result elements (oracle port)."""
    import os

    import bench

    if not oracle.ref_available():
        pytest.skip("reference build absent")
    ra, rb, k, seed = bench.RANK_A, bench.RANK_B, bench.K_SHARED, bench.SEED
    a = circuits.counter_state(seed, 2**ra)
    b = circuits.counter_state(seed + 1, 2**rb)
    ap, bp = circuits.contraction_positions(seed, ra, rb, k)
    assert (ap, bp) == bench.c1_positions(P.hash_counter)

    def body(rk):
        ta = Tensor.dense(rk, IndexTuple([2] * ra, 0), None, a)
        tb = Tensor.dense(rk, IndexTuple([2] * rb, 0), None, b)
        c = contract(ta, tb, ap, bp)
        out = c.local_data().copy()
        for t in (ta, tb, c):
            t.free()
        return out

    got = run_collect(World(1), body)
    rng = np.random.default_rng(7)
    outs = np.concatenate([[0, 2**ra - 1], rng.integers(0, 2**ra, size=4094)])
    assert rel_l2(got[outs], bench.c1_brute_force(P, outs)) < TOL
    R = oracle.ref()
    R.set_threads(os.cpu_count() or 1)
    want, wd, ws = R.contract(1, [2] * ra, 0, (1, 1, 0), a, [2] * rb, 0, (1, 1, 0), b, ap, bp)
    del a
    assert wd == [2] * ra and ws == 0
    assert rel_l2(got, want) < TOL


@pytest.mark.parametrize("scale", [1e3, 1e8])
def test_gauss_3m_ill_scaled_operands(scale):
    """The GEMM forms the complex product with Gauss's three real products
    (Im = P3 - P1 - P2). With |Re| >> |Im| the imaginary part is a difference of
    O(|Re|^2) terms: its own relative error grows like eps * |Re| / |Im|, while the
    north-star metric (relative L2 of the complex result) stays at rounding level.
    Both are pinned here against a numpy complex128 product, contraction-shaped
    (gathered A) and dense."""
    rng = np.random.default_rng(int(scale))
    da, db, ap, bp = [2] * 16, [2] * 12, [1, 4, 7, 9, 12, 14], [0, 2, 3, 5, 8, 11]
    a = rng.standard_normal(2**16) * scale + 1j * rng.standard_normal(2**16)
    b = rng.standard_normal(2**12) * scale + 1j * rng.standard_normal(2**12)

    def body(rk):
        ta = Tensor.from_global(rk, IndexTuple(da, 0), None, a)
        tb = Tensor.from_global(rk, IndexTuple(db, 0), None, b)
        return contract(ta, tb, ap, bp).to_global_vector()

    got = run_collect(World(1), body)
    want = P.contract(da, a, db, b, ap, bp)
    assert rel_l2(got, want) < 1e-14
    # per component: Re at rounding level, Im within eps * scale (the documented 3M bound)
    assert rel_l2(got.real, want.real) < 1e-14
    assert rel_l2(got.imag, want.imag) < 1e-14 * scale


@pytest.mark.parametrize("da,db,ap,bp", [
    ([2] * 18, [2] * 10, [0, 3, 5, 8, 11, 14], [9, 0, 2, 4, 6, 7]),     # N = 16, K = 64, A's innermost index open
    ([2] * 18, [2] * 10, [1, 4, 6, 9, 12, 17], [0, 1, 2, 3, 4, 5]),     # N = 16, innermost index contracted
    ([2] * 18, [2] * 10, [0, 2, 7, 13, 17], [3, 8, 1, 0, 6]),           # N = 32, K = 32
    ([2] * 17, [2] * 7, [2, 5, 9, 16], [0, 1, 2, 3]),                   # N = 8: the general narrow kernel
])
def test_narrow_n_gather_contractions(da, db, ap, bp):
    """Narrow result matrices (N = 8, 16, 32 columns: config 3's large steps under the
    flop-minimising order) through the 64 x 16 / 64 x 32 tile-aligned Gauss kernels and
    the general narrow kernel."""
    a = circuits.rng_normals(41, int(np.prod(da)))
    b = circuits.rng_normals(42, int(np.prod(db)))

    def body(rk):
        ta = Tensor.from_global(rk, IndexTuple(da, 0), None, a)
        tb = Tensor.from_global(rk, IndexTuple(db, 0), None, b)
        return contract(ta, tb, ap, bp).to_global_vector()

    assert rel_l2(run_collect(World(1), body), P.contract(da, a, db, b, ap, bp)) < TOL
