"""GPU parity of gate application and the QFT workloads (configs 0 and 2)."""
import functools

import numpy as np
import pytest

import oracle
from conftest import golden, rel_l2
from paper_2505_06119_b200 import circuits
from paper_2505_06119_b200.qtnh import DistParams, IndexTuple, Tensor, World, apply_gate, ops, run_collect

pytestmark = pytest.mark.gpu
TOL = 1e-10
P = oracle.port()


def test_gate_golden():
    meta, z = golden("gate")
    n = meta["n"]
    for i, g in enumerate(meta["gates"]):
        def body(rk):
            t = Tensor.from_global(rk, IndexTuple([2] * n, 0), None, z["state"])
            apply_gate(t, g["targets"], z[f"g{i}"])
            return t.to_global_vector()

        assert rel_l2(run_collect(World(1), body), z[f"out{i}"]) < 1e-14
    dc = meta["dist_case"]

    def dbody(rk):
        t = Tensor.from_global(rk, IndexTuple([2] * n, dc["split"]), DistParams(1, 1, 0), z["state"])
        apply_gate(t, dc["targets"], z[f"g{dc['gate']}"])
        return t.to_global_vector()

    assert rel_l2(World(dc["world"]).run(dbody)[0], z["out_dist"]) < 1e-14


def test_gate_copy_on_write():
    g = circuits.counter_state(1, 2**6)

    def body(rk):
        t = Tensor.from_global(rk, IndexTuple([2] * 6, 0), None, g)
        alias = ops.permute(t, list(range(6)), 0)  # identity permute shares the value
        apply_gate(alias, [2], circuits.H)
        return t.to_global_vector(), alias.to_global_vector()

    orig, upd = run_collect(World(1), body)
    assert np.array_equal(orig, g)
    assert rel_l2(upd, P.gate([2] * 6, g, [2], circuits.H)) < 1e-14


@pytest.mark.parametrize("dims,targets,D", [([2] * 10, [9], 2), ([2] * 10, [0, 9], 4), ([3, 4, 5, 2], [2, 0], 15),
                                            ([2] * 12, [3, 7, 1], 8), ([2] * 12, [11, 10, 0, 5], 16),
                                            ([5, 6, 7], [1], 6)])
def test_dense_gates_general(dims, targets, D):
    g = circuits.counter_state(3, int(np.prod(dims)))
    gate = circuits.rng_normals(4, D * D)

    def body(rk):
        t = Tensor.from_global(rk, IndexTuple(dims, 0), None, g)
        apply_gate(t, targets, gate)
        return t.to_global_vector()

    assert rel_l2(run_collect(World(1), body), P.gate(dims, g, targets, gate)) < 1e-14


@pytest.mark.parametrize("dims,split,dist,targets,world", [
    ([2] * 12, 1, (1, 1, 0), [0], 2),             # single distributed qubit
    ([2] * 12, 3, (1, 1, 0), [1], 8),
    ([2] * 12, 3, (1, 1, 0), [2, 7], 8),          # one distributed + one local target
    ([2] * 12, 2, (1, 1, 0), [9, 0, 4], 4),       # distributed target in the middle of the list
    ([2] * 12, 2, (1, 1, 0), [0, 1], 4),          # both distributed: swap path
    ([2] * 11, 1, (2, 1, 1), [0, 5], 6),          # stretched copies, offset
    ([2] * 11, 2, (1, 2, 0), [1], 8),             # cyclic copies
    ([3, 2, 4, 2], 2, (1, 1, 0), [1, 2], 6),      # non-qubit local dims
])
def test_dense_gates_on_distributed_targets(dims, split, dist, targets, world, peer_mode):
    """Dense gates with distributed targets: fused peer-memory gate (one
    distributed qubit target) or swap -> apply -> swap back, against the oracle."""
    g = circuits.counter_state(41, int(np.prod(dims)))
    D = int(np.prod([dims[q] for q in targets]))
    gate = circuits.rng_normals(42, D * D)

    def body(rk):
        t = Tensor.from_global(rk, IndexTuple(dims, split), DistParams(*dist), g)
        apply_gate(t, targets, gate)
        return t.to_global_vector()

    outs = [o for o in World(world).run(body) if o.size]
    want = P.gate(dims, g, targets, gate)
    for o in outs:
        assert rel_l2(o, want) < 1e-14


def test_diagonal_gates_on_distributed_targets():
    n = 12
    g = circuits.counter_state(8, 2**n)
    d = circuits.cp_diag(0.7)

    def body(rk):
        t = Tensor.from_global(rk, IndexTuple([2] * n, 3), DistParams(1, 1, 0), g)
        apply_gate(t, [1, 7], d, diagonal=True)  # one distributed, one local target
        apply_gate(t, [0, 2], d, diagonal=True)  # both distributed: scalar per rank
        return t.to_global_vector()

    want = P.gate([2] * n, P.gate([2] * n, g, [1, 7], d, diagonal=True), [0, 2], d, diagonal=True)
    assert rel_l2(World(8).run(body)[0], want) < 1e-14


def test_qft16_config0_vs_reference():
    """Config 0: QFT on 16 qubits from a seeded normalised random state, all gates,
    against the unmodified reference's gate-by-gate contraction path."""
    n = 16
    st = circuits.counter_state(2025, 2**n)
    st /= np.linalg.norm(st)

    def body(rk):
        t = Tensor.from_global(rk, IndexTuple([2] * n, 0), None, st)
        return circuits.apply_qft(t, n, swaps=True).to_global_vector()

    got = run_collect(World(1), body)
    if oracle.ref_available():
        want = oracle.ref().qft(n, st, swaps=True)
    else:
        want = P.qft(n, st, swaps=True)
    assert rel_l2(got, want) < TOL
    assert rel_l2(got, np.fft.ifft(st) * np.sqrt(2**n)) < TOL


@pytest.mark.parametrize("world,split", [(8, 3), (4, 2), (2, 1)])
def test_distributed_qft_vs_oracle(world, split):
    """Config 2 structure at reduced size: the state sharded over `world` ranks by
    its `split` leading qubits; H on a distributed qubit swaps it with a local one."""
    n = 14
    st = circuits.counter_state(7, 2**n)
    st /= np.linalg.norm(st)

    def body(rk):
        t = Tensor.from_global(rk, IndexTuple([2] * n, split), DistParams(1, 1, 0), st)
        return circuits.apply_qft(t, n, swaps=True).to_global_vector()

    got = World(world).run(body)[0]
    assert rel_l2(got, np.fft.ifft(st) * np.sqrt(2**n)) < TOL
    assert rel_l2(got, P.qft(n, st)) < TOL


def test_qft_norm_preserved_large():
    """Size-independent property at 2^26 amplitudes: unitarity (norm preserved) and
    spot amplitudes against a direct O(2^n) DFT sum."""
    n = 26
    st = circuits.counter_state(99, 2**n)
    st /= np.linalg.norm(st)

    def body(rk):
        t = Tensor.from_global(rk, IndexTuple([2] * n, 0), None, st)
        return circuits.apply_qft(t, n, swaps=True).local_data()

    got = run_collect(World(1), body)
    assert abs(np.linalg.norm(got) - 1.0) < 1e-12
    j = np.arange(2**n, dtype=np.float64)
    for k in [0, 1, 12345, 2**n - 1]:
        ph = np.exp(2j * np.pi * ((j * k) % 2**n) / 2**n)
        want = np.dot(ph, st) / np.sqrt(2**n)
        assert abs(got[k] - want) < 1e-10 * max(1.0, abs(want))


def test_fused_qft_matches_reference_qft16():
    """Config 0 through the fused layer path (one pass per QFT layer + in-place swaps)."""
    n = 16
    st = circuits.counter_state(2025, 2**n)
    st /= np.linalg.norm(st)

    def body(rk):
        t = Tensor.from_global(rk, IndexTuple([2] * n, 0), None, st)
        return circuits.apply_qft_fused(t, n).to_global_vector()

    got = run_collect(World(1), body)
    want = oracle.ref().qft(n, st) if oracle.ref_available() else P.qft(n, st)
    assert rel_l2(got, want) < TOL


@pytest.mark.parametrize("world,split", [(8, 3), (2, 1), (4, 2)])
def test_fused_qft_distributed(world, split):
    n = 14
    st = circuits.counter_state(17, 2**n)
    st /= np.linalg.norm(st)

    def body(rk):
        t = Tensor.from_global(rk, IndexTuple([2] * n, split), DistParams(1, 1, 0), st)
        return circuits.apply_qft_fused(t, n).to_global_vector()

    got = World(world).run(body)[0]
    assert rel_l2(got, P.qft(n, st)) < TOL


@pytest.mark.parametrize("dims,split,a,b,world", [([2] * 10, 0, 1, 8, 1), ([3, 4, 3, 2], 0, 0, 2, 1),
                                                  ([2] * 8, 2, 0, 6, 4), ([2] * 8, 2, 3, 7, 4)])
def test_swap_indices_bit_exact(dims, split, a, b, world):
    g = circuits.counter_state(5, int(np.prod(dims)))
    g[::7] = complex(-0.0, -0.0)
    g[1::11] = complex(-0.0, 1.0)
    perm = list(range(len(dims)))
    perm[a], perm[b] = perm[b], perm[a]

    def body(rk):
        t = Tensor.from_global(rk, IndexTuple(dims, split), DistParams(1, 1, 0), g)
        from paper_2505_06119_b200.qtnh import swap_indices
        swap_indices(t, a, b)
        return t.to_global_vector()

    got = World(world).run(body)[0]
    from conftest import bits
    assert np.array_equal(bits(got), bits(P.permute(dims, g, perm)))


@functools.lru_cache(maxsize=None)
def _oracle_qft_of_counter_state(n):
    """The oracle's QFT of test_blocked_qft's seeded state: computed once per n (the
    port takes ~10-20 s at n = 20-21 on the GPU box's host), shared by both
    redistribution forms and every split."""
    st = circuits.counter_state(23 + n, 2**n)
    st /= np.linalg.norm(st)
    return P.qft(n, st)


@pytest.mark.parametrize("n,split,world", [(8, 0, 1), (11, 0, 1), (16, 0, 1), (20, 0, 1), (21, 0, 1), (14, 2, 4), (13, 3, 8),
                                          (6, 3, 8), (7, 3, 8), (8, 3, 8), (9, 1, 2), (20, 3, 8), (19, 2, 4)])
def test_blocked_qft(n, split, world, peer_mode):
    """Cache-blocked whole-QFT kernel path (qtnh_qft) against the oracle QFT."""
    from paper_2505_06119_b200.qtnh import qft
    st = circuits.counter_state(23 + n, 2**n)
    st /= np.linalg.norm(st)

    def body(rk):
        t = Tensor.from_global(rk, IndexTuple([2] * n, split), DistParams(1, 1, 0), st)
        qft(t, swaps=True)
        return t.to_global_vector()

    got = World(world).run(body)[0]
    assert rel_l2(got, _oracle_qft_of_counter_state(n)) < TOL
    if n <= 16:
        def body2(rk):
            t = Tensor.from_global(rk, IndexTuple([2] * n, split), DistParams(1, 1, 0), st)
            qft(t, swaps=False)
            return t.to_global_vector()
        assert rel_l2(World(world).run(body2)[0], P.qft(n, st, swaps=False)) < TOL


@pytest.mark.parametrize("n,split,dist,world", [(12, 2, (2, 1, 0), 8), (12, 2, (1, 2, 0), 8), (11, 1, (1, 1, 3), 6),
                                               (12, 3, (1, 1, 0), 9)])
def test_qft_with_broadcast_copies(n, split, dist, world, peer_mode):
    """Whole QFT on a state with stretched / cyclic copies or an offset: every
    copy ends up with the oracle's result."""
    from paper_2505_06119_b200.qtnh import qft
    st = circuits.counter_state(5 + n, 2**n)
    st /= np.linalg.norm(st)

    def body(rk):
        t = Tensor.from_global(rk, IndexTuple([2] * n, split), DistParams(*dist), st)
        qft(t, swaps=True)
        return t.to_global_vector()

    want = P.qft(n, st)
    outs = [o for o in World(world).run(body) if o.size]
    assert len(outs) == dist[0] * dist[1] * 2**split
    for o in outs:
        assert rel_l2(o, want) < TOL


@pytest.mark.parametrize("dims,split,a,b,world,chunk", [
    ([2] * 12, 2, 0, 9, 4, 1 << 30),      # one chunk
    ([2] * 12, 2, 1, 4, 4, 256),          # many chunks (16 elements each)
    ([3, 3, 2, 3, 2], 1, 0, 3, 3, 96),    # dim-3 indices: two partners per rank
    ([2] * 10, 3, 2, 3, 8, 1 << 30),      # local index right after the split
])
def test_inplace_distributed_swap(dims, split, a, b, world, chunk, peer_mode):
    """Distributed <-> local index swap done in place through a bounded staging
    buffer: bit-exact against ops::permute semantics."""
    from conftest import bits
    from paper_2505_06119_b200.qtnh import check, lib, swap_indices
    g = circuits.counter_state(31, int(np.prod(dims)))
    g[::9] = complex(-0.0, -0.0)
    perm = list(range(len(dims)))
    perm[a], perm[b] = perm[b], perm[a]
    check(lib.qtnh_set_option(b"swap_chunk_bytes", float(chunk)))
    try:
        def body(rk):
            t = Tensor.from_global(rk, IndexTuple(dims, split), DistParams(1, 1, 0), g)
            swap_indices(t, a, b)
            return t.to_global_vector()

        got = World(world).run(body)[0]
    finally:
        check(lib.qtnh_set_option(b"swap_chunk_bytes", float(1 << 31)))
    assert np.array_equal(bits(got), bits(P.permute(dims, g, perm)))


def test_cuda_graph_of_a_gate_sequence():
    """A launch-bound gate sequence (config 0's QFT-16 gate by gate: 16 H, 120 CP,
    8 in-place SWAPs) captured once into a CUDA graph and replayed matches the
    direct sequence, and replays are repeatable."""
    from paper_2505_06119_b200.qtnh import swap_indices
    n = 16
    st = circuits.counter_state(61, 2**n)
    st /= np.linalg.norm(st)
    gates = circuits.qft_gates(n, swaps=True)

    def seq(t):
        for kind, q, g in gates:
            if kind == "h":
                apply_gate(t, q, g)
            elif kind == "cp":
                apply_gate(t, q, g, diagonal=True)
            else:
                swap_indices(t, q[0], q[1])

    def body(rk):
        a = Tensor.from_global(rk, IndexTuple([2] * n, 0), None, st)
        seq(a)
        direct = a.to_global_vector()
        b = Tensor.from_global(rk, IndexTuple([2] * n, 0), None, st)
        rk.synchronize()
        with rk.capture() as g:
            seq(b)
        rk.synchronize()
        untouched = b.to_global_vector()  # capture records, it does not run
        g.launch()
        once = b.to_global_vector()
        g.launch()
        twice = b.to_global_vector()
        g.free()
        return direct, untouched, once, twice

    direct, untouched, once, twice = run_collect(World(1), body)
    assert np.array_equal(untouched, st)
    assert np.array_equal(once, direct)
    assert rel_l2(direct, P.qft(n, st)) < TOL
    seq2 = P.qft(n, P.qft(n, st))
    assert rel_l2(twice, seq2) < 1e-10


@pytest.mark.parametrize("tma", ["0", "1"])
@pytest.mark.parametrize("n", [10, 11, 12, 15, 20, 23])
def test_qft_bit_reversal_pass_bit_exact(n, tma, monkeypatch):
    """The final SWAP network of the whole-QFT path is one in-place bit-reversal
    pass (gate.cu k_bitrev2, or k_bitrev_tma with QTNH_BITREV_TMA=1): QFT with swaps
    must equal QFT without swaps followed by a host bit reversal of the index, bit
    for bit."""
    from paper_2505_06119_b200.qtnh import qft
    monkeypatch.setenv("QTNH_BITREV_TMA", tma)
    st = circuits.counter_state(500 + n, 2**n)

    def body(swaps):
        def f(rk):
            t = Tensor.from_global(rk, IndexTuple([2] * n, 0), None, st)
            qft(t, swaps=swaps)
            return t.to_global_vector()
        return f

    with_swaps = run_collect(World(1), body(True))
    without = run_collect(World(1), body(False))
    idx = np.arange(2**n)
    rev = np.zeros_like(idx)
    for b in range(n):
        rev |= ((idx >> b) & 1) << (n - 1 - b)
    want = without[rev]
    want = np.where(want == 0, 0.0, want)  # signed zeros canonicalised by the pass
    assert np.array_equal(with_swaps.view(np.uint64), np.ascontiguousarray(want).view(np.uint64))
