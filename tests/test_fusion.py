"""Gate fusion: the fused block sequence must act like the
gate sequence -- checked on the CPU with a dense numpy statevector, and on the GPU
through the dense / diagonal gate kernels against the oracle's gate-by-gate run."""
import numpy as np
import pytest

from conftest import rel_l2
from paper_2505_06119_b200 import circuits, network
from paper_2505_06119_b200.mps import SINGLE_QUBIT


def dense_apply(sv, n, targets, gate):
    k = len(targets)
    t = sv.reshape([2] * n)
    g = np.asarray(gate).reshape([2] * (2 * k))
    t = np.tensordot(g, t, axes=(list(range(k, 2 * k)), targets))
    rest = [q for q in range(n) if q not in targets]
    return np.transpose(t, np.argsort(list(targets) + rest)).reshape(-1)


def rcs_gates(rows, cols, depth, seed):
    return [(list(qs), SINGLE_QUBIT[g] if kind == "1q" else circuits.FSIM)
            for kind, qs, g in network.rcs_grid_circuit(rows, cols, depth, seed)]


def qft_gate_list(n):
    out = []
    for kind, q, g in circuits.qft_gates(n, swaps=True):
        out.append((list(q), np.diag(g) if kind == "cp" else (circuits.SWAP if kind == "swap" else g)))
    return out


@pytest.mark.parametrize("kmax", [2, 3, 4])
@pytest.mark.parametrize("which", ["random", "rcs", "qft"])
def test_fusion_equivalence_cpu(kmax, which):
    rng = np.random.default_rng(kmax)
    n = 9
    if which == "random":
        gates = []
        for _ in range(80):
            k = int(rng.integers(1, 3))
            qs = [int(x) for x in rng.choice(n, size=k, replace=False)]
            gates.append((qs, rng.standard_normal((2**k, 2**k)) + 1j * rng.standard_normal((2**k, 2**k))))
    elif which == "rcs":
        gates = rcs_gates(3, 3, 6, 5)
    else:
        gates = qft_gate_list(n)
    sv = rng.standard_normal(2**n) + 1j * rng.standard_normal(2**n)
    a = sv.copy()
    for qs, g in gates:
        a = dense_apply(a, n, qs, g)
    fused = circuits.fuse_gates(gates, kmax)
    assert all(len(f.qubits) <= kmax for f in fused)
    assert sum(f.count for f in fused) == len(gates)
    assert len(fused) < len(gates)
    b = sv.copy()
    for f in fused:
        b = dense_apply(b, n, f.qubits, f.matrix)
    assert rel_l2(b, a) < 1e-13


@pytest.mark.gpu
@pytest.mark.parametrize("which", ["rcs", "qft"])
def test_fused_circuit_on_gpu_vs_oracle(which):
    import oracle
    from paper_2505_06119_b200.qtnh import IndexTuple, Tensor, World, run_collect

    P = oracle.port()
    n = 12
    gates = rcs_gates(3, 4, 8, 9) if which == "rcs" else qft_gate_list(n)
    st = circuits.counter_state(13, 2**n)
    want = st.copy()
    for qs, g in gates:
        want = P.gate([2] * n, want, qs, np.asarray(g).reshape(-1))
    fused = circuits.fuse_gates(gates, 4)

    def body(rk):
        t = Tensor.from_global(rk, IndexTuple([2] * n, 0), None, st)
        circuits.apply_fused(t, fused)
        out = t.to_global_vector()
        t.free()
        return out

    assert rel_l2(run_collect(World(1), body), want) < 1e-12
