"""Config 3 structure: a random grid circuit as a tensor network, contracted
pairwise along the seeded greedy order (SPEC contract_order), against (a) the
unmodified reference replaying the same order with its t2m -> pgemm -> m2t
contraction and (b) a statevector run of the same circuit."""
import numpy as np
import pytest

import oracle
from conftest import rel_l2
from paper_2505_06119_b200 import circuits, mps, network
from paper_2505_06119_b200.qtnh import IndexTuple, Tensor, World, apply_gate

pytestmark = pytest.mark.gpu
TOL = 1e-10


def statevector_amplitudes(rows, cols, depth, seed, open_q, fixed, P):
    n = rows * cols
    psi = np.zeros(2**n, complex)
    psi[0] = 1
    for kind, qs, g in network.rcs_grid_circuit(rows, cols, depth, seed):
        if kind == "1q":
            psi = P.gate([2] * n, psi, [qs[0]], mps.SINGLE_QUBIT[g])
        else:
            psi = P.gate([2] * n, psi, list(qs), circuits.FSIM)
    psi = psi.reshape([2] * n)
    idx = tuple(slice(None) if q in open_q else fixed[q] for q in range(n))
    return psi[idx].reshape(-1)


def gpu_tn(rows, cols, depth, seed, n_open):
    def body(rk):
        net, open_labels, open_q, fixed = network.build_rcs_network(rk, rows, cols, depth, seed, n_open)
        data = {i: net.tensors[i].to_global_vector() for i in net.tensors}
        labels = {i: list(l) for i, l in net.labels.items()}
        order = network.Network.plan(net.labels, net.dims, seed)
        last = net.contract_order(order)
        res_labels = net.labels[last]
        out = net.tensors[last].to_global_vector().reshape([2] * len(res_labels))
        perm = [res_labels.index(l) for l in open_labels]
        out = np.transpose(out, perm).reshape(-1)
        net.tensors[last].free()
        return out, open_q, fixed, order, data, labels, dict(net.dims)

    return World(1).run(body)[0]


@pytest.mark.parametrize("rows,cols,depth,n_open", [(3, 3, 6, 3), (2, 4, 8, 2), (3, 4, 5, 4)])
def test_grid_tn_vs_statevector_and_reference(rows, cols, depth, n_open):
    seed = 7
    got, open_q, fixed, order, data, labels, dims = gpu_tn(rows, cols, depth, seed, n_open)
    P = oracle.port()
    want = statevector_amplitudes(rows, cols, depth, seed, open_q, fixed, P)
    assert rel_l2(got, want) < TOL
    if not oracle.ref_available():
        return
    # replay the identical order with the reference's contraction
    R = oracle.ref()
    nxt = max(data) + 1
    for s, (a, b) in enumerate(order):
        la, lb = labels.pop(a), labels.pop(b)
        sh = [x for x in la if x in lb]
        c, cd, _ = R.contract(1, [dims[x] for x in la] or [1], 0, None, data.pop(a) if la else data.pop(a),
                              [dims[x] for x in lb] or [1], 0, None, data.pop(b),
                              [la.index(x) for x in sh], [lb.index(x) for x in sh]) if la and lb else (None, None, None)
        if c is None:  # scalar operand (not produced by these circuits)
            raise AssertionError("unexpected scalar operand")
        labels[nxt + s] = [x for x in la if x not in sh] + [x for x in lb if x not in sh]
        data[nxt + s] = c
    last = nxt + len(order) - 1
    ref = data[last].reshape([2] * len(labels[last]))
    open_labels = [l for l in labels[last]]
    # order the reference result like the GPU result (open qubits ascending)
    want_labels = sorted(open_labels, key=lambda l: int(l[1:].split(".")[0]))
    ref = np.transpose(ref, [open_labels.index(l) for l in want_labels]).reshape(-1)
    assert rel_l2(got, ref) < TOL


@pytest.mark.parametrize("world,shard_flops", [(2, 0.0), (4, 0.0), (8, 0.0)])
def test_sharded_network_contraction(world, shard_flops):
    """replicated small contractions, M-sharded large ones (a
    sharded result stays sharded; two sharded operands replicate the smaller)."""
    rows, cols, depth, n_open, seed = 3, 3, 6, 3, 7

    def body(rk):
        net, open_labels, open_q, fixed = network.build_rcs_network(rk, rows, cols, depth, seed, n_open,
                                                                    shard_flops=shard_flops)
        order = network.Network.plan(net.labels, net.dims, seed)
        last = net.contract_order(order)
        res_labels = net.labels[last]
        v = net.tensors[last].to_global_vector()
        net.tensors[last].free()
        if v.size == 0:
            return None
        out = v.reshape([2] * len(res_labels))
        out = np.transpose(out, [res_labels.index(l) for l in open_labels]).reshape(-1)
        return out, open_q, fixed, net.n_sharded, net.n_replicated

    res = [r for r in World(world).run(body) if r is not None]
    assert res
    assert res[0][3] > 0, [(r[3], r[4]) for r in res]  # some contractions ran sharded
    P = oracle.port()
    _, open_q, fixed, _, _ = res[0]
    want = statevector_amplitudes(rows, cols, depth, seed, open_q, fixed, P)
    for got, *_ in res:
        assert rel_l2(got, want) < TOL


def test_grid_patterns():
    # SPEC.md:652-656 examples
    assert network.grid_pairs("A", 1, 2) == [(0, 1)]
    assert network.grid_pairs("B", 1, 2) == []
    h = sorted(network.grid_pairs("A", 3, 3) + network.grid_pairs("B", 3, 3))
    assert len(h) == 6 and len(set(h)) == 6
    assert all(b - a == 3 for a, b in network.grid_pairs("C", 3, 3))


@pytest.mark.parametrize("rows,cols,depth,n_open", [(3, 3, 6, 3), (3, 4, 5, 4)])
def test_native_chain_executor(rows, cols, depth, n_open):
    """The whole order through one qtnh_contract_chain call equals the statevector."""
    seed = 7

    def body(rk):
        net, open_labels, open_q, fixed = network.build_rcs_network(rk, rows, cols, depth, seed, n_open)
        order = network.Network.plan(net.labels, net.dims, seed)
        last = net.contract_order_native(order)
        res_labels = net.labels[last]
        out = net.tensors[last].to_global_vector().reshape([2] * len(res_labels))
        out = np.transpose(out, [res_labels.index(l) for l in open_labels]).reshape(-1)
        net.tensors[last].free()
        return out, open_q, fixed

    got, open_q, fixed = World(1).run(body)[0]
    want = statevector_amplitudes(rows, cols, depth, seed, open_q, fixed, oracle.port())
    assert rel_l2(got, want) < TOL
