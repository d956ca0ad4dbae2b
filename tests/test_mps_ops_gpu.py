"""GPU: the MPS operations either side of the two-site update (SURVEY.md 8(f) rank 4,
SPEC.md:441-543) -- bitstring / random construction, canonical forms, overlap,
norm2 / renormalise, effective bond dimensions, sampling -- against a dense
statevector oracle (numpy) on small chains."""
import numpy as np
import pytest

from conftest import rel_l2
from paper_2505_06119_b200 import circuits, qtnh
from paper_2505_06119_b200.mps import MPS
from paper_2505_06119_b200.qtnh import World, run_collect

pytestmark = pytest.mark.gpu


def dense_from_sites(sites):
    acc = sites[0]
    for s in sites[1:]:
        acc = np.tensordot(acc, s, axes=([acc.ndim - 1], [0]))
    return acc.reshape(-1)


def site_arrays(m):
    return [t.to_global_vector().reshape(t.shape().dims) for t in m.sites]


def test_bitstring_statevector_norm_and_bonds():
    def body(rk):
        m = MPS.bitstring(rk, [1, 0, 1], chi=4)
        sv = m.to_statevector()
        out = (sv, m.norm2(), m.effective_bond_dims())
        m.free()
        return out

    sv, n2, bonds = run_collect(World(1), body)
    want = np.zeros(8, complex)
    want[0b101] = 1
    assert np.array_equal(sv, want)
    assert n2 == 1.0
    assert bonds == [1, 1]


def test_random_mps_is_normalised_and_deterministic():
    def body(rk):
        a = MPS.random(rk, 6, 4, seed=9)
        b = MPS.random(rk, 6, 4, seed=9)
        out = (a.to_statevector(), b.to_statevector(), a.bond_dims())
        a.free()
        b.free()
        return out

    va, vb, bonds = run_collect(World(1), body)
    assert np.array_equal(va, vb)
    assert abs(np.linalg.norm(va) - 1) < 1e-12
    assert bonds == [2, 4, 4, 4, 2]


@pytest.mark.parametrize("n,chi_eff,centre", [(6, 4, 0), (6, 4, 3), (7, 8, 6), (5, 3, 2)])
def test_canonicalize_keeps_state_and_orthonormalises(n, chi_eff, centre):
    def body(rk):
        m = MPS.random(rk, n, chi_eff, seed=n + centre)
        before = m.to_statevector()
        m.canonicalize(centre)
        after = m.to_statevector()
        sites = site_arrays(m)
        m.free()
        return before, after, sites

    before, after, sites = run_collect(World(1), body)
    assert rel_l2(after, before) < 1e-12
    for q, a in enumerate(sites):
        l, d, r = a.shape
        if q < centre:  # left-orthonormal: sum_{l,s} conj(A) A = I_r
            g = np.einsum("lsr,lsk->rk", a.conj(), a)
            assert np.allclose(g, np.eye(r), atol=1e-10)
        elif q > centre:  # right-orthonormal: sum_{s,r} A conj(A) = I_l
            g = np.einsum("lsr,ksr->lk", a, a.conj())
            assert np.allclose(g, np.eye(l), atol=1e-10)


def test_overlap_matches_dense_inner_product():
    def body(rk):
        a = MPS.random(rk, 6, 4, seed=1)
        b = MPS.random(rk, 6, 3, seed=2)
        out = (a.overlap(b), b.overlap(a), a.overlap(a), a.to_statevector(), b.to_statevector())
        z = MPS.bitstring(rk, [0] * 6, 4)
        o = MPS.bitstring(rk, [1] + [0] * 5, 4)
        out += (z.overlap(o),)
        for m in (a, b, z, o):
            m.free()
        return out

    ab, ba, aa, va, vb, zo = run_collect(World(1), body)
    assert abs(ab - np.vdot(vb, va)) < 1e-12
    assert abs(ba - np.vdot(va, vb)) < 1e-12
    assert abs(aa - 1) < 1e-12
    assert zo == 0


def test_norm2_scaling_and_renormalise():
    def body(rk):
        m = MPS.bitstring(rk, [0, 1, 1, 0], 2)
        m._set(2, qtnh.ops.scale(m.sites[2], 2.0))
        n4 = m.norm2()
        m.renormalise()
        n1 = m.norm2()
        m.free()
        z = MPS.bitstring(rk, [0, 0], 2)
        z._set(0, qtnh.ops.scale(z.sites[0], 0.0))
        try:
            z.renormalise()
            err = None
        except qtnh.DegenerateStateError as e:
            err = e
        z.free()
        return n4, n1, err

    n4, n1, err = run_collect(World(1), body)
    assert n4 == 4.0
    assert abs(n1 - 1) < 1e-12
    assert isinstance(err, qtnh.DegenerateStateError)


def test_truncation_lowers_norm():
    """a two-site update truncated below the Schmidt rank loses weight."""
    def body(rk):
        m = MPS.random(rk, 8, 8, seed=4, chi=8)
        m.canonicalize(3)  # orthonormal environment: the norm loss is the discarded weight
        m.chi = 2
        s, frac = m.apply_2q(3, circuits.FSIM.reshape(4, 4))
        out = (frac, m.norm2())
        m.free()
        return out

    frac, n2 = run_collect(World(1), body)
    assert frac < 1.0 and n2 < 1.0
    assert abs(n2 - frac) < 1e-10


def test_effective_bond_dims_bell_and_random():
    def body(rk):
        bell = MPS.bitstring(rk, [0, 0, 0, 0], 4)
        bell.apply_1q(1, circuits.H)
        cnot = np.eye(4, dtype=complex)[[0, 1, 3, 2]]
        bell.apply_2q(1, cnot)  # (|00> + |11>)/sqrt2 on sites 1, 2
        out = bell.effective_bond_dims()
        bell.free()
        r = MPS.random(rk, 8, 4, seed=5)
        out2 = r.effective_bond_dims()
        r.free()
        return out, out2

    b, r = run_collect(World(1), body)
    assert b == [1, 2, 1]
    assert r == [2, 4, 4, 4, 4, 4, 2]


def test_sampling_distributions():
    def body(rk):
        bits = MPS.bitstring(rk, [1, 0, 1, 1], 2)
        det = [bits.sample([0, 1, 2, 3], seed=3, draw=i) for i in range(5)]
        sub = bits.sample([3, 0], seed=3)
        bits.free()
        bell = MPS.bitstring(rk, [0, 0], 2)
        bell.apply_1q(0, circuits.H)
        bell.apply_2q(0, np.eye(4, dtype=complex)[[0, 1, 3, 2]])
        bd = [tuple(bell.sample([0, 1], seed=7, draw=i)) for i in range(200)]
        bell.free()
        uni = MPS.bitstring(rk, [0, 0], 2)
        uni.apply_1q(0, circuits.H)
        uni.apply_1q(1, circuits.H)
        ud = [tuple(uni.sample([0, 1], seed=11, draw=i)) for i in range(2000)]
        uni.free()
        return det, sub, bd, ud

    det, sub, bd, ud = run_collect(World(1), body)
    assert all(d == [1, 0, 1, 1] for d in det)
    assert sub == [1, 1]
    assert set(bd) <= {(0, 0), (1, 1)} and len(set(bd)) == 2
    for o in [(0, 0), (0, 1), (1, 0), (1, 1)]:
        f = ud.count(o) / len(ud)
        assert abs(f - 0.25) < 0.04  # 4 sigma at 2000 draws


def test_sample_requires_normalised_state():
    def body(rk):
        m = MPS.bitstring(rk, [0, 1], 2)
        m._set(0, qtnh.ops.scale(m.sites[0], 3.0))
        try:
            m.sample([0], seed=1)
            e = None
        except qtnh.PreconditionError as ex:
            e = ex
        m.free()
        return e

    assert isinstance(run_collect(World(1), body), qtnh.PreconditionError)


def dense_apply(sv, n, targets, gate):
    """Apply a gate on `targets` (qubit 0 most significant) to a dense statevector."""
    k = len(targets)
    t = sv.reshape([2] * n)
    g = gate.reshape([2] * (2 * k))
    t = np.tensordot(g, t, axes=(list(range(k, 2 * k)), targets))
    rest = [q for q in range(n) if q not in targets]
    order = list(targets) + rest
    return np.transpose(t, np.argsort(order)).reshape(-1)


@pytest.mark.parametrize("targets", [[2], [1, 2], [1, 3], [0, 2, 5], [4, 5]])
def test_apply_raw_gate_non_adjacent_vs_dense(targets):
    k = len(targets)
    gate = circuits.rng_normals(30 + k, 4**k).reshape(2**k, 2**k)
    gate, _ = np.linalg.qr(gate)  # unitary

    def body(rk):
        m = MPS.random(rk, 6, 4, seed=12, chi=64)
        before = m.to_statevector()
        m.apply_gate_sites(targets, gate)
        after = m.to_statevector()
        centre = m.centre
        m.free()
        return before, after, centre

    before, after, centre = run_collect(World(1), body)
    assert rel_l2(after, dense_apply(before, 6, targets, gate)) < 1e-10
    assert centre == targets[0]


def test_apply_raw_gate_identity_and_errors():
    def body(rk):
        m = MPS.random(rk, 5, 4, seed=3, chi=16)
        before = m.to_statevector()
        m.apply_gate_sites([1, 3], np.eye(4))
        after = m.to_statevector()
        errs = []
        for t, g in (([3, 1], np.eye(4)), ([1, 2], np.eye(2))):
            try:
                m.apply_gate_sites(t, g)
            except qtnh.InvalidArgument as e:
                errs.append(e)
        m.free()
        return before, after, errs

    before, after, errs = run_collect(World(1), body)
    assert rel_l2(after, before) < 1e-12
    assert len(errs) == 2


@pytest.mark.parametrize("first,k", [(0, 2), (2, 3), (1, 4)])
def test_apply_mpo_vs_dense(first, k):
    from paper_2505_06119_b200.mps import mpo_from_operator
    op = circuits.rng_normals(50 + k, 4**k).reshape(2**k, 2**k)
    mpo = mpo_from_operator(op, k)

    def body(rk):
        m = MPS.random(rk, 6, 4, seed=21, chi=64)
        before = m.to_statevector()
        m.apply_mpo(mpo, first)
        after = m.to_statevector()
        centre = m.centre
        m.free()
        return before, after, centre

    before, after, centre = run_collect(World(1), body)
    assert rel_l2(after, dense_apply(before, 6, list(range(first, first + k)), op)) < 1e-9
    assert centre == first


def test_apply_mpo_fsim_phase_and_identity():
    """identity MPO leaves the state; fSim on |11> gives e^{-i pi/6}."""
    from paper_2505_06119_b200.mps import mpo_from_operator

    def body(rk):
        m = MPS.bitstring(rk, [1, 1], 4)
        m.apply_mpo(mpo_from_operator(circuits.FSIM, 2))
        sv = m.to_statevector()
        m.free()
        r = MPS.random(rk, 4, 2, seed=8, chi=8)
        before = r.to_statevector()
        r.apply_mpo(mpo_from_operator(np.eye(4), 2), 1)
        after = r.to_statevector()
        r.free()
        return sv, before, after

    sv, before, after = run_collect(World(1), body)
    assert abs(sv[3] - np.exp(-1j * np.pi / 6)) < 1e-12 and np.allclose(sv[:3], 0)
    assert rel_l2(after, before) < 1e-12


def test_truncated_mpo_lowers_norm():
    from paper_2505_06119_b200.mps import mpo_from_operator
    op, _ = np.linalg.qr(circuits.rng_normals(77, 64).reshape(8, 8))

    def body(rk):
        m = MPS.random(rk, 8, 4, seed=31, chi=4)
        m.apply_mpo(mpo_from_operator(op, 3), 2)
        out = (m.norm2(), m.log_fidelity, max(m.bond_dims()))
        m.free()
        return out

    n2, logf, bmax = run_collect(World(1), body)
    assert n2 < 1.0 and logf < 0.0 and bmax <= 4


def test_canonicalize_rank_deficient_site_stays_isometric():
    """|00> then CNOT-like entangling that leaves a zero Schmidt value: bond 2 of a
    bitstring MPS after a gate has sigma = (1, 0). The canonical sites must still
    be isometries -- zero-sigma directions are dropped from the bond."""
    cnot = np.eye(4, dtype=complex)[[0, 1, 3, 2]]

    def body(rk):
        m = MPS.bitstring(rk, [0, 0, 0], chi=4)
        m.apply_layer([(0, 1)], cnot)  # product state stays product: bond (0,1) sigma = (1, 0)
        m.apply_1q(1, circuits.H)
        m.apply_layer([(1, 2)], cnot)
        before = m.to_statevector()
        m.canonicalize(2)
        after = m.to_statevector()
        out = (before, after, site_arrays(m))
        m.free()
        return out

    before, after, sites = run_collect(World(1), body)
    assert rel_l2(after, before) < 1e-12
    for q, a in enumerate(sites[:2]):
        r = a.shape[2]
        g = np.einsum("lsr,lsk->rk", a.conj(), a)
        assert np.allclose(g, np.eye(r), atol=1e-10), (q, a.shape)


def test_apply_layer_native_matches_dense_evolution():
    """qtnh_mps_apply_layer (one native call per layer) against the dense statevector
    with the same gates, no truncation (chi ample), and with truncation the kept
    weights multiply to the reported fidelity."""
    from paper_2505_06119_b200 import mps as M

    n, depth = 8, 6
    layers = M.rcs_1d_layers(n, depth, 5)

    def body(rk):
        m = MPS(rk, n, 64)
        psi = np.zeros(2**n, complex)
        psi[0] = 1
        for singles, pairs in layers:
            for q, g in enumerate(singles):
                m.apply_1q(q, M.SINGLE_QUBIT[g])
                psi = np.moveaxis(np.tensordot(M.SINGLE_QUBIT[g], np.moveaxis(psi.reshape([2] * n), q, 0),
                                               axes=([1], [0])), 0, q).reshape(-1)
            m.apply_layer(pairs, circuits.FSIM)
            for q, _ in pairs:
                t = np.moveaxis(psi.reshape([2] * n), [q, q + 1], [0, 1]).reshape(4, -1)
                t = (circuits.FSIM @ t).reshape([2, 2] + [2] * (n - 2))
                psi = np.moveaxis(t, [0, 1], [q, q + 1]).reshape(-1)
        out = (m.to_statevector(), psi, m.log_fidelity)
        m.free()
        return out

    got, want, logf = run_collect(World(1), body)
    assert logf == 0.0
    assert rel_l2(got, want) < 1e-12
