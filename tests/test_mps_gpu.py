"""Config 4 structure at reduced size: the 1-D RCS brickwork evolved as an MPS with
truncated two-site updates, against the same sequence of reference operations
(contract = t2m -> pgemm -> m2t, gate as contraction + permute back, psvd +
truncate_svd + absorb_singular_left) run by the unmodified reference."""
import numpy as np
import pytest

import oracle
from conftest import rel_l2
from paper_2505_06119_b200 import circuits, mps
from paper_2505_06119_b200.qtnh import World

pytestmark = pytest.mark.gpu
TOL = 1e-10


def reference_mps(n, layers, chi):
    R = oracle.ref()
    sites = []
    for _ in range(n):
        sites.append(([1, 2, 1], np.array([1, 0], dtype=complex)))
    fid = 0.0
    svals = []

    def gate_on(dims, data, pos, g):
        # contract(data, gate) pairing data[pos[k]] with gate input k, then permute back
        k = len(pos)
        gd = [2] * (2 * k)
        out, od, _ = R.contract(1, dims, 0, None, data, gd, 0, None, g.reshape(-1), list(pos),
                                list(range(k, 2 * k)))
        nd = len(dims)
        perm, opens = [], 0
        for p in range(nd):
            if p in pos:
                perm.append(nd - k + pos.index(p))
            else:
                perm.append(opens)
                opens += 1
        res, rd, _, _ = R.permute(1, od, 0, None, out, perm, 0)
        return rd, res

    for singles, pairs in layers:
        for q, gi in enumerate(singles):
            d, v = sites[q]
            sites[q] = gate_on(d, v, [1], mps.SINGLE_QUBIT[gi])
        for q, _ in pairs:
            (da, a), (db, b) = sites[q], sites[q + 1]
            th, td, _ = R.contract(1, da, 0, None, a, db, 0, None, b, [2], [0])
            td, th = gate_on(td, th, [1, 2], circuits.FSIM)
            m_, n_ = td[0] * td[1], td[2] * td[3]
            k = min(m_, n_)
            keep = min(chi, k)
            u, s, vh = R.svd(th.reshape(m_, n_), chi=k, absorb=0)
            if keep < k:
                fid += np.log(np.sum(s[:keep] ** 2) / np.sum(s**2))
            u, s, vh = R.svd(th.reshape(m_, n_), chi=keep, absorb=1)
            svals.append(s)
            sites[q] = ([td[0], td[1], keep], u.reshape(-1))
            sites[q + 1] = ([keep, td[2], td[3]], vh.reshape(-1))
    return sites, fid, svals


def amplitudes_np(sites, bits):
    out = []
    for b in bits:
        env = np.ones((1,), complex)
        for q, (d, v) in enumerate(sites):
            env = env @ v.reshape(d)[:, b[q], :]
        out.append(env[0])
    return np.array(out)


@pytest.mark.parametrize("n,depth,chi,batched", [(8, 6, 4, False), (10, 8, 8, True), (12, 6, 64, True),
                                                 (10, 8, 8, False)])
def test_mps_rcs_vs_reference(n, depth, chi, batched):
    if not oracle.ref_available():
        pytest.skip("reference build absent")
    seed = 40
    layers = mps.rcs_1d_layers(n, depth, seed)
    rng = np.random.default_rng(seed)
    bits = rng.integers(0, 2, size=(64, n))
    ref_sites, ref_fid, ref_s = reference_mps(n, layers, chi)
    want = amplitudes_np(ref_sites, bits)

    def body(rk):
        m, recs = mps.run_rcs_mps(rk, n, depth, chi, seed, layers=layers, batched=batched)
        amps = m.amplitudes(bits)
        res = (amps, m.log_fidelity, [r[3] for r in recs], m.bond_dims())
        m.free()
        return res

    amps, fid, svals, bonds = World(1).run(body)[0]
    assert max(bonds) <= chi
    for s_g, s_r in zip(svals, ref_s):
        assert np.allclose(s_g, s_r, rtol=1e-10, atol=1e-13)
    assert abs(fid - ref_fid) < 1e-10
    assert rel_l2(amps, want) < TOL


def test_mps_untruncated_matches_statevector():
    """chi ample: the MPS is exact, amplitudes equal a dense statevector run."""
    n, depth = 8, 5
    layers = mps.rcs_1d_layers(n, depth, 3)
    psi = np.zeros(2**n, complex)
    psi[0] = 1
    P = oracle.port()
    for singles, pairs in layers:
        for q, g in enumerate(singles):
            psi = P.gate([2] * n, psi, [q], mps.SINGLE_QUBIT[g])
        for q, _ in pairs:
            psi = P.gate([2] * n, psi, [q, q + 1], circuits.FSIM)
    bits = np.array([[(i >> (n - 1 - q)) & 1 for q in range(n)] for i in range(2**n)])

    def body(rk):
        m, _ = mps.run_rcs_mps(rk, n, depth, 64, 3, layers=layers)
        a = m.amplitudes(bits)
        m.free()
        return a

    amps = World(1).run(body)[0]
    assert rel_l2(amps, psi) < TOL


@pytest.mark.parametrize("world,n,chi", [(2, 10, 8), (3, 10, 4), (4, 12, 16),
                                         (4, 16, 8)])  # boundaries 3, 7, 11: both neighbours per layer
def test_distributed_mps_matches_single_rank(world, n, chi):
    """sites sharded over ranks, boundary pairs after one site
    exchange per layer; the final state and the total kept weight equal the
    single-rank run."""
    import numpy as np

    from paper_2505_06119_b200 import mps
    from paper_2505_06119_b200.qtnh import World

    depth, seed = 6, 5

    def single(rk):
        m, recs = mps.run_rcs_mps(rk, n, depth, chi, seed)
        out = (m.to_statevector(), m.log_fidelity)
        m.free()
        return out

    want_sv, want_logf = World(1).run(single)[0]

    def dist(rk):
        m, recs = mps.run_rcs_mps(rk, n, depth, chi, seed, distributed=True)
        out = (m.local_sites(), m.log_fidelity, len(recs))
        m.free()
        return out

    parts = World(world).run(dist)
    sites = {}
    for loc, _, _ in parts:
        sites.update(loc)
    assert sorted(sites) == list(range(n))
    acc = sites[0]
    for q in range(1, n):
        acc = np.tensordot(acc, sites[q], axes=([acc.ndim - 1], [0]))
    sv = acc.reshape(-1)
    assert np.linalg.norm(sv - want_sv) / np.linalg.norm(want_sv) < 1e-10
    assert abs(sum(p[1] for p in parts) - want_logf) < 1e-10
    assert sum(p[2] for p in parts) == sum(len(range(l % 2, n - 1, 2)) for l in range(depth))
