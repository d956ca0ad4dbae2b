"""GPU parity of the truncated SVD split (linalg::psvd + truncate_svd + absorb,
linalg.hpp:441-523) against the unmodified reference (zgesdd via OpenBLAS).

Factors are unique only up to phases, so parity is checked on the singular
values and on phase-invariant products: the truncated reconstruction U S Vh
(relative L2 <= 1e-10, north star), U^H U = I, Vh Vh^H = I, and the absorbed
factors' product."""
import ctypes as C

import numpy as np
import pytest

import oracle
from conftest import golden, rel_l2
from paper_2505_06119_b200 import circuits, qtnh
from paper_2505_06119_b200.qtnh import (ABSORB_LEFT, ABSORB_NONE, ABSORB_RIGHT, ABSORB_SPLIT, IndexTuple, Tensor,
                                        World, run_collect)

pytestmark = pytest.mark.gpu
TOL = 1e-10


def gpu_svd(a, chi=0, absorb=ABSORB_NONE):
    m, n = a.shape

    def body(rk):
        t = Tensor.from_global(rk, IndexTuple([m, n], 0), None, a.reshape(-1))
        u, s, vh = qtnh.svd(t, [0], [1], chi, absorb)
        k = s.size
        return u.to_global_vector().reshape(m, k), s, vh.to_global_vector().reshape(k, n)

    return run_collect(World(1), body)


def test_svd_golden_truncated_and_padded():
    meta, z = golden("svd")
    a = z["a"]
    u, s, vh = gpu_svd(a, chi=16, absorb=ABSORB_LEFT)
    assert np.allclose(s, z["s"], rtol=1e-12, atol=1e-13)
    assert rel_l2(u @ vh, z["u"] @ z["vh"]) < TOL
    u2, s2, vh2 = gpu_svd(a, chi=64, absorb=ABSORB_NONE)  # chi > rank: zero padding (linalg.hpp:488-501)
    assert s2.shape == (64,) and np.all(s2[40:] == 0)
    assert np.all(u2[:, 40:] == 0)
    assert np.allclose(s2, z["s_pad"], rtol=1e-12, atol=1e-13)
    assert rel_l2((u2 * s2) @ vh2, a) < TOL


@pytest.mark.parametrize("m,n,chi", [(64, 64, 0), (96, 130, 40), (130, 96, 40), (1, 7, 0), (7, 1, 0),
                                     (256, 256, 100), (33, 47, 60)])
def test_svd_shapes_vs_numpy(m, n, chi):
    a = circuits.rng_normals(m * 7 + n, m * n).reshape(m, n)
    k = min(m, n)
    u, s, vh = gpu_svd(a, chi=chi)
    sv = np.linalg.svd(a, compute_uv=False)
    kk = chi if chi > 0 else k
    keep = min(kk, k)
    assert np.allclose(s[:keep], sv[:keep], rtol=1e-12, atol=1e-12 * sv[0])
    assert np.all(s[keep:] == 0)
    U, S, VH = np.linalg.svd(a, full_matrices=False)
    want = (U[:, :keep] * S[:keep]) @ VH[:keep]
    assert rel_l2((u * s) @ vh, want) < TOL
    assert np.allclose(u[:, :keep].conj().T @ u[:, :keep], np.eye(keep), atol=1e-12)
    assert np.allclose(vh[:keep] @ vh[:keep].conj().T, np.eye(keep), atol=1e-12)


def test_absorb_modes():
    a = circuits.rng_normals(3, 50 * 40).reshape(50, 40)
    _, s, _ = gpu_svd(a, chi=20)
    for mode in (ABSORB_LEFT, ABSORB_RIGHT, ABSORB_SPLIT):
        u, s2, vh = gpu_svd(a, chi=20, absorb=mode)
        assert np.allclose(s2, s, rtol=1e-13)
        U, S, VH = np.linalg.svd(a, full_matrices=False)
        assert rel_l2(u @ vh, (U[:, :20] * S[:20]) @ VH[:20]) < TOL
        if mode == ABSORB_LEFT:
            assert np.allclose(np.linalg.norm(u, axis=0), s, rtol=1e-12)
        if mode == ABSORB_RIGHT:
            assert np.allclose(np.linalg.norm(vh, axis=1), s, rtol=1e-12)
        if mode == ABSORB_SPLIT:
            assert np.allclose(np.linalg.norm(u, axis=0), np.sqrt(s), rtol=1e-12)


def test_rank_deficient_and_zero():
    rng = np.random.default_rng(2)
    b = rng.standard_normal((60, 5)) + 1j * rng.standard_normal((60, 5))
    c = rng.standard_normal((5, 50)) + 1j * rng.standard_normal((5, 50))
    a = b @ c  # rank 5
    u, s, vh = gpu_svd(a, chi=8)
    assert np.all(s[5:] < 1e-12 * s[0])
    assert rel_l2((u * s) @ vh, a) < TOL
    z = np.zeros((8, 6), complex)
    u, s, vh = gpu_svd(z)
    assert np.all(s == 0) and np.all((u * s) @ vh == 0)


@pytest.mark.parametrize("cross", ["1", "0"])
def test_svd_graded_spectrum(cross, monkeypatch):
    """Singular values spanning 12 decades (an MPS theta's graded spectrum): the
    cross-Gram sweeps must hand over to full Grams and still converge to the
    truncated reconstruction within the north-star tolerance."""
    import subprocess
    import sys
    code = (
        "import numpy as np, sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests');"
        "from test_svd_gpu import gpu_svd; from conftest import rel_l2;"
        "rng = np.random.default_rng(7); n = 320;"
        "q1, _ = np.linalg.qr(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)));"
        "q2, _ = np.linalg.qr(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)));"
        "sv = np.logspace(0, -12, n); a = (q1 * sv) @ q2.conj().T;"
        "u, s, vh = gpu_svd(a, chi=160);"
        "U, S, VH = np.linalg.svd(a, full_matrices=False);"
        "assert np.allclose(s, S[:160], rtol=1e-9, atol=1e-15), 'singular values';"
        "assert rel_l2((u * s) @ vh, (U[:, :160] * S[:160]) @ VH[:160]) < 1e-10, 'reconstruction';"
        "print('ok')"
    )
    import os
    env = dict(os.environ, QTNH_SVD_CROSS=cross)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-3000:]


def test_svd_vs_reference_theta_like():
    """MPS two-site theta (chi_l, d, d, chi_r) -> (chi_l d) x (d chi_r), truncated."""
    if not oracle.ref_available():
        pytest.skip("reference build absent")
    R = oracle.ref()
    chi = 64
    a = circuits.rng_normals(77, (2 * chi) ** 2).reshape(2 * chi, 2 * chi)
    ru, rs, rvh = R.svd(a, chi=chi, absorb=1)
    u, s, vh = gpu_svd(a, chi=chi, absorb=ABSORB_LEFT)
    assert np.allclose(s, rs, rtol=1e-12)
    assert rel_l2(u @ vh, ru @ rvh) < TOL


def test_svd_batched_device_api():
    import torch

    batch, m, n, chi = 3, 70, 90, 30
    a = np.stack([circuits.rng_normals(10 + i, m * n).reshape(m, n) for i in range(batch)])
    ta = torch.from_numpy(a).cuda()
    tu = torch.empty((batch, m, chi), dtype=torch.complex128, device="cuda")
    ts = torch.empty((batch, chi), dtype=torch.float64, device="cuda")
    tv = torch.empty((batch, chi, n), dtype=torch.complex128, device="cuda")

    def body(rk):
        rk.set_stream(torch.cuda.current_stream().cuda_stream)
        qtnh.check(qtnh.lib.qtnh_svd_device(rk._h, batch, m, n, C.c_void_p(ta.data_ptr()), chi, ABSORB_RIGHT,
                                            C.c_void_p(tu.data_ptr()), C.c_void_p(ts.data_ptr()),
                                            C.c_void_p(tv.data_ptr())))
        torch.cuda.synchronize()

    World(1).run(body)
    for i in range(batch):
        U, S, VH = np.linalg.svd(a[i], full_matrices=False)
        assert np.allclose(ts[i].cpu().numpy(), S[:chi], rtol=1e-12)
        assert rel_l2(tu[i].cpu().numpy() @ tv[i].cpu().numpy(), (U[:, :chi] * S[:chi]) @ VH[:chi]) < TOL


@pytest.mark.slow
def test_svd_c4_size_vs_reference():
    """Config 4 shape: theta 2048 x 2048 truncated to chi = 1024, against zgesdd."""
    if not oracle.ref_available():
        pytest.skip("reference build absent")
    import os

    R = oracle.ref()
    R.set_threads(os.cpu_count() or 1)
    n, chi = 2048, 1024
    # a realistic spectrum: decaying singular values (entangled MPS bond)
    rng = np.random.default_rng(4)
    q1, _ = np.linalg.qr(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
    q2, _ = np.linalg.qr(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
    sv = np.exp(-np.arange(n) / 300.0)
    a = (q1 * sv) @ q2
    ru, rs, rvh = R.svd(a, chi=chi, absorb=1)
    u, s, vh = gpu_svd(a, chi=chi, absorb=ABSORB_LEFT)
    assert np.allclose(s, rs, rtol=1e-11, atol=1e-13)
    assert rel_l2(u @ vh, ru @ rvh) < TOL


def _with_spectrum(m, n, s, seed):
    rng = np.random.default_rng(seed)
    u, _ = np.linalg.qr(rng.standard_normal((m, m)) + 1j * rng.standard_normal((m, m)))
    v, _ = np.linalg.qr(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
    k = min(m, n)
    return (u[:, :k] * np.asarray(s)) @ v[:, :k].conj().T


@pytest.mark.parametrize("case", ["two_exact", "two_tight", "gapped_wide", "no_gap", "rect"])
def test_svd_spectral_split_path(case):
    """The truncated SVD's spectral-split path (svd_split.cu: projector of A A^H by
    Newton-Schulz, quarter-size Jacobi solves) against numpy on matrices with a
    chosen spectrum: exactly two values (config 4's thetas), two tight clusters,
    a wide gap (may fall back), no gap (must fall back); the result is the same
    truncated factorisation either way, and the path actually taken is checked
    where it is certain."""
    m, n, chi = 256, 256, 128
    if case == "two_exact":
        s = [0.7] * chi + [0.36] * (m - chi)
    elif case == "two_tight":
        s = list(0.7 * (1 + 1e-7 * np.linspace(0, 1, chi))) + list(0.36 * (1 + 1e-7 * np.linspace(0, 1, m - chi)))
    elif case == "gapped_wide":
        s = list(np.linspace(0.8, 0.6, chi)) + list(np.linspace(0.3, 0.1, m - chi))
    elif case == "no_gap":
        s = list(np.linspace(1.0, 0.01, m))
    else:
        m, n, chi = 192, 320, 96
        s = [0.9] * chi + [0.2] * (m - chi)
    s = np.sort(np.asarray(s))[::-1]
    a = _with_spectrum(m, n, s, 7)
    before = int(qtnh.lib.qtnh_svd_split_count())
    u, sv, vh = gpu_svd(a, chi=chi, absorb=ABSORB_LEFT)
    took = int(qtnh.lib.qtnh_svd_split_count()) - before
    U, S, VH = np.linalg.svd(a, full_matrices=False)
    want = (U[:, :chi] * S[:chi]) @ VH[:chi]
    assert rel_l2(u @ vh, want) < TOL
    assert np.max(np.abs(sv - S[:chi])) <= TOL * S[0]
    # Vh rows orthonormal; U = U_true S (absorb left): U^H U = S^2
    assert np.allclose(vh @ vh.conj().T, np.eye(chi), atol=1e-12)
    assert np.allclose(u.conj().T @ u, np.diag(sv**2), atol=1e-12)
    if case in ("two_exact", "two_tight", "rect"):
        assert took == 1
    if case == "no_gap":
        assert took == 0


def _iso_cols(u):
    return np.abs(u.conj().T @ u - np.eye(u.shape[1])).max()


@pytest.mark.parametrize("m,n,rank", [(48, 40, 5), (40, 48, 5), (8, 6, 0), (64, 64, 1), (300, 260, 120)])
def test_svd_null_directions_are_completed(m, n, rank):
    """Rank-deficient input: the bases stay isometries on their non-absorbed side
    (zgesdd's do, linalg.hpp:441-471) -- null singular directions get an
    orthonormal completion instead of zero / noise vectors -- and U S Vh is
    unchanged."""
    rng = np.random.default_rng(m + n + rank)
    x = rng.standard_normal((m, max(rank, 1))) + 1j * rng.standard_normal((m, max(rank, 1)))
    y = rng.standard_normal((max(rank, 1), n)) + 1j * rng.standard_normal((max(rank, 1), n))
    a = (x @ y) * (1.0 if rank else 0.0)
    k = min(m, n)
    for mode in (ABSORB_NONE, ABSORB_LEFT, ABSORB_RIGHT):
        u, s, vh = gpu_svd(a, chi=0, absorb=mode)
        assert s.shape == (k,)
        assert np.all(s[rank:] <= 1e-12 * max(s[0], 1.0))
        if rank:
            assert np.allclose(s[:rank], np.linalg.svd(a, compute_uv=False)[:rank], rtol=1e-12)
        uu = u if mode != ABSORB_LEFT else None
        vv = vh if mode != ABSORB_RIGHT else None
        if uu is not None:
            assert _iso_cols(uu) < 1e-12, mode
        if vv is not None:
            assert _iso_cols(vv.conj().T) < 1e-12, mode
        prod = (u * s) @ vh if mode == ABSORB_NONE else u @ vh
        if rank:
            assert rel_l2(prod, a) < TOL
        else:
            assert np.abs(prod).max() == 0.0


def test_svd_null_cnot_bell_bond():
    """SPEC example: |00> then CNOT gives a Bell pair; its 2 x 2 theta has sigma = (1/sqrt2,
    1/sqrt2) but H alone on |00> gives rank 1: the second direction is null and
    must still be a unit vector orthogonal to the first."""
    a = np.array([[1.0, 0.0], [1.0, 0.0]], dtype=np.complex128) / np.sqrt(2)
    u, s, vh = gpu_svd(a, chi=2, absorb=ABSORB_NONE)
    assert np.allclose(s, [1.0, 0.0], atol=1e-15)
    assert _iso_cols(u) < 1e-14 and _iso_cols(vh.conj().T) < 1e-14
    assert rel_l2((u * s) @ vh, a) < 1e-14


def test_svd_device_batch_null_completion():
    """qtnh_svd_device: a batch mixing a full-rank and a rank-3 matrix; the
    rank-deficient one gets orthonormal completions, the other is untouched."""
    import torch

    m, n, chi = 40, 56, 20
    rng = np.random.default_rng(11)
    full = rng.standard_normal((m, n)) + 1j * rng.standard_normal((m, n))
    low = (rng.standard_normal((m, 3)) + 1j * rng.standard_normal((m, 3))) @ (
        rng.standard_normal((3, n)) + 1j * rng.standard_normal((3, n)))
    a = np.stack([full, low])
    ta = torch.from_numpy(a).cuda()
    tu = torch.empty((2, m, chi), dtype=torch.complex128, device="cuda")
    ts = torch.empty((2, chi), dtype=torch.float64, device="cuda")
    tv = torch.empty((2, chi, n), dtype=torch.complex128, device="cuda")

    def body(rk):
        rk.set_stream(torch.cuda.current_stream().cuda_stream)
        qtnh.check(qtnh.lib.qtnh_svd_device(rk._h, 2, m, n, C.c_void_p(ta.data_ptr()), chi, ABSORB_NONE,
                                            C.c_void_p(tu.data_ptr()), C.c_void_p(ts.data_ptr()),
                                            C.c_void_p(tv.data_ptr())))
        torch.cuda.synchronize()

    World(1).run(body)
    for i in range(2):
        u, s, vh = tu[i].cpu().numpy(), ts[i].cpu().numpy(), tv[i].cpu().numpy()
        assert _iso_cols(u) < 1e-12 and _iso_cols(vh.conj().T) < 1e-12
        U, S, VH = np.linalg.svd(a[i], full_matrices=False)
        keep = 3 if i else chi
        assert np.allclose(s[:keep], S[:keep], rtol=1e-12)
        assert rel_l2((u * s) @ vh, (U[:, :chi] * S[:chi]) @ VH[:chi]) < TOL


@pytest.mark.parametrize("m,n,values", [(384, 384, (0.70719, 0.35957)), (256, 512, (1.0, 1.0)),
                                        (320, 320, (0.9, 0.5, 0.5000001, 0.1))])
def test_svd_clustered_spectrum_full_jacobi(m, n, values):
    """Exactly (or nearly) equal singular values in large clusters, chi = min(m, n) so
    the call takes the plain Jacobi: inside a cluster the sweeps end on the stagnation
    rule (off-norm within 10x of the tolerance and no longer falling), which must
    leave S, the isometries and the reconstruction at the parity tolerance."""
    k = min(m, n)
    rng = np.random.default_rng(m + n)
    q1, _ = np.linalg.qr(rng.standard_normal((m, k)) + 1j * rng.standard_normal((m, k)))
    q2, _ = np.linalg.qr(rng.standard_normal((n, k)) + 1j * rng.standard_normal((n, k)))
    sv = np.sort(np.repeat(np.asarray(values), -(-k // len(values)))[:k])[::-1]
    a = (q1 * sv) @ q2.conj().T
    u, s, vh = gpu_svd(a)
    assert np.max(np.abs(s - sv)) < TOL * sv[0]
    assert rel_l2((u * s) @ vh, a) < TOL
    assert np.max(np.abs(u.conj().T @ u - np.eye(k))) < TOL
    assert np.max(np.abs(vh @ vh.conj().T - np.eye(k))) < TOL
