"""NumPy model of the blocked one-sided Jacobi in csrc/svd.cu (same circle-method
tournament over 16-row blocks, one parallel inner sweep on each pair's 32 x 32
Gram, W^H applied to the pair's rows), used to tell algorithmic sweep counts from
kernel effects (item 1). Slow (pure Python loops): n <= 256.

  python tools/svd_block_model.py [n] [graded_decades] [--pair-sort] [--adapt]
"""
import sys

import numpy as np


def inner_sweep(G, B, thr=0.0):
    """One parallel cyclic Jacobi sweep on the Hermitian 2B x 2B G; returns V."""
    P2 = 2 * B
    G = G.copy()
    V = np.eye(P2, dtype=complex)
    for step in range(P2 - 1):
        M = np.eye(P2, dtype=complex)
        for tid in range(B):
            if tid == 0:
                p, q = step, P2 - 1
            else:
                p, q = (step + tid) % (P2 - 1), (step - tid + (P2 - 1)) % (P2 - 1)
            if p > q:
                p, q = q, p
            a, b, x = G[p, p].real, G[q, q].real, G[p, q]
            r2 = abs(x) ** 2
            c, s, ph = 1.0, 0.0, 1.0
            if r2 > 0 and not (r2 <= max(1e-34, thr * thr) * abs(a * b)):
                inv = 1 / np.sqrt(r2)
                ph = np.conj(x) * inv
                tau = 0.5 * (b - a) * inv
                t = np.copysign(1.0, tau) / (abs(tau) + np.sqrt(tau * tau + 1))
                c = 1 / np.sqrt(t * t + 1)
                s = t * c
            M[p, p], M[q, p], M[p, q], M[q, q] = c, -s * ph, s, c * ph
        V = V @ M
        G = M.conj().T @ G @ M
    return V


def off(X):
    G = X @ X.conj().T
    d = np.sqrt(np.real(np.diag(G)))
    R = np.abs(G) / np.maximum(np.outer(d, d), 1e-300)
    np.fill_diagonal(R, 0)
    return R.max()


def run(A, B=16, max_sweeps=60, tol=1e-13, pair_sort=False, adapt=None):
    X = A.copy()
    nblk2 = X.shape[0] // B
    npairs, rounds = nblk2 // 2, nblk2 - 1
    hist = []
    for sw in range(max_sweeps):
        hist.append(off(X))
        if hist[-1] < tol:
            return sw, hist
        for rd in range(rounds):
            for k in range(npairs):
                p, q = (rd, nblk2 - 1) if k == 0 else ((rd + k) % rounds, (rd - k + rounds) % rounds)
                idx = np.r_[p * B:(p + 1) * B, q * B:(q + 1) * B]
                Xp = X[idx]
                G = Xp @ Xp.conj().T
                V = inner_sweep(G, B, adapt(hist[-1]) if (adapt and sw > 0) else 0.0)
                if pair_sort:
                    d = np.real(np.diag(V.conj().T @ G @ V))
                    order = np.argsort(-d) if p < q else np.argsort(d)
                    V = V[:, order]
                X[idx] = V.conj().T @ Xp
    return max_sweeps, hist


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    n = int(args[0]) if args else 128
    dec = float(args[1]) if len(args) > 1 else 0.0
    rng = np.random.default_rng(7)
    if dec > 0:
        q1, _ = np.linalg.qr(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
        q2, _ = np.linalg.qr(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
        A = (q1 * np.logspace(0, -dec, n)) @ q2.conj().T
    else:
        A = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    # rotation threshold from the previous off-norm: skip |G_pq| < thr sqrt(G_pp G_qq)
    adapt = (lambda o: 0.1 * o * o) if "--adapt" in sys.argv else None
    sw, hist = run(A, pair_sort="--pair-sort" in sys.argv, adapt=adapt)
    print("sweeps", sw, " ".join("%.1e" % h for h in hist))
