import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
import oracle
from conftest import rel_l2, bits
from paper_2505_06119_b200 import circuits, qtnh
from paper_2505_06119_b200.qtnh import DistParams, IndexTuple, Tensor, World, apply_gate, ops, run_collect, ABSORB_NONE
P = oracle.port()
bad = 0
# gates on sharded qubit states
for seed in range(60):
    rng = np.random.default_rng(5000 + seed)
    world = int(rng.choice([1, 2, 4, 8])); lw = int(np.log2(world))
    n = int(rng.integers(max(lw + 2, 3), 13))
    split = lw
    k = int(rng.integers(1, 4))
    targets = [int(x) for x in rng.permutation(n)[:k]]
    D = 2 ** k
    diag = bool(rng.integers(0, 2))
    gate = circuits.rng_normals(seed, D if diag else D * D)
    g = circuits.counter_state(seed + 1, 2 ** n)
    def body(rk):
        t = Tensor.from_global(rk, IndexTuple([2] * n, split), DistParams(1, 1, 0), g)
        apply_gate(t, targets, gate, diagonal=diag)
        return t.to_global_vector()
    try:
        got = World(world).run(body)[0]
        want = P.gate([2] * n, g, targets, gate, diagonal=diag)
        e = rel_l2(got, want)
        if not e < 1e-12:
            bad += 1; print("GATE MISMATCH", seed, world, n, targets, diag, e, flush=True)
    except Exception as ex:
        bad += 1; print("GATE ERROR", seed, world, n, targets, diag, repr(ex)[:200], flush=True)
# svd random shapes
def gpu_svd(a, chi):
    m, n = a.shape
    def body(rk):
        t = Tensor.from_global(rk, IndexTuple([m, n], 0), None, a.reshape(-1))
        u, s, vh = qtnh.svd(t, [0], [1], chi, ABSORB_NONE)
        k = s.size
        return u.to_global_vector().reshape(m, k), s, vh.to_global_vector().reshape(k, n)
    return run_collect(World(1), body)
for seed in range(40):
    rng = np.random.default_rng(7000 + seed)
    m, n = int(rng.integers(1, 200)), int(rng.integers(1, 200))
    k = min(m, n)
    chi = int(rng.integers(0, k + 20))
    a = circuits.rng_normals(seed + 50, m * n).reshape(m, n)
    if seed % 3 == 0 and k > 4:  # rank deficient
        r = int(rng.integers(1, k))
        a = a[:, :r] @ circuits.rng_normals(seed + 90, r * n).reshape(r, n)
    try:
        u, s, vh = gpu_svd(a, chi)
        U, S, VH = np.linalg.svd(a, full_matrices=False)
        keep = min(chi if chi > 0 else k, k)
        want = (U[:, :keep] * S[:keep]) @ VH[:keep]
        e1 = rel_l2((u * s) @ vh, want) if np.linalg.norm(want) > 0 else np.linalg.norm((u * s) @ vh)
        e2 = np.max(np.abs(s[:keep] - S[:keep])) / max(S[0], 1e-300)
        if not (e1 < 1e-10 and e2 < 1e-10 and s.size == (chi if chi > 0 else k)):
            bad += 1; print("SVD MISMATCH", seed, m, n, chi, e1, e2, s.size, flush=True)
    except Exception as ex:
        bad += 1; print("SVD ERROR", seed, m, n, chi, repr(ex)[:200], flush=True)
print("bad", bad)
