import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2505_06119_b200 import mps
from paper_2505_06119_b200.qtnh import World
# larger bonds than the suite's cases: the layer's shape groups run on two host threads
# (big_work >= 1e9) and single-matrix SVDs replay their sweeps as graphs (>= 512 rows)
n, depth, chi, seed = 24, 22, 512, 5
def single(rk):
    m, recs = mps.run_rcs_mps(rk, n, depth, chi, seed)
    out = ({q: t.to_global_vector() for q, t in enumerate(m.sites)}, m.log_fidelity); m.free(); return out
want_sites, want_logf = World(1).run(single)[0]
for world in (2, 3):
    def dist(rk):
        m, recs = mps.run_rcs_mps(rk, n, depth, chi, seed, distributed=True)
        out = (m.local_sites(), m.log_fidelity, len(recs)); m.free(); return out
    parts = World(world).run(dist)
    sites = {}
    for loc, _, _ in parts: sites.update(loc)
    worst = max(float(np.max(np.abs(sites[q].reshape(-1) - want_sites[q]))) for q in range(n))
    print("world", world, "max |site diff|", worst, "logf diff", abs(sum(p[1] for p in parts) - want_logf), flush=True)
