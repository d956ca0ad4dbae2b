import time, sys, os
sys.path.insert(0, os.getcwd())
t0=time.time()
import numpy as np
import oracle
from paper_2505_06119_b200 import circuits
from paper_2505_06119_b200.qtnh import IndexTuple, Tensor, World, DistParams, qft, lib, check
print("import", time.time()-t0, flush=True)
P = oracle.port()
def T(label, f):
    t=time.time(); r=f(); print(f"{label}: {time.time()-t:.3f}s", flush=True); return r
for rep in range(3):
  for n, split, world in [(7,3,8),(8,0,1),(20,0,1)]:
    st = T("counter_state", lambda: circuits.counter_state(23+n, 2**n))
    st /= np.linalg.norm(st)
    def body(rk):
        t1=time.time()
        t = Tensor.from_global(rk, IndexTuple([2]*n, split), DistParams(1,1,0), st)
        t2=time.time()
        qft(t, swaps=True)
        rk.synchronize()
        t3=time.time()
        v = t.to_global_vector()
        t4=time.time()
        return (t2-t1, t3-t2, t4-t3)
    w = T(f"World({world})", lambda: World(world))
    r = T("run", lambda: w.run(body))
    print("  phases rank0", r[0], flush=True)
    T("del", lambda: w.__del__() if hasattr(w,'__del__') else None)
    T("oracle qft", lambda: P.qft(n, st))
