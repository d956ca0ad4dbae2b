"""Gate-kernel throughput on a 2^30 state (16 GiB): dense 1-/2-/3-/4-qubit gates on
inner, middle and outer targets and a diagonal CP, 32 B per amplitude per gate."""
import os
import sys

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch

from paper_2505_06119_b200 import circuits
from paper_2505_06119_b200.qtnh import IndexTuple, Tensor, World, apply_gate

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
cases = [("H q0", [0], circuits.H, False), ("H q15", [15], circuits.H, False), ("H q29", [n - 1], circuits.H, False),
         ("fSim q3,q20", [3, 20], circuits.FSIM, False), ("3q", [2, 11, 25], np.eye(8), False),
         ("4q", [1, 9, 17, 28], np.eye(16), False), ("CP diag", [7, 22], circuits.cp_diag(0.3), True)]


def body(rk):
    st = torch.cuda.Stream()
    rk.set_stream(st.cuda_stream)
    t = Tensor.dense(rk, IndexTuple([2] * n, 0), None, None)
    for name, tg, g, diag in cases:
        apply_gate(t, tg, g, diagonal=diag)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(4):
            apply_gate(t, tg, g, diagonal=diag)
        e1.record(st)
        e1.synchronize()
        ms = e0.elapsed_time(e1) / 4
        print(f"{name:12s} {ms:7.3f} ms  {32 * 2**n / ms / 1e6:7.0f} GB/s (32 B/amp convention)")


World(1).run(body)
