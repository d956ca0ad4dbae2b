"""Config 0 (QFT-16, 144 gates on a 1 MiB state, latency-bound): gate by gate with
one launch per gate vs the same sequence replayed from a CUDA graph."""
import os
import sys
import time

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch

from paper_2505_06119_b200 import circuits
from paper_2505_06119_b200.qtnh import IndexTuple, Tensor, World, apply_gate, swap_indices

n = 16
gates = circuits.qft_gates(n, swaps=True)


def seq(t):
    for kind, q, g in gates:
        if kind == "h":
            apply_gate(t, q, g)
        elif kind == "cp":
            apply_gate(t, q, g, diagonal=True)
        else:
            swap_indices(t, q[0], q[1])


def body(rk):
    t = Tensor.dense(rk, IndexTuple([2] * n, 0), None, None)
    for _ in range(3):
        seq(t)
    rk.synchronize()
    reps = 20
    t0 = time.perf_counter()
    for _ in range(reps):
        seq(t)
    rk.synchronize()
    direct = (time.perf_counter() - t0) / reps
    with rk.capture() as g:
        seq(t)
    g.launch()
    rk.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        g.launch()
    rk.synchronize()
    graph = (time.perf_counter() - t0) / reps
    print(f"QFT-16 gate by gate ({len(gates)} gates): direct {direct * 1e3:.3f} ms, CUDA graph {graph * 1e3:.3f} ms "
          f"({direct / graph:.1f}x)")


World(1).run(body)
