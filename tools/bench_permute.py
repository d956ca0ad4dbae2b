"""Permutation throughput of the strided-copy engine on a 2^28 qubit tensor (4 GiB):
full bit reversal, a C1-style random permutation, and single qubit moves."""
import os
import sys

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch

from paper_2505_06119_b200.qtnh import IndexTuple, Tensor, World, ops

n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
rng = np.random.default_rng(5)
perms = {"reverse": list(reversed(range(n))), "random": [int(x) for x in rng.permutation(n)],
         "swap_0_last": [n - 1] + list(range(1, n - 1)) + [0], "rotate1": list(range(1, n)) + [0]}


def body(rk):
    st = torch.cuda.Stream()
    rk.set_stream(st.cuda_stream)
    t = Tensor.dense(rk, IndexTuple([2] * n, 0), None, None)
    for name, p in perms.items():
        u = ops.permute(t, p, 0)
        u.free()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(5):
            u = ops.permute(t, p, 0)
            u.free()
        e1.record(st)
        e1.synchronize()
        ms = e0.elapsed_time(e1) / 5
        print(f"{name:12s} {ms:7.3f} ms  {32 * 2**n / ms / 1e6:7.0f} GB/s")


World(1).run(body)
