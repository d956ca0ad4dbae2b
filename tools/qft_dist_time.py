"""Whole-QFT time on a state sharded over a local world (all ranks on this GPU):
usage: python tools/qft_dist_time.py n world [peer_direct 0|1]"""
import os
import sys
import threading

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch

from paper_2505_06119_b200 import qtnh
from paper_2505_06119_b200.qtnh import DistParams, IndexTuple, Tensor, World, check, lib

n, w = int(sys.argv[1]), int(sys.argv[2])
if len(sys.argv) > 3:
    check(lib.qtnh_set_option(b"peer_direct", float(sys.argv[3])))
k = w.bit_length() - 1
res = []
lock = threading.Lock()


def body(rk):
    st = torch.cuda.Stream()
    rk.set_stream(st.cuda_stream)
    t = Tensor.dense(rk, IndexTuple([2] * n, k), DistParams(1, 1, 0), None)
    for rep in range(3):
        rk.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        qtnh.qft(t)
        e1.record(st)
        e1.synchronize()
        if rep == 2:
            with lock:
                res.append(e0.elapsed_time(e1))


World(w).run(body)
print(f"qft n={n} world={w} (one GPU) peer_direct={sys.argv[3] if len(sys.argv) > 3 else 1}: {max(res):.2f} ms")
