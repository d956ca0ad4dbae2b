"""Time the two redistribution forms of the local world on the device:
peer-memory kernels vs pack -> exchange -> unpack. World of `w` ranks; on one
GPU all ranks share the device (peer pointers are plain device pointers), so
this measures the HBM cost of each form; on an NVLink node the same code moves
the bytes over NVLink.
usage: python tools/bench_redistribute.py [n_qubits] [world]"""
import os
import sys
import threading

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch

from paper_2505_06119_b200 import qtnh
from paper_2505_06119_b200.qtnh import DistParams, IndexTuple, Tensor, World, check, lib

n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
w = int(sys.argv[2]) if len(sys.argv) > 2 else 2
k = w.bit_length() - 1
res = {}
lock = threading.Lock()


def body(rk):
    st = torch.cuda.Stream()
    rk.set_stream(st.cuda_stream)
    t = Tensor.dense(rk, IndexTuple([2] * n, k), DistParams(1, 1, 0), None)
    perms = {}
    for lb in (n - 1, k):
        perm = list(range(n))
        perm[0], perm[lb] = perm[lb], perm[0]
        perms[lb] = perm
    for mode in (1, 0):
        if rk.rank() == 0:
            check(lib.qtnh_set_option(b"peer_direct", float(mode)))
        rk.barrier()
        for op in ("swap", "permute", "swap_outer", "permute_outer"):
            for rep in range(4):
                rk.barrier()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                lb = k if op.endswith("outer") else n - 1
                if op.startswith("swap"):
                    qtnh.swap_indices(t, 0, lb)
                else:
                    u = qtnh.ops.permute(t, perms[lb], k)
                e1.record(st)
                e1.synchronize()
                if op.startswith("permute"):
                    u.free()
                ms = e0.elapsed_time(e1)
                if rep == 3:
                    with lock:
                        res.setdefault((mode, op), []).append(ms)
    check(lib.qtnh_set_option(b"peer_direct", 1.0))


World(w).run(body)
tot = 16 * 2**n
for (mode, op), v in sorted(res.items()):
    ms = max(v)
    moved = tot if op.startswith("permute") else tot * (1 - 1 / 2)  # swap moves half the state
    print(f"{'peer' if mode else 'exchange':8s} {op:14s} n={n} world={w}: {ms:8.3f} ms  "
          f"(algorithmic r+w {2 * moved / ms / 1e6:7.1f} GB/s on one device)")
