"""Random circuit (config 3's 5x6 grid, depth 14) on a 30-qubit statevector (16 GiB):
gate-by-gate vs fused into <= 4-qubit blocks (circuits.fuse_gates). Reports device
time, state passes and the HBM rate per pass (32 B / amplitude / pass)."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=5)
    ap.add_argument("--cols", type=int, default=6)
    ap.add_argument("--depth", type=int, default=14)
    ap.add_argument("--seed", type=int, default=2025)
    ap.add_argument("--kmax", type=int, default=4)
    args = ap.parse_args()
    import numpy as np
    import torch

    from paper_2505_06119_b200 import circuits, mps, network, qtnh
    from paper_2505_06119_b200.qtnh import IndexTuple, Tensor, World

    n = args.rows * args.cols
    gates = [(list(qs), mps.SINGLE_QUBIT[g] if kind == "1q" else circuits.FSIM)
             for kind, qs, g in network.rcs_grid_circuit(args.rows, args.cols, args.depth, args.seed)]
    fused = circuits.fuse_gates(gates, args.kmax)
    out = {"n": n, "depth": args.depth, "gates": len(gates), "fused_blocks": len(fused),
           "fused_diagonal_blocks": sum(f.diagonal for f in fused),
           "block_sizes": {k: sum(len(f.qubits) == k for f in fused) for k in range(1, args.kmax + 1)}}

    def body(rk):
        st = torch.cuda.Stream()
        rk.set_stream(st.cuda_stream)
        t = Tensor.dense(rk, IndexTuple([2] * n, 0), None, None)
        v = torch.as_tensor(mps._DevView(t.device_ptr(), 2**n), device="cuda")

        def run(fn):
            with torch.cuda.stream(st):
                v.zero_()
                v[0] = 1.0
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            fn()
            e1.record(st)
            e1.synchronize()
            return e0.elapsed_time(e1) / 1e3

        out["gate_by_gate_s"] = run(lambda: [qtnh.apply_gate(t, qs, g) for qs, g in gates])
        ref = v[: 1 << 20].clone()
        out["fused_s"] = run(lambda: circuits.apply_fused(t, fused))
        out["fused_vs_gate_by_gate_rel_l2"] = float((v[: 1 << 20] - ref).norm() / ref.norm())
        out["norm_after"] = float(v.norm())
        byts = 32.0 * 2**n
        out["gate_by_gate_GBps_per_pass"] = len(gates) * byts / out["gate_by_gate_s"] / 1e9
        out["fused_GBps_per_pass"] = len(fused) * byts / out["fused_s"] / 1e9
        out["speedup"] = out["gate_by_gate_s"] / out["fused_s"]
        t.free()

    World(1).run(body)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
