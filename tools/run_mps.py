"""Config 4: 40-qubit 1-D RCS (depth 20) evolved as an MPS with chi = 1024 on one
GPU; reports total / per-layer time, bond dimensions, the truncation fidelity
(product of kept-weight ratios) and the amplitudes of 1024 seeded bitstrings."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=40)
    ap.add_argument("--depth", type=int, default=20)
    ap.add_argument("--chi", type=int, default=1024)
    ap.add_argument("--seed", type=int, default=2025)
    ap.add_argument("--bitstrings", type=int, default=1024)
    ap.add_argument("--amps-out", default="", help="save the bitstring amplitudes (.npy) for run-to-run comparison")
    ap.add_argument("--sequential", action="store_true", help="one SVD per update instead of batched layers")
    ap.add_argument("--world", type=int, default=1,
                    help="ranks (thread per rank, round-robin over the visible GPUs); > 1 shards the sites "
                         "(DistMPS, one site exchange per boundary per layer)")
    ap.add_argument("--reserve-gb", type=float, default=48,
                    help="map this much of the stream-ordered pool up front (option pool_reserve_gb)")
    args = ap.parse_args()
    import numpy as np
    import torch

    from paper_2505_06119_b200 import circuits, mps
    from paper_2505_06119_b200.qtnh import World
    from paper_2505_06119_b200 import qtnh as _q

    _q.check(_q.lib.qtnh_set_option(b"pool_reserve_gb", float(args.reserve_gb)))

    out = {"n": args.n, "depth": args.depth, "chi": args.chi}
    layers = mps.rcs_1d_layers(args.n, args.depth, args.seed)

    logf = {}

    def body(rk):
        torch.cuda.synchronize()
        rk.barrier()
        t0 = time.perf_counter()
        rk.set_stream(torch.cuda.current_stream().cuda_stream)
        m = mps.DistMPS(rk, args.n, args.chi) if args.world > 1 else mps.MPS(rk, args.n, args.chi)
        per_layer = []
        upd = 0
        for li, (singles, pairs) in enumerate(layers):
            tl = time.perf_counter()
            for q, g in enumerate(singles):
                m.apply_1q(q, mps.SINGLE_QUBIT[g])
            if args.sequential:
                for (q, _) in pairs:
                    m.apply_2q(q, circuits.FSIM)
            else:
                m.apply_layer(pairs, circuits.FSIM)
            upd += len(pairs)
            torch.cuda.synchronize()
            per_layer.append(time.perf_counter() - tl)
        rk.barrier()
        total = time.perf_counter() - t0
        logf[rk.rank()] = m.log_fidelity
        if args.world > 1:
            if rk.rank() == 0:
                out.update(total_s=total, per_layer_s=per_layer, updates=upd, world=args.world)
            m.free()
            return
        rng = np.random.default_rng(args.seed)
        bits = rng.integers(0, 2, size=(args.bitstrings, args.n))
        ta = time.perf_counter()
        amps = m.amplitudes(bits)
        if args.amps_out:
            np.save(args.amps_out, np.asarray(amps))
        out.update(total_s=total, per_layer_s=per_layer, updates=upd, bond_dims=m.bond_dims(),
                   fidelity=float(np.exp(m.log_fidelity)), amp_time_s=time.perf_counter() - ta,
                   amp_norm2_sum=float(np.sum(np.abs(amps) ** 2)), amp_first=[str(a) for a in amps[:4]])
        m.free()

    ngpu = max(1, torch.cuda.device_count())
    World(args.world, devices=[r % ngpu for r in range(args.world)]).run(body)
    if args.world > 1:
        out["fidelity"] = float(np.exp(sum(logf.values())))
        out["gpus"] = min(ngpu, args.world)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
