"""Per-contraction profile of config 3 (5x6 depth-14 RCS network): each pairwise
contraction of the planned order timed with CUDA events (second pass, pool warm),
classified by arithmetic intensity; prints the totals and the top contractions."""
import json
import math
import os
import sys

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))


def main():
    import torch

    from paper_2505_06119_b200 import network
    from paper_2505_06119_b200.qtnh import World, check, lib

    check(lib.qtnh_set_option(b"pool_reserve_gb", float(os.environ.get("RESERVE_GB", "120"))))

    rows, cols, depth, seed, n_open = 5, 6, 14, 2025, 6
    res = {}

    def body(rk):
        rk.set_stream(torch.cuda.current_stream().cuda_stream)
        order = None
        for rep in range(2):
            net, *_ = network.build_rcs_network(rk, rows, cols, depth, seed, n_open)
            if order is None:
                order = network.Network.plan(net.labels, net.dims, seed, trials=int(os.environ.get("TRIALS", "2048")),
                                             max_log2_size=float(os.environ.get("CAP", "30")))
            nxt = max(net.tensors) + 1
            recs = []
            for s, (a, b) in enumerate(order):
                la, lb = net.labels[a], net.labels[b]
                sh = [x for x in la if x in lb]
                M = math.prod(net.dims[x] for x in la if x not in sh)
                N = math.prod(net.dims[x] for x in lb if x not in sh)
                K = math.prod(net.dims[x] for x in sh)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                geo = {"a_dims": net.tensors[a].shape().dims, "b_dims": net.tensors[b].shape().dims,
                       "apos": [la.index(x) for x in sh], "bpos": [lb.index(x) for x in sh]}
                e0.record()
                net.contract_pair(a, b, nxt + s)
                e1.record()
                recs.append((e0, e1, M, N, K, geo))
            torch.cuda.synchronize()
            res["recs"] = [(e0.elapsed_time(e1), M, N, K) for e0, e1, M, N, K, _ in recs]
            res["geo"] = [g for *_, g in recs]
            for t in list(net.tensors.values()):
                t.free()

    World(1).run(body)
    recs = res["recs"]
    tot = sum(r[0] for r in recs)
    out = {"total_ms": tot, "n": len(recs)}
    cats = {"compute(>=16 flop/B)": [0.0, 0.0, 0.0], "memory": [0.0, 0.0, 0.0]}
    for ms, M, N, K in recs:
        fl, by = 8.0 * M * N * K, 16.0 * (M * K + K * N + M * N)
        c = "compute(>=16 flop/B)" if fl / by >= 16 else "memory"
        cats[c][0] += ms
        cats[c][1] += fl
        cats[c][2] += by
    out["by_class"] = {k: {"ms": v[0], "TFLOPs": v[1] / max(v[0], 1e-9) / 1e9, "GBps": v[2] / max(v[0], 1e-9) / 1e6}
                       for k, v in cats.items()}
    idx = sorted(range(len(recs)), key=lambda i: -recs[i][0])[:12]
    out["top"] = []
    for i in idx:
        ms, M, N, K = recs[i]
        out["top"].append({"ms": ms, "M": M, "N": N, "K": K, "TFLOPs": 8.0 * M * N * K / ms / 1e9,
                           "GBps": 16.0 * (M * K + K * N + M * N) / ms / 1e6, **res["geo"][i]})
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
