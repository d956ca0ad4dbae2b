"""Config 3: 5x6 grid random circuit, depth 14, as a tensor network contracted on
one GPU along the seeded greedy order down to the 64 amplitudes of 6 open qubits
(24 output bits fixed by seed). Reports the order's sum of 8MNK flops and bytes,
the contraction time, and the check against a 30-qubit statevector run of the
same circuit on the GPU."""
import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=5)
    ap.add_argument("--cols", type=int, default=6)
    ap.add_argument("--depth", type=int, default=14)
    ap.add_argument("--open", type=int, default=6)
    ap.add_argument("--seed", type=int, default=2025)
    ap.add_argument("--no-statevector", action="store_true")
    ap.add_argument("--trials", type=int, default=2048)
    ap.add_argument("--cap", type=float, default=30.0,
                    help="memory budget of the order search: log2 of the largest intermediate (elements); 0 = smallest peak first")
    ap.add_argument("--world", type=int, default=1,
                    help="ranks (thread per rank over the visible GPUs): tensors replicated, contractions of "
                         ">= --shard-flops M-sharded")
    ap.add_argument("--shard-flops", type=float, default=1e11)
    ap.add_argument("--reserve-gb", type=float, default=120,
                    help="map this much of the stream-ordered pool up front (option pool_reserve_gb)")
    args = ap.parse_args()
    import numpy as np
    import torch

    from paper_2505_06119_b200 import circuits, mps, network
    from paper_2505_06119_b200.qtnh import IndexTuple, Tensor, World, apply_gate
    from paper_2505_06119_b200 import qtnh as _q

    _q.check(_q.lib.qtnh_set_option(b"pool_reserve_gb", float(args.reserve_gb)))

    out = {"rows": args.rows, "cols": args.cols, "depth": args.depth, "open": args.open}

    import threading

    planned = threading.Event()
    shared = {}

    def body(rk):
        rk.set_stream(torch.cuda.current_stream().cuda_stream)
        net, open_labels, open_q, fixed = network.build_rcs_network(rk, args.rows, args.cols, args.depth,
                                                                    args.seed, args.open, args.shard_flops)
        if rk.rank() == 0:  # the order is host-only and identical on every rank: plan once
            out["n_tensors"] = len(net.tensors)
            t0 = time.perf_counter()
            shared["order"] = network.Network.plan(net.labels, net.dims, args.seed, trials=args.trials, max_log2_size=args.cap)
            out["plan_s"] = time.perf_counter() - t0
            planned.set()
        planned.wait()
        order = shared["order"]
        if rk.rank() != 0:
            last = net.contract_order(order)
            net.tensors[last].to_global_vector()  # collective when the result is sharded
            net.tensors[last].free()
            return
        # cost of the order (SURVEY.md 8(d) C3 convention)
        labels = {k: list(v) for k, v in net.labels.items()}
        nxt = max(labels) + 1
        flops = 0.0
        byts = 0.0
        biggest = 0
        for s, (a, b) in enumerate(order):
            la, lb = labels.pop(a), labels.pop(b)
            sh = [x for x in la if x in lb]
            M = math.prod(net.dims[x] for x in la if x not in sh)
            N = math.prod(net.dims[x] for x in lb if x not in sh)
            K = math.prod(net.dims[x] for x in sh)
            flops += 8.0 * M * N * K
            byts += 16.0 * (M * K + K * N + M * N)
            biggest = max(biggest, M * N)
            labels[nxt + s] = [x for x in la if x not in sh] + [x for x in lb if x not in sh]
        out.update(order_len=len(order), order_flops=flops, order_bytes=byts, largest_intermediate=biggest)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        last = net.contract_order_native(order) if args.world == 1 else net.contract_order(order)
        e1.record()
        e1.synchronize()
        out["world"] = args.world
        out["executor"] = "native chain (qtnh_contract_chain)" if args.world == 1 else "python loop"
        out["sharded_contractions"] = net.n_sharded
        out["contract_s_wall"] = time.perf_counter() - t0
        out["contract_s_device"] = e0.elapsed_time(e1) / 1e3
        out["achieved_TFLOPs"] = flops / out["contract_s_device"] / 1e12
        res_labels = net.labels[last]
        amp = net.tensors[last].to_global_vector().reshape([2] * len(res_labels))
        amp = np.transpose(amp, [res_labels.index(l) for l in open_labels]).reshape(-1)
        net.tensors[last].free()
        out["amp_norm2"] = float(np.sum(np.abs(amp) ** 2))
        if not args.no_statevector and args.world == 1:
            n = args.rows * args.cols
            st = Tensor.dense(rk, IndexTuple([2] * n, 0), None, None)
            one = torch.zeros(1, dtype=torch.complex128)
            one[0] = 1
            # |0...0>: write amplitude 0
            import ctypes as C
            torch.cuda.synchronize()
            v = torch.as_tensor(mps._DevView(st.device_ptr(), 2**n), device="cuda")
            v[0] = 1.0
            t1 = time.perf_counter()
            for kind, qs, g in network.rcs_grid_circuit(args.rows, args.cols, args.depth, args.seed):
                apply_gate(st, list(qs), mps.SINGLE_QUBIT[g] if kind == "1q" else circuits.FSIM)
            torch.cuda.synchronize()
            out["statevector_s"] = time.perf_counter() - t1
            psi = v.reshape([2] * n)
            idx = tuple(slice(None) if q in open_q else fixed[q] for q in range(n))
            want = psi[idx].reshape(-1).cpu().numpy()
            out["rel_l2_vs_statevector"] = float(np.linalg.norm(amp - want) / np.linalg.norm(want))
            st.free()

    ngpu = max(1, torch.cuda.device_count())
    World(args.world, devices=[r % ngpu for r in range(args.world)]).run(body)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
