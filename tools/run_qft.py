"""Config 2 on one GPU: QFT on a 33-qubit statevector (2^33 complex128 = 128 GiB,
in place), seeded counter-based normalised random input generated on the device.

Reports (CUDA events on the rank stream):
  * per-gate times of the gate-by-gate path (dense H, diagonal CP, in-place SWAP)
    on the full state and the HBM fraction at 32 B/amplitude per gate;
  * the whole QFT through the fused-layer path (one pass per layer + swaps);
  * correctness at full size: norm preservation and spot amplitudes against a
    direct O(2^n) DFT sum over the input (chunked, computed before the QFT).
"""
import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


class DevView:
    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<c16", "data": (ptr, False), "version": 3}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=33)
    ap.add_argument("--seed", type=int, default=2025)
    ap.add_argument("--spots", type=int, default=4)
    args = ap.parse_args()
    import ctypes as C

    import numpy as np
    import torch

    from paper_2505_06119_b200 import circuits, qtnh
    from paper_2505_06119_b200.qtnh import IndexTuple, Tensor, apply_gate

    n = args.n
    N = 2**n
    out = {"n": n, "bytes_state": 16 * N}
    peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0

    def body(rk):
        st = torch.cuda.Stream()
        rk.set_stream(st.cuda_stream)
        with torch.cuda.stream(st):
            t = Tensor.dense(rk, IndexTuple([2] * n, 0), None, None)
            psi = torch.as_tensor(DevView(t.device_ptr(), N), device="cuda")
            qtnh.check(qtnh.lib.qtnh_counter_complex_normals_device(C.c_void_p(st.cuda_stream), args.seed, 0, N,
                                                                    C.c_void_p(t.device_ptr())))
            chunk = 2**27
            nrm2 = 0.0
            for c0 in range(0, N, chunk):
                nrm2 += float(psi[c0:c0 + chunk].abs().pow(2).sum())
            psi.mul_(1.0 / math.sqrt(nrm2))
            # spot amplitudes y_k = sum_j x_j exp(2 pi i j k / N) / sqrt(N)
            rng = np.random.default_rng(args.seed)
            ks = [0, 1, N - 1] + [int(x) for x in rng.integers(2, N - 1, size=max(0, args.spots - 3))]
            want = {}
            for k in ks:
                acc = torch.zeros((), dtype=torch.complex128, device="cuda")
                for c0 in range(0, N, chunk):
                    j = torch.arange(c0, c0 + chunk, dtype=torch.int64, device="cuda")
                    ph = torch.remainder(j * k, N).to(torch.float64) * (2 * math.pi / N)
                    acc += (psi[c0:c0 + chunk] * torch.polar(torch.ones_like(ph), ph)).sum()
                want[k] = complex(acc.item()) / math.sqrt(N)
            torch.cuda.synchronize()

            def timed(fn, reps=3):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                for _ in range(reps):
                    fn()
                e1.record(st)
                e1.synchronize()
                return e0.elapsed_time(e1) / reps

            # per-gate timings on the full state (gate-by-gate path); each op is
            # applied an even number of times so the state is unchanged afterwards
            gates = {}
            H = circuits.H
            gates["H_dense_q0"] = timed(lambda: apply_gate(t, [0], H), 2)
            gates["H_dense_q16"] = timed(lambda: apply_gate(t, [16], H), 2)
            gates["H_dense_q32"] = timed(lambda: apply_gate(t, [n - 1], H), 2)
            ph = circuits.cp_diag(0.25)
            phc = np.conj(ph)
            gates["CP_diag_q3_q20"] = (timed(lambda: apply_gate(t, [3, 20], ph, diagonal=True), 1)
                                       + timed(lambda: apply_gate(t, [3, 20], phc, diagonal=True), 1)) / 2
            gates["SWAP_inplace_q2_qn-3"] = timed(lambda: qtnh.swap_indices(t, 2, n - 3), 2)
            gates["qft_layer_fused_q5"] = timed(lambda: qtnh.qft_layer(t, 5), 1)
            torch.cuda.synchronize()
            # undo the single fused layer by re-initialising (layer is not an involution)
            qtnh.check(qtnh.lib.qtnh_counter_complex_normals_device(C.c_void_p(st.cuda_stream), args.seed, 0, N,
                                                                    C.c_void_p(t.device_ptr())))
            psi.mul_(1.0 / math.sqrt(nrm2))
            per = {}
            for k, ms in gates.items():
                gbs = 32.0 * N / (ms * 1e-3) / 1e9
                per[k] = {"ms": ms, "GBps_algorithmic": gbs, "frac_of_hbm": gbs / peak}
            out["per_gate"] = per
            n_h, n_cp, n_sw = n, n * (n - 1) // 2, n // 2
            out["gate_by_gate_estimate_s"] = (n_h * gates["H_dense_q16"] + n_cp * gates["CP_diag_q3_q20"]
                                              + n_sw * gates["SWAP_inplace_q2_qn-3"]) / 1e3
            out["gate_counts"] = {"H": n_h, "CP": n_cp, "SWAP": n_sw, "total": n_h + n_cp + n_sw}
            # the full QFT, cache-blocked path (qtnh_qft)
            torch.cuda.synchronize()
            e0b, e1b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0b.record(st)
            qtnh.qft(t, swaps=True)
            e1b.record(st)
            e1b.synchronize()
            msb = e0b.elapsed_time(e1b)
            out["qft_blocked_s"] = msb / 1e3
            out["qft_blocked_effective_GBps"] = (n_h + n_cp + n_sw) * 32.0 * N / (msb * 1e-3) / 1e9
            errs_b = {}
            for k, w in want.items():
                g = complex(psi[k].item())
                errs_b[str(k)] = abs(g - w) / max(abs(w), 1e-300)
            out["blocked_spot_rel_err"] = errs_b
            # restore the input for the layer-by-layer run
            qtnh.check(qtnh.lib.qtnh_counter_complex_normals_device(C.c_void_p(st.cuda_stream), args.seed, 0, N,
                                                                    C.c_void_p(t.device_ptr())))
            psi.mul_(1.0 / math.sqrt(nrm2))
            # the full QFT, fused layer-by-layer path
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            circuits.apply_qft_fused(t, n)
            e1.record(st)
            e1.synchronize()
            ms = e0.elapsed_time(e1)
            out["qft_fused_s"] = ms / 1e3
            out["qft_fused_effective_GBps"] = (n_h + n_cp + n_sw) * 32.0 * N / (ms * 1e-3) / 1e9
            out["qft_fused_passes"] = n + n // 2
            out["qft_fused_pass_GBps"] = (n * 32.0 * N + n_sw * 16.0 * N) / (ms * 1e-3) / 1e9
            nrm_after = 0.0
            for c0 in range(0, N, chunk):
                nrm_after += float(psi[c0:c0 + chunk].abs().pow(2).sum())
            out["norm_after"] = math.sqrt(nrm_after)
            errs = {}
            for k, w in want.items():
                g = complex(psi[k].item())
                errs[str(k)] = abs(g - w) / max(abs(w), 1e-300)
            out["spot_rel_err"] = errs
            out["spot_max_abs_err"] = max(abs(complex(psi[k].item()) - w) for k, w in want.items())
            t.free()

    qtnh.World(1).run(body)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
