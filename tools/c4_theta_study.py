"""Config 4 SVD study on a REAL saturated theta (2048 x 2048, chi = 1024): evolves
the 40-site MPS to its first saturated layer, takes the first saturated pair's
theta (contract + fSim, on the host from the captured sites), and reports
  * its spectrum around the cut (sigma_1, sigma_chi, sigma_chi+1, sigma_n, cluster
    widths) from numpy's LAPACK SVD;
  * our Jacobi SVD's sweeps and time on it (single and as a batch of 8 copies);
  * how many Newton-Schulz sign iterations a spectral-projector split at the cut
    would need (the eigenvalues of H = theta theta^H shifted by a mid-gap mu).

  python tools/c4_theta_study.py [--out theta.npy]
"""
import argparse
import ctypes as C
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="")
    ap.add_argument("--layer", type=int, default=-1, help="capture at this layer (default: first saturated)")
    ap.add_argument("--pairs", type=int, default=1, help="saturated pairs to analyse (spectra only after the first)")
    args = ap.parse_args()
    import numpy as np
    import torch

    import bench_legs
    from paper_2505_06119_b200 import circuits, qtnh
    from paper_2505_06119_b200.qtnh import World

    res = {}

    def body(rk):
        st = torch.cuda.Stream()
        rk.set_stream(st.cuda_stream)
        with torch.cuda.stream(st):
            _, cap = bench_legs.gpu_c4(rk, st, torch, depth=(args.layer + 1 if args.layer >= 0 else 12),
                                       capture=args.pairs, bitstrings=4,
                                       capture_layer=(args.layer if args.layer >= 0 else None))
        chi = 1024
        spectra = []
        for c in cap:
            a = c["a"].reshape(chi * 2, chi)
            b = c["b"].reshape(chi, 2 * chi)
            th = (a @ b).reshape(chi, 2, 2, chi)
            th = np.einsum("ijkl,aklb->aijb", circuits.FSIM.reshape(2, 2, 2, 2), th).reshape(2 * chi, 2 * chi)
            sv = np.linalg.svd(th, compute_uv=False)
            vals, counts = [], []
            for x in sv:
                if vals and abs(x - vals[-1]) <= 1e-9 * sv[0]:
                    counts[-1] += 1
                else:
                    vals.append(float(x))
                    counts.append(1)
            spectra.append({"site": c["q"], "clusters": len(vals), "values": vals[:12], "multiplicities": counts[:12],
                            "sigma_chi": float(sv[chi - 1]), "sigma_chi+1": float(sv[chi])})
        res["spectra"] = spectra
        c = cap[0]
        a = c["a"].reshape(chi * 2, chi)
        b = c["b"].reshape(chi, 2 * chi)
        th = (a @ b).reshape(chi, 2, 2, chi)
        th = np.einsum("ijkl,aklb->aijb", circuits.FSIM.reshape(2, 2, 2, 2), th).reshape(2 * chi, 2 * chi)
        if args.out:
            np.save(args.out, th)
        t0 = time.time()
        s = np.linalg.svd(th, compute_uv=False)
        res["numpy_svd_s"] = time.time() - t0
        res["sigma"] = {"1": s[0], "chi": s[chi - 1], "chi+1": s[chi], "n": s[-1]}
        res["top_cluster_rel_width"] = float((s[0] - s[chi - 1]) / s[0])
        res["bottom_cluster_rel_width"] = float((s[chi] - s[-1]) / s[chi]) if s[chi] > 0 else None
        res["gap_ratio_chi"] = float(s[chi] / s[chi - 1])
        res["kept_weight"] = float(np.sum(s[:chi] ** 2) / np.sum(s**2))
        res["distinct_top_1e-12"] = int(np.sum(np.abs(np.diff(s[:chi])) > 1e-12 * s[0]))
        hist, edges = np.histogram(s, bins=16)
        res["hist"] = [int(x) for x in hist]
        res["hist_edges"] = [float(x) for x in edges]
        # sign-iteration count for the projector at the cut: eigenvalues of H - mu
        lam = s**2
        mu = 0.5 * (lam[chi - 1] + lam[chi])
        x = (lam - mu) / np.max(np.abs(lam - mu))
        it = 0
        while np.max(np.abs(np.abs(x) - 1)) > 1e-14 and it < 100:
            x = 1.5 * x - 0.5 * x**3
            it += 1
        res["newton_schulz_iterations"] = it
        # our SVD on it
        dev = torch.from_numpy(th).cuda()
        for bt in (1, 8):
            A = dev.unsqueeze(0).repeat(bt, 1, 1).contiguous()
            U = torch.empty((bt, 2 * chi, chi), dtype=torch.complex128, device="cuda")
            S = torch.empty((bt, chi), dtype=torch.float64, device="cuda")
            V = torch.empty((bt, chi, 2 * chi), dtype=torch.complex128, device="cuda")
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            qtnh.check(qtnh.lib.qtnh_svd_device(rk._h, bt, 2 * chi, 2 * chi, C.c_void_p(A.data_ptr()), chi, 1,
                                                C.c_void_p(U.data_ptr()), C.c_void_p(S.data_ptr()),
                                                C.c_void_p(V.data_ptr())))
            e1.record(st)
            e1.synchronize()
            res[f"ours_batch{bt}"] = {"ms_per_svd": e0.elapsed_time(e1) / bt,
                                      "sweeps": int(qtnh.lib.qtnh_last_error_info()),
                                      "s_rel_err": float(np.max(np.abs(S[0].cpu().numpy() - s[:chi])) / s[0])}

        # cuSOLVER via torch (sanity ceiling only; not the hot path): full SVD of the
        # theta and of a random 2048^2 matrix, and the Hermitian eigensolver on A A^H
        rnd = torch.randn(2 * chi, 2 * chi, dtype=torch.complex128, device="cuda")
        for name, mat in (("theta", dev), ("random", rnd)):
            for drv in ("gesvd", "gesvdj", "gesvda", None):
                try:
                    torch.linalg.svd(mat, full_matrices=False, driver=drv)
                    torch.cuda.synchronize()
                    t0 = time.time()
                    torch.linalg.svd(mat, full_matrices=False, driver=drv)
                    torch.cuda.synchronize()
                    res[f"cusolver_svd_{drv}_{name}_ms"] = 1e3 * (time.time() - t0)
                except Exception as e:  # noqa: BLE001
                    res[f"cusolver_svd_{drv}_{name}_ms"] = f"n/a: {type(e).__name__}"
            hm = mat @ mat.conj().T
            torch.linalg.eigh(hm)
            torch.cuda.synchronize()
            t0 = time.time()
            torch.linalg.eigh(hm)
            torch.cuda.synchronize()
            res[f"cusolver_eigh_{name}_ms"] = 1e3 * (time.time() - t0)
        res["split_count"] = int(qtnh.lib.qtnh_svd_split_count())

    World(1).run(body)
    print(json.dumps(res, default=float))


if __name__ == "__main__":
    main()
