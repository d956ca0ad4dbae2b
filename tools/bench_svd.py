"""Time the batched Jacobi SVD at the config-4 shape (theta 2048 x 2048 -> chi 1024)
and smaller ones, with CUDA events; report sweeps and the convention TFLOP/s
(88 n^3 real flops per n x n complex SVD)."""
import ctypes as C
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main(shapes):
    import numpy as np
    import torch

    from paper_2505_06119_b200 import qtnh

    out = []

    def body(rk):
        st = torch.cuda.Stream()
        rk.set_stream(st.cuda_stream)
        with torch.cuda.stream(st):
            for batch, n, chi in shapes:
                rng = np.random.default_rng(0)
                a = torch.from_numpy(rng.standard_normal((batch, n, n)) + 1j * rng.standard_normal((batch, n, n))).cuda()
                if os.environ.get("BENCH_SVD_SPECTRUM") == "two":
                    # config 4's early saturated thetas: two singular values, chi-fold each
                    # (input generation only: torch QR of the random matrices)
                    q1 = torch.linalg.qr(a)[0]
                    q2 = torch.linalg.qr(a.transpose(1, 2).conj().contiguous())[0]
                    sv = torch.tensor([0.70719] * chi + [0.35957] * (n - chi), dtype=torch.float64, device="cuda")
                    a = (q1 * sv) @ q2.transpose(1, 2).conj()
                    a = a.contiguous()
                u = torch.empty((batch, n, chi), dtype=torch.complex128, device="cuda")
                s = torch.empty((batch, chi), dtype=torch.float64, device="cuda")
                vh = torch.empty((batch, chi, n), dtype=torch.complex128, device="cuda")
                args = (rk._h, batch, n, n, C.c_void_p(a.data_ptr()), chi, 1, C.c_void_p(u.data_ptr()),
                        C.c_void_p(s.data_ptr()), C.c_void_p(vh.data_ptr()))
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                qtnh.check(qtnh.lib.qtnh_svd_device(*args))
                e1.record(st)
                e1.synchronize()
                sweeps = int(qtnh.lib.qtnh_last_error_info())
                ms = e0.elapsed_time(e1)
                # accuracy on matrix 0: truncated reconstruction vs numpy
                a0 = a[0].cpu().numpy()
                U, S, VH = np.linalg.svd(a0, full_matrices=False)
                want = (U[:, :chi] * S[:chi]) @ VH[:chi]
                got = u[0].cpu().numpy() @ vh[0].cpu().numpy()
                err = float(np.linalg.norm(got - want) / np.linalg.norm(want))
                flops = batch * 88.0 * n**3
                out.append({"batch": batch, "n": n, "chi": chi, "ms": ms, "ms_per_svd": ms / batch,
                            "sweeps": sweeps, "conv_tflops": flops / ms / 1e9, "rel_err": err})
                print(json.dumps(out[-1]), flush=True)

    qtnh.World(1).run(body)


if __name__ == "__main__":
    shapes = [(1, 256, 128), (1, 1024, 512), (1, 2048, 1024), (4, 1024, 512)]
    if len(sys.argv) > 1:
        shapes = [tuple(int(x) for x in s.split("x")) for s in sys.argv[1:]]
    main(shapes)
