"""Tuning harness: time the DMMA zgemm variants (QTNH_ZGEMM_VARIANT) at the C1 and
C4 shapes with CUDA events, check numerics on a row block, compare to cuBLAS."""
import ctypes as C
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SHAPES = [(2**21, 128, 128), (2048, 2048, 1024), (4096, 4096, 4096), (2**20, 64, 64)]


def run_one():
    import numpy as np
    import torch

    from paper_2505_06119_b200 import qtnh

    w = qtnh.World(1)
    out = {}

    def body(rk):
        st = torch.cuda.Stream()
        rk.set_stream(st.cuda_stream)
        with torch.cuda.stream(st):
            for (m, n, k) in SHAPES:
                a = torch.randn(m, k, dtype=torch.complex128, device="cuda")
                b = torch.randn(k, n, dtype=torch.complex128, device="cuda")
                c = torch.empty(m, n, dtype=torch.complex128, device="cuda")
                args = (rk._h, m, n, k, C.c_void_p(a.data_ptr()), C.c_void_p(b.data_ptr()), C.c_void_p(c.data_ptr()))
                for _ in range(3):
                    qtnh.check(qtnh.lib.qtnh_zgemm_device(*args))
                reps = 10
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                for _ in range(reps):
                    qtnh.check(qtnh.lib.qtnh_zgemm_device(*args))
                e1.record(st)
                e1.synchronize()
                ms = e0.elapsed_time(e1) / reps
                ref = a[:256] @ b
                err = float((c[:256] - ref).abs().max() / ref.abs().max())
                # cuBLAS ceiling (sanity only)
                e0.record(st)
                for _ in range(reps):
                    torch.matmul(a, b, out=c)
                e1.record(st)
                e1.synchronize()
                ms_cublas = e0.elapsed_time(e1) / reps
                f = 8.0 * m * n * k
                out[f"{m}x{n}x{k}"] = {"ms": ms, "tflops": f / ms / 1e9, "cublas_tflops": f / ms_cublas / 1e9,
                                       "err": err}
                del a, b, c

    w.run(body)
    print(json.dumps(out))


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "one":
        run_one()
        sys.exit(0)
    variants = sys.argv[1:] or ["12", "106", "122"]
    for v in variants:
        env = dict(os.environ, QTNH_ZGEMM_VARIANT=v)
        r = subprocess.run([sys.executable, __file__, "one"], env=env, capture_output=True, text=True)
        print("variant", v, r.stdout.strip() or r.stderr[-2000:], flush=True)
