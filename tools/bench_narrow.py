"""Tall-skinny contractions of config 3's flop-minimising order: dense zgemm against
the gathered contraction with the same (M, N, K), GB/s and TFLOP/s per shape."""
import ctypes as C, json, os, sys
sys.path.insert(0, os.environ.get('GRAFT_REPO_ROOT', os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2505_06119_b200 import qtnh
from paper_2505_06119_b200.qtnh import IndexTuple, Tensor, World, contract

SHAPES = [(25, 5, 5), (24, 4, 6), (23, 7, 5), (24, 6, 6), (23, 5, 5)]
if os.environ.get("NARROW_SHAPES"):  # e.g. NARROW_SHAPES=24x4x6 for one ncu capture
    SHAPES = [tuple(int(x) for x in t.split("x")) for t in os.environ["NARROW_SHAPES"].split(",")]

def body(rk):
    st = torch.cuda.Stream(); rk.set_stream(st.cuda_stream)
    with torch.cuda.stream(st):
        for lm, ln, lk in SHAPES:
            m, n, k = 2**lm, 2**ln, 2**lk
            a = torch.randn(m, k, dtype=torch.complex128, device="cuda")
            b = torch.randn(k, n, dtype=torch.complex128, device="cuda")
            c = torch.empty(m, n, dtype=torch.complex128, device="cuda")
            args = (rk._h, m, n, k, C.c_void_p(a.data_ptr()), C.c_void_p(b.data_ptr()), C.c_void_p(c.data_ptr()))
            def timeit(f, reps=5):
                for _ in range(2): f()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                for _ in range(reps): f()
                e1.record(st); e1.synchronize()
                return e0.elapsed_time(e1) / reps
            ms_d = timeit(lambda: qtnh.check(qtnh.lib.qtnh_zgemm_device(*args)))
            del c
            # gathered: A as a rank-(lm+lk) qubit tensor, contracted positions spread out
            ra = lm + lk
            ta = Tensor.from_device(rk, IndexTuple([2] * ra, 0), None, a.data_ptr()) if hasattr(Tensor, "from_device") else None
            tb = Tensor.from_device(rk, IndexTuple([2] * (lk + ln), 0), None, b.data_ptr())
            out = {}
            for name, ap in (("high", list(range(lk))), ("spread", [0, 1] + list(range(4, 4 + lk - 2))), ("low", list(range(ra - lk, ra)))):
                def f():
                    contract(ta, tb, ap, list(range(lk))).free()
                out[name] = timeit(f)
            by = 16.0 * (m * k + k * n + m * n)
            fl = 8.0 * m * n * k
            print(json.dumps({"M": lm, "N": ln, "K": lk, "dense_ms": ms_d, "dense_GBps": by / ms_d / 1e6, "dense_TF": fl / ms_d / 1e9,
                              **{f"gather_{k2}_ms": v for k2, v in out.items()},
                              **{f"gather_{k2}_GBps": by / v / 1e6 for k2, v in out.items()}}), flush=True)
            ta.free(); tb.free(); del a, b
World(1).run(body)
