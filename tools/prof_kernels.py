"""Small driver that launches each secondary hot-path kernel a few times, for ncu
captures (gate application, fused QFT group pass, SVD round kernels, remap)."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch

    from paper_2505_06119_b200 import circuits, qtnh
    from paper_2505_06119_b200.qtnh import IndexTuple, Tensor, World, apply_gate, ops

    def body(rk):
        rk.set_stream(torch.cuda.current_stream().cuda_stream)
        n = 28
        st = Tensor.dense(rk, IndexTuple([2] * n, 0), None, None)
        for _ in range(3):
            apply_gate(st, [13], circuits.H)
            apply_gate(st, [3, 20], circuits.FSIM)
        qtnh.qft(st, swaps=True)
        p = ops.permute(st, list(reversed(range(n))), 0)
        p.free()
        st.free()
        a = torch.randn(1024, 1024, dtype=torch.complex128, device="cuda")
        u = torch.empty(1024, 512, dtype=torch.complex128, device="cuda")
        s = torch.empty(512, dtype=torch.float64, device="cuda")
        vh = torch.empty(512, 1024, dtype=torch.complex128, device="cuda")
        qtnh.check(qtnh.lib.qtnh_svd_device(rk._h, 1, 1024, 1024, C.c_void_p(a.data_ptr()), 512, 1,
                                            C.c_void_p(u.data_ptr()), C.c_void_p(s.data_ptr()),
                                            C.c_void_p(vh.data_ptr())))
        torch.cuda.synchronize()

    World(1).run(body)
    print("ok")


if __name__ == "__main__":
    main()
