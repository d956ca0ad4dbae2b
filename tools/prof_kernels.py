"""Driver that launches every hot-path kernel on C1/C2-scale data, for ncu captures
(one kernel family per ncu run, see tools/ncu_all.sh): dense / diagonal gates,
QFT group / low / bit-reversal passes, strided copy (permute), Gauss zgemm (dense
and gathered), SVD round kernels, peer-memory swap and distributed QFT layers."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch

    from paper_2505_06119_b200 import circuits, qtnh
    from paper_2505_06119_b200.qtnh import DistParams, IndexTuple, Tensor, World, apply_gate, contract, ops

    def body(rk):
        rk.set_stream(torch.cuda.current_stream().cuda_stream)
        n = 28
        st = Tensor.dense(rk, IndexTuple([2] * n, 0), None, None)
        for _ in range(2):
            apply_gate(st, [13], circuits.H)
            apply_gate(st, [3, 20], circuits.FSIM)
            apply_gate(st, [5, 17], circuits.cp_diag(0.3), diagonal=True)
            qtnh.swap_indices(st, 2, 25)
        qtnh.qft(st, swaps=True)
        p = ops.permute(st, list(reversed(range(n))), 0)
        p.free()
        # C1-shaped contraction (gathered A) and a dense GEMM
        a = Tensor.dense(rk, IndexTuple([2] * 24, 0), None, None)
        b = Tensor.dense(rk, IndexTuple([2] * 14, 0), None, None)
        ap, bp = circuits.contraction_positions(7, 24, 14, 7)
        c = contract(a, b, ap, bp)
        c.free()
        a.free()
        b.free()
        st.free()
        x = torch.randn(1024, 1024, dtype=torch.complex128, device="cuda")
        u = torch.empty(1024, 512, dtype=torch.complex128, device="cuda")
        s = torch.empty(512, dtype=torch.float64, device="cuda")
        vh = torch.empty(512, 1024, dtype=torch.complex128, device="cuda")
        qtnh.check(qtnh.lib.qtnh_svd_device(rk._h, 1, 1024, 1024, C.c_void_p(x.data_ptr()), 512, 1,
                                            C.c_void_p(u.data_ptr()), C.c_void_p(s.data_ptr()),
                                            C.c_void_p(vh.data_ptr())))
        torch.cuda.synchronize()

    World(1).run(body)

    # peer-memory kernels: a 2^27 state sharded over 8 ranks sharing the GPU
    def body8(rk):
        t = Tensor.dense(rk, IndexTuple([2] * 27, 3), DistParams(1, 1, 0), None)
        qtnh.swap_indices(t, 0, 3)
        apply_gate(t, [1], circuits.H)
        qtnh.qft(t, swaps=True)
        rk.synchronize()
        t.free()

    World(8).run(body8)
    print("ok")


if __name__ == "__main__":
    main()
