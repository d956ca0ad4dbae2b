"""Why does the batch-8 2048^2 SVD take 192 ms per matrix inside bench.py and 97 ms in
tools/bench_svd.py? Times the same call between the stages bench.py goes through."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import bench
from paper_2505_06119_b200 import circuits, qtnh
from paper_2505_06119_b200.qtnh import DistParams, IndexTuple, Tensor, World, apply_gate, contract

lib = qtnh.lib
stream = torch.cuda.Stream()


def svd8(rk, tag):
    nn, chi, bt = 2048, 1024, 8
    rng = np.random.default_rng(0)
    a = torch.from_numpy(rng.standard_normal((bt, nn, nn)) + 1j * rng.standard_normal((bt, nn, nn))).cuda()
    u = torch.empty((bt, nn, chi), dtype=torch.complex128, device="cuda")
    s = torch.empty((bt, chi), dtype=torch.float64, device="cuda")
    vh = torch.empty((bt, chi, nn), dtype=torch.complex128, device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    qtnh.check(lib.qtnh_svd_device(rk._h, bt, nn, nn, C.c_void_p(a.data_ptr()), chi, 1, C.c_void_p(u.data_ptr()),
                                   C.c_void_p(s.data_ptr()), C.c_void_p(vh.data_ptr())))
    e1.record(stream)
    e1.synchronize()
    print(f"{tag}: {e0.elapsed_time(e1) / bt:.1f} ms per SVD, sweeps {int(lib.qtnh_last_error_info())}", flush=True)


def body(rk):
    rk.set_stream(stream.cuda_stream)
    with torch.cuda.stream(stream):
        svd8(rk, "fresh")
        RA, RB, K = bench.RANK_A, bench.RANK_B, bench.K_SHARED
        a_host = torch.empty(2**RA, dtype=torch.complex128).pin_memory()
        lib.qtnh_counter_complex_normals(1, 0, 2**RA, a_host.numpy().ctypes.data, 16)
        b_host = torch.from_numpy(circuits.counter_state(2, 2**RB)).pin_memory()
        c_host = torch.empty(2**RA, dtype=torch.complex128).pin_memory()
        svd8(rk, "after pinning 8.6 GB")
        ta = Tensor.dense(rk, IndexTuple([2] * RA, 0), DistParams(1, 1, 0), None)
        tb = Tensor.dense(rk, IndexTuple([2] * RB, 0), DistParams(1, 1, 0), None)
        qtnh.check(lib.qtnh_tensor_upload_local(ta._h, C.c_void_p(a_host.data_ptr())))
        qtnh.check(lib.qtnh_tensor_upload_local(tb._h, C.c_void_p(b_host.data_ptr())))
        ap, bp = circuits.contraction_positions(bench.SEED, RA, RB, K)
        for _ in range(5):
            contract(ta, tb, ap, bp).free()
        rk.synchronize()
        svd8(rk, "after 5 resident contractions")
        dims_a = (C.c_int64 * RA)(*([2] * RA))
        dims_b = (C.c_int64 * RB)(*([2] * RB))
        ap_c, bp_c = (C.c_int * K)(*ap), (C.c_int * K)(*bp)
        qtnh.check(lib.qtnh_contract_host(rk._h, RA, dims_a, C.c_void_p(a_host.data_ptr()), RB, dims_b,
                                          C.c_void_p(b_host.data_ptr()), K, ap_c, bp_c,
                                          C.c_void_p(c_host.data_ptr()), None))
        rk.synchronize()
        svd8(rk, "after contract_host")
        ta.free()
        tb.free()
        st = Tensor.dense(rk, IndexTuple([2] * 30, 0), None, None)
        for _ in range(4):
            apply_gate(st, [15], circuits.H)
        rk.synchronize()
        st.free()
        svd8(rk, "after 2^30 gates")
        nn, chi = 2048, 1024
        a = torch.randn(nn, nn, dtype=torch.complex128, device="cuda")
        u = torch.empty((nn, chi), dtype=torch.complex128, device="cuda")
        s = torch.empty((chi,), dtype=torch.float64, device="cuda")
        vh = torch.empty((chi, nn), dtype=torch.complex128, device="cuda")
        qtnh.check(lib.qtnh_svd_device(rk._h, 1, nn, nn, C.c_void_p(a.data_ptr()), chi, 1, C.c_void_p(u.data_ptr()),
                                       C.c_void_p(s.data_ptr()), C.c_void_p(vh.data_ptr())))
        svd8(rk, "after a batch-1 SVD")


World(1, [0]).run(body)
