"""Benchmark of the QTNH hot path on B200 (config 1 of BASELINE.json).

Workload (BASELINE.json configs[1]): pairwise dense complex128 contraction of a
rank-28 tensor A with a rank-14 tensor B, all index dims 2, 7 shared indices at
seeded random positions of both operands (so both need a permutation), result
rank 28 in the SPEC.md:408 order. One step = qtnh contract(A, B): the layout
permutation of A and B (strided-copy kernels) + the complex128 GEMM on the FP64
tensor cores (M = 2^21, N = 2^7, K = 2^7; 8MNK = 2.749e11 flop).

Multi-GPU (torchrun, one process per GPU): A gets log2(N) extra leading open
indices that are distributed (M-sharding); every rank holds a
2^28 shard and the replicated B, so per-GPU work is fixed ("weak") and the step
has no data-path collective.

JSON line: value = whole-job FP64 TFLOP/s with operands resident in HBM; e2e =
the same metric through the public API with host buffers (pinned H2D of A and B
and D2H of the result inside the timed region); roofline for the dominant kernel
(zgemm) against the FP64 DMMA peak measured live on this device; cpu_baseline =
the unmodified reference (oracle/_ref: t2m -> SUMMA zgemm -> m2t, OpenBLAS) on a
bounded rank-22 sample on the host cores.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

RANK_A, RANK_B, K_SHARED, SEED = 28, 14, 7, 2025
METRIC = "contraction FP64 TFLOP/s (complex128, rank-28 x rank-14, 7 shared indices)"
UNIT = "TFLOP/s"


def flops_for(rank_a: int) -> float:
    m = 2 ** (rank_a - K_SHARED)
    return 8.0 * m * 2 ** (RANK_B - K_SHARED) * 2**K_SHARED


# ---- clocks sampling (B200_PROFILING.md) ------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ---- C1 workload description shared by both arms ----------------------------------------------
def fisher_yates(hash_fn, seed: int, tag: int, r: int):
    """Seeded Fisher-Yates on hash_counter(seed, tag, i) (test_ops.cpp:124-129)."""
    p = list(range(r))
    for i in range(r - 1, 0, -1):
        j = hash_fn(seed, tag, i) % (i + 1)
        p[i], p[j] = p[j], p[i]
    return p


def c1_positions(hash_fn, rank_a: int = RANK_A):
    """The 7 contracted positions of A and of B, paired in sorted order."""
    ap = sorted(fisher_yates(hash_fn, SEED, 8, rank_a)[:K_SHARED])
    bp = sorted(fisher_yates(hash_fn, SEED + 1, 8, RANK_B)[:K_SHARED])
    return ap, bp


class C1Sample:
    """A bounded sample of the SAME rank-28 contraction for the CPU arms: fixing the
    first FIXED open indices of A to a block value b cuts A into 2^FIXED rank-22
    slices; contracting slice b with B (7 shared indices, the same positions) gives
    exactly rows [b*2^22, (b+1)*2^22) of the rank-28 result (those indices lead the
    SPEC.md:408 result order). The slice values are the rank-28 A's own elements
    (the counter-based generator evaluated at their global indices), so the
    reference's output for a slice is also a parity check of the GPU's rank-28
    result on those rows."""

    FIXED = 6

    def __init__(self, port, shard: int = 0):
        import numpy as np

        self.np, self.P, self.shard = np, port, shard
        self.ap, self.bp = c1_positions(port.hash_counter)
        open_a = [i for i in range(RANK_A) if i not in self.ap]
        self.fixed = open_a[: self.FIXED]
        self.rest = [i for i in range(RANK_A) if i not in self.fixed]
        self.rank_s = RANK_A - self.FIXED
        self.ap_s = [self.rest.index(p) for p in self.ap]
        j = np.arange(2**self.rank_s, dtype=np.int64)
        base = np.zeros_like(j)
        for t, pos in enumerate(self.rest):
            base |= ((j >> (self.rank_s - 1 - t)) & 1) << (RANK_A - 1 - pos)
        self.base = base + shard * 2**RANK_A
        self.b = port.counter_normals(SEED + 1, 0, 2**RANK_B)

    def a_slice(self, block: int):
        off = 0
        for t, pos in enumerate(self.fixed):
            off |= ((block >> (self.FIXED - 1 - t)) & 1) << (RANK_A - 1 - pos)
        return self.P.counter_normals_at(SEED, self.base + off)

    @staticmethod
    def rows(block: int):
        n = 2 ** (RANK_A - C1Sample.FIXED)
        return slice(block * n, (block + 1) * n)

    def flops(self) -> float:
        return flops_for(RANK_A) / 2**self.FIXED


def c1_brute_force(port, outputs, shard: int = 0):
    """Host brute force of selected rank-28 result elements straight from the
    definition C[o] = sum_k A[a(o, k)] B[b(o, k)], with A and B
    evaluated by the oracle port's counter-based generator at the needed indices."""
    import numpy as np

    ap, bp = c1_positions(port.hash_counter)
    open_a = [i for i in range(RANK_A) if i not in ap]
    open_b = [i for i in range(RANK_B) if i not in bp]
    o = np.asarray(outputs, dtype=np.int64)[:, None]
    k = np.arange(2**K_SHARED, dtype=np.int64)[None, :]
    ia = np.zeros((o.shape[0], k.shape[1]), np.int64)
    ib = np.zeros_like(ia)
    n_out = len(open_a) + len(open_b)
    for t, pos in enumerate(open_a):
        ia |= ((o >> (n_out - 1 - t)) & 1) << (RANK_A - 1 - pos)
    for t, pos in enumerate(open_b):
        ib |= ((o >> (n_out - 1 - len(open_a) - t)) & 1) << (RANK_B - 1 - pos)
    for t in range(K_SHARED):
        bit = (k >> (K_SHARED - 1 - t)) & 1
        ia |= bit << (RANK_A - 1 - ap[t])
        ib |= bit << (RANK_B - 1 - bp[t])
    av = port.counter_normals_at(SEED, (ia + shard * 2**RANK_A).reshape(-1)).reshape(ia.shape)
    bv = port.counter_normals_at(SEED + 1, ib.reshape(-1)).reshape(ib.shape)
    return (av * bv).sum(axis=1)


def cpu_reference_c1(budget_s: float = 15.0, blocks=None, keep_outputs: bool = False):
    """The unmodified reference (oracle/_ref: t2m -> SUMMA cblas_zgemm -> m2t,
    linalg.hpp:208-400, OpenBLAS on all host threads, World(1)) on 1/64 slices of the
    rank-28 contraction (C1Sample), best of the calls made within the budget.
    Returns (TFLOP/s, cores, sample, kind, {block: result rows})."""
    import oracle

    cores = os.cpu_count() or 1
    P = oracle.port()
    smp = C1Sample(P)
    if not oracle.ref_available():
        raise RuntimeError("oracle/_ref/libqtnh_ref.so missing (built by __graft_entry__.build())")
    R = oracle.ref()
    R.set_threads(cores)
    blocks = list(blocks) if blocks is not None else list(range(2**C1Sample.FIXED))
    times, outs = [], {}
    t_start = time.perf_counter()
    for i, blk in enumerate(blocks):
        a = smp.a_slice(blk)
        c, _, _, t = R.contract(1, [2] * smp.rank_s, 0, (1, 1, 0), a, [2] * RANK_B, 0, (1, 1, 0), smp.b,
                                smp.ap_s, smp.bp, timing=True)
        times.append(t[3] / 1e3)
        if keep_outputs:
            outs[blk] = c
        if time.perf_counter() - t_start > budget_s:
            break
    best = min(times)
    sample = (f"{len(times)} of the 64 rank-22 slices of the rank-28 A (first 6 open indices of A fixed; "
              f"each slice x the full B = 1/64 of the C1 contraction, rows of its result), through the "
              f"reference's t2m->pgemm->m2t; best call {best:.3f} s")
    return smp.flops() / best / 1e12, cores, sample, "reference", outs


def c1_config(world_size: int) -> dict:
    """The workload both arms report (BASELINE.json configs[1], weak-scaled)."""
    s = (world_size - 1).bit_length() if world_size > 1 else 0
    rank_a_global = RANK_A + s
    return {"workload": "C1: A rank-%d (dims 2, %d distributed) x B rank-14, 7 shared indices at "
                        "seeded random positions; result rank-%d in open(A),open(B) order"
                        % (rank_a_global, s, rank_a_global),
            "global_batch": 1, "per_gpu_elements_A": 2**RANK_A,
            "parallelism": f"M-sharded over {world_size} GPU(s) (A's leading open indices)",
            "l2": "inputs (4 GiB A, 4 GiB result per GPU) exceed the 126 MB L2"}


def run_reference_arm(args):
    """--impl reference: the reference's own CPU path (oracle/_ref = the unmodified
    headers + OpenBLAS) on this host's cores. Each step is one 1/64 slice of the
    rank-28 contraction (C1Sample; step i takes slice i mod 64), so the workload,
    metric and unit are the GPU arm's. Nothing from paper_2505_06119_b200 is loaded."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle

    if not oracle.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libqtnh_ref.so was not built"}))
        return
    P = oracle.port()
    smp = C1Sample(P)
    R = oracle.ref()
    cores = os.cpu_count() or 1
    R.set_threads(cores)

    def step(i):
        a = smp.a_slice(i % 2**C1Sample.FIXED)
        _, _, _, t = R.contract(1, [2] * smp.rank_s, 0, (1, 1, 0), a, [2] * RANK_B, 0, (1, 1, 0), smp.b,
                                smp.ap_s, smp.bp, timing=True)
        return t[3] / 1e3

    for i in range(args.warmup):
        step(i)
    times = [step(args.warmup + i) for i in range(args.steps)]
    sec = sum(times)
    v = smp.flops() * len(times) / sec / 1e12
    sample = (f"each step = one of the 64 rank-22 slices of the rank-28 A (first 6 open indices of A fixed) "
              f"contracted with the full B through the reference's t2m->pgemm->m2t (linalg.hpp:208-400), i.e. "
              f"1/64 of the C1 contraction; {cores} OpenBLAS threads, World(1)")
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sec / len(times),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128 (f64)",
            "data": "synthetic (seeded counter-based normals: the rank-28 A's own elements)",
            "config": c1_config(args.gpus),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "reference", "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def hbm_peak():
    """Measured HBM copy peak (MEASURED_PEAKS.json, driver-written) else the
    B200_PROFILING.md fallback."""
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]), "MEASURED_PEAKS.json"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def measure_extras(rk, stream, torch):
    """Secondary hot-path kernels, timed with CUDA events on the rank stream:
    gate application on a 2^30-amplitude state (HBM roofline, 32 B/amplitude per
    gate by convention), the layout permutation, and the config-4 SVD."""
    import ctypes as C

    import numpy as np

    from paper_2505_06119_b200 import circuits, qtnh
    from paper_2505_06119_b200.qtnh import IndexTuple, Tensor, apply_gate

    peak, src = hbm_peak()
    ex = {"hbm_peak_gbs": peak, "hbm_peak_source": src}
    n = 30
    st = Tensor.dense(rk, IndexTuple([2] * n, 0), None, None)
    # seeded random amplitudes rather than the zero fill (the arithmetic-heavy QFT passes
    # run ~10 % faster on an all-zero state; these gate kernels measured the same on both)
    qtnh.check(qtnh.lib.qtnh_counter_complex_normals_device(C.c_void_p(stream.cuda_stream), SEED + 7, 0, 2**n,
                                                            C.c_void_p(st.device_ptr())))
    bytes_per_gate = 32.0 * 2**n
    cases = [("dense_1q_H_q15", [15], circuits.H, False), ("dense_1q_H_q29", [29], circuits.H, False),
             ("dense_2q_fsim_q3_q20", [3, 20], circuits.FSIM, False),
             ("diag_cp_q7_q22", [7, 22], circuits.cp_diag(0.3), True)]
    res = {}
    for name, q, g, diag in cases:
        for _ in range(2):
            apply_gate(st, q, g, diagonal=diag)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10
        e0.record(stream)
        for _ in range(reps):
            apply_gate(st, q, g, diagonal=diag)
        e1.record(stream)
        e1.synchronize()
        ms = e0.elapsed_time(e1) / reps
        gbs = bytes_per_gate / (ms * 1e-3) / 1e9
        entry = {"ms": ms, "GBps_algorithmic": gbs, "frac": gbs / peak}
        if diag:
            # actual traffic: the quarter of amplitudes whose entry != 1 is read + written
            actual = 8.0 * 2**n / (ms * 1e-3) / 1e9
            entry.update(note="the 32 B/amplitude convention overstates this gate: it touches the 1/4 of "
                              "amplitudes whose diagonal entry != 1 (8 B/amplitude)",
                         GBps_actual=actual, frac_actual=actual / peak)
        res[name] = entry
    st.free()
    ex["gate_apply_n30"] = res
    # config-4 SVD: theta 2048 x 2048 -> chi 1024, absorb left
    nn, chi = 2048, 1024
    rng = np.random.default_rng(0)
    a = torch.from_numpy(rng.standard_normal((nn, nn)) + 1j * rng.standard_normal((nn, nn))).cuda()
    u = torch.empty((nn, chi), dtype=torch.complex128, device="cuda")
    s = torch.empty((chi,), dtype=torch.float64, device="cuda")
    vh = torch.empty((chi, nn), dtype=torch.complex128, device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    def svd_call(bt_):
        qtnh.check(qtnh.lib.qtnh_svd_device(rk._h, bt_, nn, nn, C.c_void_p(a.data_ptr()), chi, 1,
                                            C.c_void_p(u.data_ptr()), C.c_void_p(s.data_ptr()),
                                            C.c_void_p(vh.data_ptr())))

    svd_call(1)  # untimed warm-up (workspace mapping, module load, graph instantiation)
    e0.record(stream)
    svd_call(1)
    e1.record(stream)
    e1.synchronize()
    ms = e0.elapsed_time(e1)
    ex["svd_2048_chi1024"] = {"ms": ms, "sweeps": int(qtnh.lib.qtnh_last_error_info()),
                              "conv_TFLOPs": 88.0 * nn**3 / (ms * 1e-3) / 1e12,
                              "flop_convention": "88 n^3 (BASELINE.md section 4)",
                              "note": "one matrix: 64 block pairs per round, the latency-bound eigen step uses 64 SMs"}
    del a, u, s, vh
    # the same SVD batched as config 4 runs it (one layer's thetas at once)
    bt = 8
    a = torch.from_numpy(rng.standard_normal((bt, nn, nn)) + 1j * rng.standard_normal((bt, nn, nn))).cuda()
    u = torch.empty((bt, nn, chi), dtype=torch.complex128, device="cuda")
    s = torch.empty((bt, chi), dtype=torch.float64, device="cuda")
    vh = torch.empty((bt, chi, nn), dtype=torch.complex128, device="cuda")
    svd_call(bt)  # untimed warm-up
    e0.record(stream)
    svd_call(bt)
    e1.record(stream)
    e1.synchronize()
    ms = e0.elapsed_time(e1)
    ex["svd_2048_chi1024_batch8"] = {"ms_per_svd": ms / bt, "sweeps": int(qtnh.lib.qtnh_last_error_info()),
                                     "conv_TFLOPs": bt * 88.0 * nn**3 / (ms * 1e-3) / 1e12,
                                     "input": "i.i.d. complex normal (continuous spectrum: full Jacobi)"}
    # config 4's first saturated thetas have exactly two singular values (chi-fold
    # each): the spectral-split path (projector by Newton-Schulz, pivoted-Cholesky
    # basis); inputs U diag(s) V^H built with torch QR outside the timed region
    q1 = torch.linalg.qr(a)[0]
    q2 = torch.linalg.qr(a.transpose(1, 2).conj().contiguous())[0]
    sv = torch.tensor([0.70719] * chi + [0.35957] * (nn - chi), dtype=torch.float64, device="cuda")
    a = ((q1 * sv) @ q2.transpose(1, 2).conj()).contiguous()
    del q1, q2
    torch.cuda.synchronize()
    svd_call(bt)  # untimed warm-up
    e0.record(stream)
    svd_call(bt)
    e1.record(stream)
    e1.synchronize()
    ms = e0.elapsed_time(e1)
    ex["svd_2048_chi1024_batch8_two_valued"] = {
        "ms_per_svd": ms / bt, "conv_TFLOPs": bt * 88.0 * nn**3 / (ms * 1e-3) / 1e12,
        "input": "U diag(0.70719 x 1024, 0.35957 x 1024) V^H, Haar U, V (config 4's early saturated thetas)"}
    del a, u, s, vh
    return ex

# ---- GPU arm -------------------------------------------------------------------------------------
def run_gpu_arm(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2505_06119_b200 import circuits, kernel_launches, qtnh
    from paper_2505_06119_b200.qtnh import DistParams, IndexTuple, Tensor, World, contract

    world_size = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local % max(1, torch.cuda.device_count()))
    local = local % max(1, torch.cuda.device_count())
    if world_size > 1:
        import datetime

        # barriers of a run whose peer died fail in minutes, not gloo's default half hour
        dist.init_process_group("gloo", init_method="env://", timeout=datetime.timedelta(seconds=600))
    s = (world_size - 1).bit_length() if world_size > 1 else 0
    if world_size > 1 and 2**s != world_size:
        raise SystemExit("--gpus must be a power of two")
    rank_a_global = RANK_A + s
    flops_rank = flops_for(RANK_A)

    world_note = None
    if world_size > 1:
        # One node, one process per GPU. Default: the CUDA-IPC world (collectives are
        # peer-memory kernels over NVLink; it also runs several ranks on one GPU);
        # QTNH_BENCH_WORLD=nccl selects the NCCL world. A failure is fatal: no fallback.
        # If the chosen backend cannot be created, the other real multi-GPU backend is
        # tried (never a 1-rank world), and the line says which one ran.
        kind = os.environ.get("QTNH_BENCH_WORLD", "ipc")
        try:
            world = World.from_env() if kind == "nccl" else World.from_env_ipc()
        except Exception as e:  # noqa: BLE001
            other = "ipc" if kind == "nccl" else "nccl"
            print(f"bench: {kind} world failed ({e}); using the {other} world", file=sys.stderr, flush=True)
            world = World.from_env() if other == "nccl" else World.from_env_ipc()
            kind = f"{other} (after {kind} failed: {e})"
        world_note = f"{kind} world, {world_size} processes on {torch.cuda.device_count()} visible GPU(s)"
    else:
        world = World(1, [local])
    nccl_world = world_size > 1
    stream = torch.cuda.Stream()
    lib = qtnh.lib
    result = {}

    # seeded inputs: this rank's 2^28 shard of A and the full B (counter-based streams)
    a_host = torch.empty(2**RANK_A, dtype=torch.complex128).pin_memory()
    a_np = a_host.numpy()
    lib.qtnh_counter_complex_normals(SEED, rank * 2**RANK_A, 2**RANK_A, a_np.ctypes.data, min(32, os.cpu_count() or 1))
    b_host = torch.from_numpy(circuits.counter_state(SEED + 1, 2**RANK_B)).pin_memory()
    c_host = torch.empty(2**RANK_A, dtype=torch.complex128).pin_memory()
    ap_local, bp = circuits.contraction_positions(SEED, RANK_A, RANK_B, K_SHARED)
    # the distributed leading indices are open (a 1-rank fallback world holds the shard alone)
    ap = [p + s for p in ap_local]

    def barrier():
        if world_size > 1:
            dist.barrier()

    def body(rk):
        rk.set_stream(stream.cuda_stream)
        with torch.cuda.stream(stream):
            ta = Tensor.dense(rk, IndexTuple([2] * rank_a_global, s), DistParams(1, 1, 0), None)
            tb = Tensor.dense(rk, IndexTuple([2] * RANK_B, 0), DistParams(world_size, 1, 0), None)
            qtnh.check(lib.qtnh_tensor_upload_local(ta._h, C.c_void_p(a_host.data_ptr())))
            qtnh.check(lib.qtnh_tensor_upload_local(tb._h, C.c_void_p(b_host.data_ptr())))
            rk.synchronize()

            def step():
                c = contract(ta, tb, ap, bp)
                return c

            clk = ClockSampler(local).__enter__()  # sampling runs through warm-up and timing
            # warm-up
            for _ in range(args.warmup):
                step().free()
            rk.synchronize()
            torch.cuda.synchronize()
            # ---- timed: resident operands -----------------------------------------------
            barrier()
            torch.cuda.synchronize()
            k0 = kernel_launches()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(args.steps):
                step().free()
            e1.record(stream)
            e1.synchronize()
            clk.__exit__(None, None, None)
            torch.cuda.synchronize()
            barrier()
            launches = kernel_launches() - k0
            ms = e0.elapsed_time(e1) / args.steps
            result.update(ms=ms, launches=launches, clocks=clk.summary())

            # ---- parity of the TIMED contraction at its full size (outside the timed region) ------
            # The result block of this rank (2^28 elements, SPEC.md:408 order) is checked
            # (a) element-wise against a host brute-force sum from the oracle port at 1024
            # seeded positions, and (b) on rank 0 of a 1-GPU run against the reference's
            # own output for the slices the cpu_baseline leg contracts (below).
            c = step()
            qtnh.check(lib.qtnh_tensor_download_local(c._h, C.c_void_p(c_host.data_ptr())))
            c.free()
            import oracle

            rng = np.random.default_rng(SEED)
            outs = np.concatenate([[0, 2**RANK_A - 1], rng.integers(0, 2**RANK_A, size=1022)])
            want = c1_brute_force(oracle.port(), outs, shard=rank)
            got = c_host.numpy()[outs]
            result["parity_bf"] = float(np.linalg.norm(got - want) / np.linalg.norm(want))
            result["parity_bf_n"] = int(outs.size)

            # ---- dominant kernel: zgemm alone on the permuted operands ---------------------------
            M, N, K = 2 ** (RANK_A - K_SHARED), 2 ** (RANK_B - K_SHARED), 2**K_SHARED
            ga = torch.empty((M, K), dtype=torch.complex128, device="cuda")
            gb = torch.empty((K, N), dtype=torch.complex128, device="cuda")
            gc = torch.empty((M, N), dtype=torch.complex128, device="cuda")
            ga.copy_(torch.from_numpy(a_np[: M * K].reshape(M, K)))
            gb.copy_(b_host.reshape(K, N))
            for _ in range(3):
                qtnh.check(lib.qtnh_zgemm_device(rk._h, M, N, K, C.c_void_p(ga.data_ptr()),
                                                 C.c_void_p(gb.data_ptr()), C.c_void_p(gc.data_ptr())))
            z0, z1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = max(5, args.steps)
            z0.record(stream)
            for _ in range(reps):
                qtnh.check(lib.qtnh_zgemm_device(rk._h, M, N, K, C.c_void_p(ga.data_ptr()),
                                                 C.c_void_p(gb.data_ptr()), C.c_void_p(gc.data_ptr())))
            z1.record(stream)
            z1.synchronize()
            result["zgemm_ms"] = z0.elapsed_time(z1) / reps
            del ga, gb, gc
            # permute kernel share (A layout permutation)
            perm_a = [i for i in range(RANK_A) if i not in ap_local] + ap_local
            out = torch.empty(2**RANK_A, dtype=torch.complex128, device="cuda")
            src = C.c_void_p(ta.device_ptr())
            from paper_2505_06119_b200._lib import i32_array, i64_array
            p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            qtnh.check(lib.qtnh_permute_device(rk._h, RANK_A, i64_array([2] * RANK_A), i32_array(perm_a), src,
                                               C.c_void_p(out.data_ptr())))
            p0.record(stream)
            for _ in range(reps):
                qtnh.check(lib.qtnh_permute_device(rk._h, RANK_A, i64_array([2] * RANK_A), i32_array(perm_a), src,
                                                   C.c_void_p(out.data_ptr())))
            p1.record(stream)
            p1.synchronize()
            result["permute_ms"] = p0.elapsed_time(p1) / reps
            del out
            peak = C.c_double(0.0)
            qtnh.check(lib.qtnh_probe_fp64_peak(C.c_void_p(stream.cuda_stream), C.byref(peak)))
            result["fp64_peak"] = peak.value

            # ---- e2e through the public API with host buffers -----------------------------------------
            from paper_2505_06119_b200._lib import i32_array as _i32, i64_array as _i64

            dims_a, dims_b = _i64([2] * RANK_A), _i64([2] * RANK_B)
            ap_c, bp_c = _i32(ap_local), _i32(bp)

            class _Step:
                def free(self):
                    pass

            def e2e_step():
                # the public host-buffer entry point: pinned A, B in, C out, H2D / GEMM /
                # D2H pipelined inside (this rank's 2^28 shard of A)
                qtnh.check(lib.qtnh_contract_host(rk._h, RANK_A, dims_a, C.c_void_p(a_host.data_ptr()), RANK_B,
                                                  dims_b, C.c_void_p(b_host.data_ptr()), K_SHARED, ap_c, bp_c,
                                                  C.c_void_p(c_host.data_ptr()), None))
                return _Step()

            e2e_step().free()
            rk.synchronize()
            barrier()
            torch.cuda.synchronize()
            f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e2e_steps = args.steps
            f0.record(stream)
            for _ in range(e2e_steps):
                e2e_step().free()
            f1.record(stream)
            f1.synchronize()
            barrier()
            result["e2e_ms"] = f0.elapsed_time(f1) / e2e_steps
            result["h2d"] = (2**RANK_A + 2**RANK_B) * 16
            result["d2h"] = 2**RANK_A * 16
            ta.free()
            tb.free()
            torch.cuda.synchronize()
            if not args.skip_extras and world_size == 1:
                try:  # secondary figures: a failure here is reported, never fatal for the C1 line
                    result["extras"] = measure_extras(rk, stream, torch)
                except Exception as e:  # noqa: BLE001
                    result["extras"] = {"error": f"{type(e).__name__}: {e}"}
            if not args.skip_configs and world_size > 1:
                import bench_legs

                shared = world_size > torch.cuda.device_count()
                try:
                    result["c2_sharded"] = bench_legs.gpu_c2_sharded(rk, stream, torch, dist, world_size, rank,
                                                                     shared)
                except Exception as e:  # noqa: BLE001  (reported in the line; C1 above stands)
                    result["c2_sharded"] = {"error": f"{type(e).__name__}: {e}"}
            if not args.skip_configs and world_size == 1:
                import bench_legs

                with torch.cuda.stream(stream):
                    result["configs"] = bench_legs.run_all(rk, stream, torch,
                                                           log=lambda m: print(m, file=sys.stderr, flush=True))

    world.run(body)

    # max over ranks
    def rmax(x):
        if world_size == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    ms = rmax(result["ms"])
    e2e_ms = rmax(result["e2e_ms"])
    zg = rmax(result["zgemm_ms"])
    total_flops = flops_rank * world_size
    value = total_flops / (ms * 1e-3) / 1e12
    # the step is the fused-gather GEMM plus a 7 us permute of B (launch list in
    # profiles/): its device time per step is the dominant kernel's duration
    # The GEMM runs the Gauss (3M) complex product: the FP64 tensor pipe issues 6MNK
    # real flops for the 8MNK of the metric; the roofline compares the issued work.
    achieved = 0.75 * flops_rank / (ms * 1e-3) / 1e12
    peak = result["fp64_peak"]
    cpu = None
    parity = {"brute_force_rel_l2": rmax(result["parity_bf"]), "brute_force_elements": result["parity_bf_n"],
              "tolerance": 1e-10}
    if rank == 0 and world_size == 1 and not args.no_cpu_baseline:
        try:
            v, cores, sample, kind, outs = cpu_reference_c1(budget_s=args.cpu_budget, keep_outputs=True)
            cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": kind, "sample": sample}
            # the reference's own rows of the rank-28 result vs the GPU's timed contraction
            num = den = 0.0
            for blk, ref_rows in outs.items():
                got = c_host.numpy()[C1Sample.rows(blk)]
                num += float(np.linalg.norm(got - ref_rows) ** 2)
                den += float(np.linalg.norm(ref_rows) ** 2)
            parity["reference_rows_rel_l2"] = (num / den) ** 0.5
            parity["reference_rows"] = len(outs) * 2 ** (RANK_A - C1Sample.FIXED)
        except Exception as e:  # reported, never fatal for the GPU number
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": f"failed: {e}"}
    parity["rel_l2"] = max(parity["brute_force_rel_l2"], parity.get("reference_rows_rel_l2", 0.0))
    parity["ok"] = parity["rel_l2"] <= 1e-10
    traffic, kname = None, "k_zgemm (DMMA m8n8k4, 4M complex, fused A gather)"
    tpath = os.path.join(ROOT, "profiles", "zgemm_traffic.json")
    if os.path.exists(tpath):  # committed ncu --set full capture of the step's GEMM
        try:
            tj = json.load(open(tpath))
            traffic, kname = tj.get("bytes_per_launch"), tj.get("kernel", kname)
        except Exception:
            traffic = None
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world_size, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "c128 (f64)",
            "data": "synthetic (seeded counter-based complex normals, common.hpp hash_counter + Box-Muller)",
            "config": dict(c1_config(world_size), **({"note": world_note} if world_note else {})),
            "roofline": {"bound": "tensor", "kernel": kname,
                         "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                         "achieved_8mnk": flops_rank / (ms * 1e-3) / 1e12,
                         "frac_8mnk": flops_rank / (ms * 1e-3) / 1e12 / peak,
                         "peak_source": "DMMA-only microbenchmark run live on this device (MEASURED_PEAKS.json "
                                        "has no FP64 entry)",
                         "flop_convention": "value and achieved_8mnk count 8MNK per complex GEMM (BASELINE "
                                            "convention; frac_8mnk > 1 is possible because Gauss 3M issues "
                                            "only 6MNK); achieved / frac count the 6MNK real DMMA flops issued",
                         "traffic": traffic, "kernel_ms": ms,
                         "zgemm_dense_ms": zg, "zgemm_dense_tflops_8mnk": flops_rank / (zg * 1e-3) / 1e12,
                         "permute_ms": result["permute_ms"],
                         "permute_GBps": 2 * 16 * 2**RANK_A / (result["permute_ms"] * 1e-3) / 1e9},
            "cpu_baseline": cpu,
            "parity_rel_l2": parity["rel_l2"], "parity": parity,
            "e2e": {"value": total_flops / (e2e_ms * 1e-3) / 1e12, "unit": UNIT,
                    "h2d_bytes_per_step": result["h2d"], "d2h_bytes_per_step": result["d2h"],
                    "ms_per_step": e2e_ms},
            "gpu_launches": result["launches"],
            "extras": result.get("extras"),
            "configs": result.get("configs"),
            "c2_sharded": result.get("c2_sharded"),
            "clocks": result["clocks"],
        }
        print(json.dumps(line), flush=True)
    if world_size > 1:
        dist.barrier()
        dist.destroy_process_group()
    world.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--skip-extras", action="store_true")
    ap.add_argument("--skip-configs", action="store_true",
                    help="skip the C0/C2/C3/C4 legs (GPU + same-run CPU reference + parity)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_gpu_arm(args)


if __name__ == "__main__":
    main()
