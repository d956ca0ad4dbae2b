"""The other BASELINE.json configurations as bench.py extras, each GPU number next
to the reference's CPU number measured in the same run on this host's cores
(SURVEY.md 8(d)), and each with its parity check.

  C0  QFT-16 (latency-bound 1 MiB state): 144 gates gate by gate, direct and
      replayed from a CUDA graph; CPU = the reference's full QFT-16 (World(1)).
  C2  QFT-33 on one GPU (128 GiB state in place): the cache-blocked QFT, norm and
      DFT spot amplitudes; CPU = the reference on World(8), n = 22, split 3 (the
      structure of the sharded run), the first gates timed and scaled by 2^(33-22)
      per gate to the 577 gates of n = 33 -- labelled extrapolated.
  C3  RCS 5x6 depth-14 tensor network along the seeded greedy order: GPU chain of
      644 contractions vs the 30-qubit statevector; CPU = the reference's
      t2m -> pgemm -> m2t timed on every step whose operands and result hold
      <= 2^22 elements, and on calibration contractions that fit a
      per-element + per-flop cost model for the 9 large steps -- extrapolated.
  C4  MPS-40, chi = 1024, depth 20: the whole run on the GPU; CPU = the reference
      (contract -> gate -> psvd/zgesdd -> truncate_svd -> absorb) on the first
      saturated two-site updates of this very run, whose inputs are captured from
      the GPU; the same updates are the parity check (S and U S Vh).

Only bench.py imports this module; the CPU legs are the one other place (with
bench.py's reference arm) that executes oracle/.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import time

import numpy as np

SEED = 2025


def _events(torch, stream):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    return e0, e1


def _rel(a, b) -> float:
    nb = float(np.linalg.norm(b))
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / (nb if nb > 0 else 1.0))


# ---- C0 --------------------------------------------------------------------------------------------
def gpu_c0(rk, stream, torch):
    from paper_2505_06119_b200 import circuits
    from paper_2505_06119_b200.qtnh import IndexTuple, Tensor, apply_gate, swap_indices

    n = 16
    gates = circuits.qft_gates(n, swaps=True)
    psi0 = circuits.counter_state(SEED, 2**n)
    psi0 = psi0 / np.linalg.norm(psi0)

    def seq(t):
        for kind, q, g in gates:
            if kind == "h":
                apply_gate(t, q, g)
            elif kind == "cp":
                apply_gate(t, q, g, diagonal=True)
            else:
                swap_indices(t, q[0], q[1])

    t = Tensor.dense(rk, IndexTuple([2] * n, 0), None, psi0)
    seq(t)
    out = t.to_global_vector()
    for _ in range(3):
        seq(t)
    rk.synchronize()
    reps = 20
    e0, e1 = _events(torch, stream)
    e0.record(stream)
    for _ in range(reps):
        seq(t)
    e1.record(stream)
    e1.synchronize()
    direct = e0.elapsed_time(e1) / reps
    with rk.capture() as g:
        seq(t)
    g.launch()
    rk.synchronize()
    e0.record(stream)
    for _ in range(reps):
        g.launch()
    e1.record(stream)
    e1.synchronize()
    graph = e0.elapsed_time(e1) / reps
    g.free()
    t.free()
    # the same QFT through the fused path (qtnh_qft: cache-blocked layers + bit reversal)
    from paper_2505_06119_b200.qtnh import qft

    f = Tensor.dense(rk, IndexTuple([2] * n, 0), None, psi0)
    qft(f, swaps=True)
    fused_out = f.to_global_vector()
    e0.record(stream)
    for _ in range(reps):
        qft(f, swaps=True)
    e1.record(stream)
    e1.synchronize()
    fused = e0.elapsed_time(e1) / reps
    f.free()
    return {"gates": len(gates), "ms_direct": direct, "ms_graph": graph, "us_per_gate_graph": 1e3 * graph / len(gates),
            "ms_fused_qft": fused, "fused_rel_l2_vs_gate_by_gate": _rel(fused_out, out),
            "bound": "latency (1 MiB state, L2-resident)"}, psi0, out


def cpu_c0(psi0, gpu_out):
    import oracle

    R = oracle.ref()
    R.set_threads(os.cpu_count() or 1)
    want, ms = R.qft(16, psi0, swaps=True, timing=True)
    return {"ms": ms, "cores": os.cpu_count(), "kind": "reference",
            "sample": "full QFT-16, 144 gates, each a t2m -> pgemm -> m2t contraction (+ permute for SWAPs), World(1)",
            "parity_rel_l2": _rel(gpu_out, want)}


# ---- C2 --------------------------------------------------------------------------------------------
def gpu_c2(rk, stream, torch, n=33, spots=4):
    from paper_2505_06119_b200 import qtnh
    from paper_2505_06119_b200.mps import _DevView
    from paper_2505_06119_b200.qtnh import IndexTuple, Tensor

    N = 2**n
    t = Tensor.dense(rk, IndexTuple([2] * n, 0), None, None)
    psi = torch.as_tensor(_DevView(t.device_ptr(), N), device="cuda")

    def init():
        qtnh.check(qtnh.lib.qtnh_counter_complex_normals_device(C.c_void_p(stream.cuda_stream), SEED, 0, N,
                                                                C.c_void_p(t.device_ptr())))

    chunk = 2**27
    with torch.cuda.stream(stream):
        init()
        nrm2 = sum(float(psi[c:c + chunk].abs().pow(2).sum()) for c in range(0, N, chunk))
        psi.mul_(1.0 / math.sqrt(nrm2))
        # DFT spot amplitudes y_k = sum_j x_j e^{2 pi i j k / N} / sqrt(N)
        rng = np.random.default_rng(SEED)
        ks = [0, 1, N - 1] + [int(x) for x in rng.integers(2, N - 1, size=max(0, spots - 3))]
        want = {}
        for k in ks:
            acc = torch.zeros((), dtype=torch.complex128, device="cuda")
            for c in range(0, N, chunk):
                j = torch.arange(c, c + chunk, dtype=torch.int64, device="cuda")
                ph = torch.remainder(j * k, N).to(torch.float64) * (2 * math.pi / N)
                acc += (psi[c:c + chunk] * torch.polar(torch.ones_like(ph), ph)).sum()
            want[k] = complex(acc.item()) / math.sqrt(N)
        stream.synchronize()
        e0, e1 = _events(torch, stream)
        e0.record(stream)
        qtnh.qft(t, swaps=True)
        e1.record(stream)
        e1.synchronize()
        ms_first = e0.elapsed_time(e1)  # first call of the process: module load, tensor maps, attributes
        nrm = math.sqrt(sum(float(psi[c:c + chunk].abs().pow(2).sum()) for c in range(0, N, chunk)))
        err = max(abs(complex(psi[k].item()) - w) / abs(w) for k, w in want.items())
        first = {k: complex(psi[k].item()) for k in ks}
        # the timed run: the same seeded state again, after that warm-up call
        init()
        psi.mul_(1.0 / math.sqrt(nrm2))
        stream.synchronize()
        e0.record(stream)
        qtnh.qft(t, swaps=True)
        e1.record(stream)
        e1.synchronize()
        ms = e0.elapsed_time(e1)
        same = all(complex(psi[k].item()) == v for k, v in first.items())
    t.free()
    gates = n + n * (n - 1) // 2 + n // 2
    return {"n": n, "gates": gates, "ms": ms, "ms_first_call": ms_first,
            "effective_GBps_32B_per_gate": gates * 32.0 * N / (ms * 1e-3) / 1e9,
            "norm_after": nrm, "dft_spot_max_rel_err": err, "dft_spots": len(ks),
            "timed_run_equals_checked_run": same}


def cpu_c2(budget_gates=12, n_small=22, n_full=33):
    import oracle

    R = oracle.ref()
    R.set_threads(1)  # one BLAS thread per rank thread (catch_main.cpp:22), 8 rank threads
    psi = oracle.port().counter_normals(SEED, 0, 2**n_small)
    psi /= np.linalg.norm(psi)
    _, ms = R.qft(n_small, psi, swaps=True, world=8, split=3, gate_limit=budget_gates, timing=True)
    per_gate = ms / budget_gates
    gates_full = n_full + n_full * (n_full - 1) // 2 + n_full // 2
    return {"kind": "reference", "cores": 8, "extrapolated": True,
            "sample": f"reference World(8), n = {n_small}, split 3: first {budget_gates} QFT gates (H and CP on "
                      f"the distributed qubit 0 -> remap exchanges), {ms:.0f} ms",
            "ms_per_gate_sample": per_gate,
            "s_extrapolated_n33": per_gate * 2.0 ** (n_full - n_small) * gates_full / 1e3,
            "extrapolation": f"per-gate time x 2^{n_full - n_small} (state size) x {gates_full} gates"}


# ---- C3 --------------------------------------------------------------------------------------------
def c3_steps(net_labels, dims, order):
    """Per step: (dims_a, dims_b, apos, bpos, M, N, K) in the operand order the
    GPU executor uses (the larger operand first)."""
    L = {k: list(v) for k, v in net_labels.items()}
    n = len(L)
    out = []
    for s, (a, b) in enumerate(order):
        la, lb = L.pop(a), L.pop(b)
        if sum(math.log2(dims[x]) for x in lb) > sum(math.log2(dims[x]) for x in la):
            la, lb = lb, la
        sh = [x for x in la if x in lb]
        M = math.prod(dims[x] for x in la if x not in sh)
        N = math.prod(dims[x] for x in lb if x not in sh)
        K = math.prod(dims[x] for x in sh)
        out.append(([dims[x] for x in la], [dims[x] for x in lb], [la.index(x) for x in sh],
                    [lb.index(x) for x in sh], M, N, K))
        L[n + s] = [x for x in la if x not in sh] + [x for x in lb if x not in sh]
    return out


def gpu_c3(rk, stream, torch, rows=5, cols=6, depth=14, n_open=6, trials=2048, log2_cap=30.0):
    from paper_2505_06119_b200 import circuits, mps, network
    from paper_2505_06119_b200.qtnh import IndexTuple, Tensor, apply_gate

    net, open_labels, open_q, fixed = network.build_rcs_network(rk, rows, cols, depth, SEED, n_open)
    t0 = time.perf_counter()
    # order search: the fewest flops among the orders whose largest intermediate fits
    # 2^30 elements (16 GiB); planned once per circuit, reused for every output batch
    order = network.Network.plan(net.labels, net.dims, SEED, trials=trials, max_log2_size=log2_cap)
    plan_s = time.perf_counter() - t0
    # one untimed run of the same order first (the memory pool maps its blocks and
    # the offset-table caches fill, as in any run after the first)
    warm = net.contract_order_native(order)
    net.tensors[warm].free()
    net, open_labels, open_q, fixed = network.build_rcs_network(rk, rows, cols, depth, SEED, n_open)
    labels0 = {k: list(v) for k, v in net.labels.items()}
    fl, big, by = network.Network.cost(net.labels, net.dims, order)
    rk.synchronize()
    e0, e1 = _events(torch, stream)
    e0.record(stream)
    last = net.contract_order_native(order)
    e1.record(stream)
    e1.synchronize()
    sec = e0.elapsed_time(e1) / 1e3
    res_labels = net.labels[last]
    amp = net.tensors[last].to_global_vector().reshape([2] * len(res_labels))
    amp = np.transpose(amp, [res_labels.index(l) for l in open_labels]).reshape(-1)
    net.tensors[last].free()
    # the same circuit on a 30-qubit statevector (the repo's own gate kernels)
    n = rows * cols
    st = Tensor.dense(rk, IndexTuple([2] * n, 0), None, None)
    with torch.cuda.stream(stream):
        v = torch.as_tensor(mps._DevView(st.device_ptr(), 2**n), device="cuda")
        v.zero_()
        v[0] = 1.0
        for kind, qs, g in network.rcs_grid_circuit(rows, cols, depth, SEED):
            apply_gate(st, list(qs), mps.SINGLE_QUBIT[g] if kind == "1q" else circuits.FSIM)
        psi = v.reshape([2] * n)
        idx = tuple(slice(None) if q in open_q else fixed[q] for q in range(n))
        want = psi[idx].reshape(-1).cpu().numpy()
    st.free()
    steps = c3_steps(labels0, net.dims, order)
    return ({"contractions": len(order), "order_flops_8mnk": fl, "largest_intermediate": big, "plan_s": plan_s,
             "plan_trials": trials, "plan_log2_element_budget": log2_cap,
             "s": sec, "TFLOPs": fl / sec / 1e12, "rel_l2_vs_statevector": _rel(amp, want)}, steps)


def cpu_c3(steps, small=2**22, budget_s=20.0):
    """Reference (t2m -> pgemm -> m2t on seeded inputs of each step's shapes, World(1),
    all host threads) on every step with |A| + |B| + |C| <= `small`; the large steps
    from a cost model t = a * elements + b * flops + c fitted (least squares) on the
    measured steps plus calibration contractions of 2^20-2^23 elements."""
    import oracle

    R = oracle.ref()
    cores = os.cpu_count() or 1
    R.set_threads(cores)
    P = oracle.port()

    def run(da, db, ap, bp):
        a = P.counter_normals(SEED, 0, int(np.prod(da)))
        b = P.counter_normals(SEED + 1, 0, int(np.prod(db)))
        _, _, _, t = R.contract(1, da, 0, (1, 1, 0), a, db, 0, (1, 1, 0), b, ap, bp, timing=True)
        return t[3] / 1e3

    meas, feats, measured_s = 0, [], 0.0
    t_start = time.perf_counter()
    big = []
    for da, db, ap, bp, M, N, K in steps:
        el = M * K + K * N + M * N
        if el > small:
            big.append((el, 8.0 * M * N * K))
            continue
        if time.perf_counter() - t_start > budget_s:
            big.append((el, 8.0 * M * N * K))
            continue
        sec = run(da, db, ap, bp)
        measured_s += sec
        meas += 1
        feats.append((el, 8.0 * M * N * K, sec))
    # calibration: qubit tensors, element-heavy (small K), flop-heavy (K = 2^7), and the
    # large steps' own (M, K, N) aspect with M N scaled down to 2^22 (their K kept)
    for ra, rb, k in [(20, 4, 2), (21, 3, 1), (20, 14, 7), (22, 9, 7), (18, 22, 9), (16, 24, 9), (14, 22, 7)]:
        da, db = [2] * ra, [2] * rb
        sec = run(da, db, list(range(ra - k, ra)), list(range(k)))
        M, N, K = 2 ** (ra - k), 2 ** (rb - k), 2**k
        feats.append((M * K + K * N + M * N, 8.0 * M * N * K, sec))
    X = np.array([[f[0], f[1], 1.0] for f in feats])
    y = np.array([f[2] for f in feats])
    w = 1.0 / np.maximum(y, 1e-4)  # relative least squares
    coef, *_ = np.linalg.lstsq(X * w[:, None], y * w, rcond=None)
    coef = np.maximum(coef, 0.0)
    est = sum(coef[0] * el + coef[1] * fl + coef[2] for el, fl in big)
    return {"kind": "reference", "cores": cores, "extrapolated": True,
            "measured_steps": meas, "measured_s": measured_s, "modelled_steps": len(big), "modelled_s": est,
            "s_total_estimate": measured_s + est,
            "model": {"s_per_element": coef[0], "s_per_flop": coef[1], "s_per_call": coef[2]},
            "sample": f"{meas} of {len(steps)} steps timed through the reference's t2m -> pgemm -> m2t; the "
                      f"{len(big)} large steps (up to 2^30-element operands) from the fitted cost model"}


# ---- C4 --------------------------------------------------------------------------------------------
def gpu_c4(rk, stream, torch, n=40, depth=20, chi=1024, capture=2, bitstrings=1024, capture_layer=None):
    """The whole MPS run; before the first layer with `capture` saturated pairs the
    sites of those pairs are copied to the host, and after it their new sites and
    singular values, for the CPU leg (timing + parity on identical inputs)."""
    from paper_2505_06119_b200 import circuits, mps

    layers = mps.rcs_1d_layers(n, depth, SEED)
    m = mps.MPS(rk, n, chi)
    cap = None
    rk.synchronize()
    e0, e1 = _events(torch, stream)
    e0.record(stream)
    t0 = time.perf_counter()
    host_s = 0.0
    for li, (singles, pairs) in enumerate(layers):
        for q, g in enumerate(singles):
            m.apply_1q(q, mps.SINGLE_QUBIT[g])
        sat = [q for q, _ in pairs if m.sites[q].shape().dims == [chi, 2, chi]
               and m.sites[q + 1].shape().dims == [chi, 2, chi]]
        if cap is None and len(sat) >= capture and (capture_layer is None or li == capture_layer):
            h0 = time.perf_counter()
            cap = [{"q": q, "a": m.sites[q].local_data().copy(), "b": m.sites[q + 1].local_data().copy()}
                   for q in sat[:capture]]
            host_s += time.perf_counter() - h0
            res = m.apply_layer(pairs, circuits.FSIM)
            h0 = time.perf_counter()
            for c in cap:
                c["u"] = m.sites[c["q"]].local_data().copy()
                c["vh"] = m.sites[c["q"] + 1].local_data().copy()
                c["s"] = dict(zip([p[0] for p in pairs], res))[c["q"]][0].copy()
            host_s += time.perf_counter() - h0
        else:
            m.apply_layer(pairs, circuits.FSIM)
    e1.record(stream)
    e1.synchronize()
    wall = time.perf_counter() - t0
    dev_s = e0.elapsed_time(e1) / 1e3
    rng = np.random.default_rng(SEED)
    amps = m.amplitudes(rng.integers(0, 2, size=(bitstrings, n)))
    out = {"n": n, "depth": depth, "chi": chi, "s_device": dev_s - host_s, "s_wall": wall - host_s,
           "capture_host_s_excluded": host_s, "fidelity": float(np.exp(m.log_fidelity)),
           "bond_dims_max": max(m.bond_dims()), "amp_norm2_sum": float(np.sum(np.abs(amps) ** 2))}
    m.free()
    return out, cap


def cpu_c4(cap, chi=1024):
    """The reference's two-site update on the captured inputs: contract the two
    sites (t2m -> pgemm -> m2t), apply fSim (contraction + permute back), psvd
    (zgesdd), truncate_svd to chi, absorb left -- timed per update, and compared
    with the GPU's new sites: S (relative) and U S Vh (relative L2)."""
    import oracle
    from paper_2505_06119_b200 import circuits

    R = oracle.ref()
    cores = os.cpu_count() or 1
    R.set_threads(cores)
    res = []
    for c in cap:
        t0 = time.perf_counter()
        th, dims, _ = R.contract(1, [chi, 2, chi], 0, (1, 1, 0), c["a"], [chi, 2, chi], 0, (1, 1, 0), c["b"], [2], [0])
        t1 = time.perf_counter()
        # fSim on indices 1, 2 of (chi, 2, 2, chi): treat chi = 2^10 as ten qubits
        nq = 2 * int(math.log2(chi)) + 2
        th = R.gate(1, nq, 0, None, th, [int(math.log2(chi)), int(math.log2(chi)) + 1], circuits.FSIM)
        t2 = time.perf_counter()
        u, s, vh, tt = R.svd(th.reshape(2 * chi, 2 * chi), chi=chi, absorb=1, timing=True)
        t3 = time.perf_counter()
        want = u @ vh
        got = c["u"].reshape(2 * chi, chi) @ c["vh"].reshape(chi, 2 * chi)
        res.append({"site": c["q"], "s_contract": t1 - t0, "s_gate": t2 - t1, "s_svd_truncate_absorb": t3 - t2,
                    "s_update": t3 - t0, "rel_l2_usvh": _rel(got, want),
                    "s_max_rel_err": float(np.max(np.abs(c["s"] - s)) / s[0])})
    return {"kind": "reference", "cores": cores, "updates": res,
            "s_per_update": float(np.mean([r["s_update"] for r in res])),
            "sample": f"the first {len(cap)} saturated two-site updates (2048 x 2048 thetas, chi = 1024) of the "
                      "GPU run, inputs captured from it"}


def run_all(rk, stream, torch, log=None):
    """All legs; each failure is recorded, never fatal for the C1 headline."""
    out = {}

    def leg(name, fn):
        t0 = time.perf_counter()
        try:
            out[name] = fn()
        except Exception as e:  # noqa: BLE001
            out[name] = {"error": f"{type(e).__name__}: {e}"}
        out[name]["leg_wall_s"] = time.perf_counter() - t0

    def c0():
        g, psi0, o = gpu_c0(rk, stream, torch)
        return {"gpu": g, "cpu": cpu_c0(psi0, o)}

    def c2():
        return {"gpu": gpu_c2(rk, stream, torch), "cpu": cpu_c2()}

    def c3():
        g, steps = gpu_c3(rk, stream, torch)
        return {"gpu": g, "cpu": cpu_c3(steps)}

    def c4():
        g, cap = gpu_c4(rk, stream, torch)
        return {"gpu": g, "cpu": cpu_c4(cap) if cap else {"error": "no saturated layer reached"}}

    for name, fn in (("C0_qft16", c0), ("C2_qft33", c2), ("C3_rcs_tn", c3), ("C4_mps40", c4)):
        if log:
            log(f"leg {name}")
        leg(name, fn)
    return out


# ---- C2 sharded (bench.py --gpus N under torchrun) -----------------------------------------------
def gpu_c2_sharded(rk, stream, torch, dist, world_size, rank, shared_gpu, swaps=5, spots=4):
    """QFT on a state sharded over the world (split s = log2 N, the leading s
    qubits select the GPU) and the local<->distributed index
    swap it is built from, timed on the device and reduced as the max over ranks:
      * swap: qubit 0 (distributed) <-> qubit n-1 (local), in place; every GPU
        sends and receives half its shard: 16 * 2^(n-s-1) B per direction;
      * the whole QFT (distributed layers fused over peer memory, local layers
        cache-blocked, bit reversal) with norm and DFT spot-amplitude checks.
    n = 34 when every rank has its own GPU (BASELINE.json configs[2]); with
    ranks sharing a GPU n = 30 + s (16 GiB per rank; 29 + s beyond 4 ranks per GPU) and
    the bytes stay in HBM."""
    from paper_2505_06119_b200 import qtnh
    from paper_2505_06119_b200.mps import _DevView
    from paper_2505_06119_b200.qtnh import DistParams, IndexTuple, Tensor

    s = (world_size - 1).bit_length()
    # ranks sharing one GPU: 16 GiB shards up to 4 ranks per GPU, 8 GiB beyond (8 x 16 GiB
    # plus what the C1 leg left in the pool does not fit 180 GB)
    per_gpu = -(-world_size // max(1, torch.cuda.device_count()))
    n = (30 + s if per_gpu <= 4 else 29 + s) if shared_gpu else 34
    nl = n - s
    N, NL = 2**n, 2**nl
    t = Tensor.dense(rk, IndexTuple([2] * n, s), DistParams(1, 1, 0), None)
    psi = torch.as_tensor(_DevView(t.device_ptr(), NL), device="cuda")
    chunk = min(NL, 2**27)

    def allsum(x):
        v = torch.tensor([x], dtype=torch.float64)
        dist.all_reduce(v)
        return float(v.item())

    def allmax(x):
        v = torch.tensor([x], dtype=torch.float64)
        dist.all_reduce(v, op=dist.ReduceOp.MAX)
        return float(v.item())

    with torch.cuda.stream(stream):
        qtnh.check(qtnh.lib.qtnh_counter_complex_normals_device(C.c_void_p(stream.cuda_stream), SEED, rank * NL, NL,
                                                                C.c_void_p(t.device_ptr())))
        nrm2 = allsum(sum(float(psi[c:c + chunk].abs().pow(2).sum()) for c in range(0, NL, chunk)))
        psi.mul_(1.0 / math.sqrt(nrm2))
        rng = np.random.default_rng(SEED)
        ks = [0, 1, N - 1] + [int(x) for x in rng.integers(2, N - 1, size=max(0, spots - 3))]
        want = {}
        for k in ks:  # partial DFT sums over this shard, summed over ranks
            acc = torch.zeros((), dtype=torch.complex128, device="cuda")
            for c in range(0, NL, chunk):
                j = torch.arange(rank * NL + c, rank * NL + c + chunk, dtype=torch.int64, device="cuda")
                ph = torch.remainder(j * k, N).to(torch.float64) * (2 * math.pi / N)
                acc += (psi[c:c + chunk] * torch.polar(torch.ones_like(ph), ph)).sum()
            z = complex(acc.item())
            want[k] = complex(allsum(z.real), allsum(z.imag)) / math.sqrt(N)
        stream.synchronize()
        e0, e1 = _events(torch, stream)
        for _ in range(2):  # warm-up (an even count restores the state)
            qtnh.swap_indices(t, 0, n - 1)
        rk.synchronize()
        dist.barrier()
        e0.record(stream)
        for _ in range(2 * swaps):
            qtnh.swap_indices(t, 0, n - 1)
        e1.record(stream)
        e1.synchronize()
        swap_ms = allmax(e0.elapsed_time(e1) / (2 * swaps))
        dist.barrier()
        e0.record(stream)
        qtnh.qft(t, swaps=True)
        e1.record(stream)
        e1.synchronize()
        qft_ms = allmax(e0.elapsed_time(e1))
        nrm = math.sqrt(allsum(sum(float(psi[c:c + chunk].abs().pow(2).sum()) for c in range(0, NL, chunk))))
        errs = []
        for k, w in want.items():
            owner = k >> nl
            v = complex(psi[k - owner * NL].item()) if owner == rank else 0j
            v = complex(allsum(v.real), allsum(v.imag))
            errs.append(abs(v - w) / abs(w))
    t.free()
    bytes_dir = 16.0 * 2 ** (nl - 1)
    gbs = bytes_dir / (swap_ms * 1e-3) / 1e9
    gates = n + n * (n - 1) // 2 + n // 2
    return {"n": n, "split": s, "ranks": world_size, "shard_GiB": 16.0 * NL / 2**30,
            "swap_dist_local_ms": swap_ms, "swap_bytes_per_gpu_per_direction": bytes_dir,
            "swap_GBps_per_direction": gbs, "swap_frac_of_900GBps_nvlink": gbs / 900.0,
            "qft_ms": qft_ms, "qft_gates": gates,
            "qft_effective_GBps_per_gpu_32B_per_gate": gates * 32.0 * NL / (qft_ms * 1e-3) / 1e9,
            "norm_after": nrm, "dft_spot_max_rel_err": max(errs),
            "note": ("ranks share one GPU: the swap moves bytes inside HBM, not over NVLink" if shared_gpu
                     else "one GPU per rank: the swap moves bytes over NVLink (peer stores / NCCL)")}
