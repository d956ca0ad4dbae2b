"""Full-size oracle parity for the configurations whose GPU runs were checked only
against the repo's own kernels (VERDICT r1 'What's missing' 4):

* C3 -- the 5x6 depth-14 RCS network contracted on the GPU along the seeded greedy
  order, against the host replay of the same order (oracle.network_contract,
  numpy tensordot = the SPEC contraction, up to 2^30-element intermediates);
* C4 -- the first saturated two-site updates (2048 x 2048 thetas, chi = 1024) of
  the real 40-site run, against the unmodified reference's contract -> gate ->
  psvd (zgesdd) -> truncate_svd -> absorb_singular_left on the same inputs
  (linalg.hpp:208-523): S and U S Vh within the north-star 1e-10.
Both need the GPU box's host (~100 GB of RAM for C3, 16 cores)."""
import os

import numpy as np
import pytest

import oracle
from conftest import rel_l2
from paper_2505_06119_b200 import network, qtnh
from paper_2505_06119_b200.qtnh import World

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
TOL = 1e-10
SEED = 2025


def test_c3_full_network_vs_host_replay():
    items, open_labels, open_q, fixed = network.rcs_network_spec(5, 6, 14, SEED, 6)
    labels = {i: list(l) for i, (_, l) in enumerate(items)}
    dims = {}
    for a, l in items:
        dims.update(zip(l, a.shape))
    order = network.Network.plan(labels, dims, SEED, trials=2048, max_log2_size=30.0)  # the bench leg's order

    def body(rk):
        net, ol, _, _ = network.build_rcs_network(rk, 5, 6, 14, SEED, 6)
        assert ol == open_labels and net.labels == labels
        last = net.contract_order_native(order)
        res_labels = net.labels[last]
        amp = net.tensors[last].to_global_vector().reshape([2] * len(res_labels))
        net.tensors[last].free()
        return np.transpose(amp, [res_labels.index(x) for x in open_labels]).reshape(-1)

    # Map the pool once for this network only: left set, every later world of the
    # process would map 120 GB at creation and trim it at destruction (~2 s a world).
    qtnh.check(qtnh.lib.qtnh_set_option(b"pool_reserve_gb", 120.0))
    try:
        got = World(1).run(body)[0]
    finally:
        qtnh.check(qtnh.lib.qtnh_set_option(b"pool_reserve_gb", 0.0))
    want, wl = oracle.network_contract(items, order)
    want = np.transpose(want, [wl.index(x) for x in open_labels]).reshape(-1)
    assert rel_l2(got, want) < TOL


def test_c4_saturated_updates_vs_reference():
    import torch

    import bench_legs

    if not oracle.ref_available():
        pytest.skip("reference build absent")
    out = {}

    def body(rk):
        st = torch.cuda.Stream()
        rk.set_stream(st.cuda_stream)
        with torch.cuda.stream(st):
            g, cap = bench_legs.gpu_c4(rk, st, torch, depth=12, capture=2, bitstrings=16)
        out["gpu"], out["cap"] = g, cap

    World(1).run(body)
    assert out["cap"], "the run reached no layer with two saturated pairs"
    cpu = bench_legs.cpu_c4(out["cap"])
    for upd in cpu["updates"]:
        assert upd["rel_l2_usvh"] < TOL, upd
        assert upd["s_max_rel_err"] < TOL, upd
