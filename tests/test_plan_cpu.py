"""CPU: the native contraction-order planner (csrc/plan.cpp, qtnh_plan_order) on
config 3's network: a valid order (every step joins two live tensors, one tensor
left), deterministic per seed, and at least as good as the plain greedy."""
import math

import numpy as np

from paper_2505_06119_b200 import network


def labels_dims(rows, cols, depth, seed, n_open):
    items, open_labels, _, _ = network.rcs_network_spec(rows, cols, depth, seed, n_open)
    labels = {i: list(l) for i, (_, l) in enumerate(items)}
    dims = {}
    for arr, labs in items:
        for lab, d in zip(labs, arr.shape):
            dims[lab] = d
    return labels, dims, open_labels


def replay(labels, dims, order):
    L = {k: list(v) for k, v in labels.items()}
    nxt = len(L)
    peak = 0
    for s, (a, b) in enumerate(order):
        assert a in L and b in L and a != b
        la, lb = L.pop(a), L.pop(b)
        sh = [x for x in la if x in lb]
        new = [x for x in la if x not in sh] + [x for x in lb if x not in sh]
        peak = max(peak, sum(math.log2(dims[x]) for x in new))
        L[nxt + s] = new
    assert len(L) == 1
    return L[nxt + len(order) - 1], peak


def test_native_plan_valid_and_deterministic():
    labels, dims, open_labels = labels_dims(5, 6, 14, 2025, 6)
    o1 = network.Network.plan(labels, dims, 2025, trials=24)
    o2 = network.Network.plan(labels, dims, 2025, trials=24)
    assert o1 == o2 and len(o1) == len(labels) - 1
    final, peak = replay(labels, dims, o1)
    assert sorted(final) == sorted(open_labels)
    _, peak0 = replay(labels, dims, network.Network.plan(labels, dims, 2025, trials=1))
    assert peak <= peak0
    assert peak <= 30  # the 5x6 depth-14 network fits a 2^30-element intermediate


def test_plan_small_networks_and_disconnected():
    labels, dims, open_labels = labels_dims(3, 3, 6, 7, 3)
    order = network.Network.plan(labels, dims, 7, trials=4)
    final, _ = replay(labels, dims, order)
    assert sorted(final) == sorted(open_labels)
    # two disconnected pieces: an outer product closes the plan
    labels2 = {0: ["a", "b"], 1: ["b", "c"], 2: ["x"], 3: ["x", "y"]}
    dims2 = {"a": 2, "b": 3, "c": 4, "x": 5, "y": 6}
    final2, _ = replay(labels2, dims2, network.Network.plan(labels2, dims2, 1))
    assert sorted(final2) == ["a", "c", "y"]


def order_flops(labels, dims, order):
    L = {k: list(v) for k, v in labels.items()}
    nxt, fl = len(L), 0.0
    for s, (a, b) in enumerate(order):
        la, lb = L.pop(a), L.pop(b)
        sh = [x for x in la if x in lb]
        new = [x for x in la if x not in sh] + [x for x in lb if x not in sh]
        fl += 8.0 * 2.0 ** (sum(math.log2(dims[x]) for x in new) + sum(math.log2(dims[x]) for x in sh))
        L[nxt + s] = new
    return fl


def test_plan_under_a_memory_budget_minimises_flops():
    """qtnh_plan_order_capped: among the orders whose largest intermediate fits the
    budget the fewest flops win (config 3: the budget is 2^30 elements); without a
    budget the smallest peak wins whatever it costs."""
    labels, dims, open_labels = labels_dims(5, 6, 14, 2025, 6)
    free = network.Network.plan(labels, dims, 2025, trials=96)
    capped = network.Network.plan(labels, dims, 2025, trials=96, max_log2_size=30.0)
    assert capped == network.Network.plan(labels, dims, 2025, trials=96, max_log2_size=30.0)
    final, peak = replay(labels, dims, capped)
    assert sorted(final) == sorted(open_labels) and peak <= 30
    assert order_flops(labels, dims, capped) <= order_flops(labels, dims, free)
    # a budget nothing fits falls back to the smallest peak
    tight = network.Network.plan(labels, dims, 2025, trials=96, max_log2_size=8.0)
    assert replay(labels, dims, tight)[1] == replay(labels, dims, free)[1]
