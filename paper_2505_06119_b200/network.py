"""Tensor networks contracted pairwise on the GPU (SPEC network::contract /
contract_order; config 3 of BASELINE.json).

A network is a set of device tensors whose indices carry labels; a label shared
by two tensors is a bond. Contracting a pair sums over all their shared labels
with qtnh.contract (result order open(a) then open(b)). The order is
either supplied or chosen greedily: repeatedly contract the connected pair with
the smallest result (ties broken by a seeded hash), the order SURVEY.md 8(d)
fixes for config 3. The order is computed once on the host (plan()) and can be
replayed by the reference oracle for parity.
"""
from __future__ import annotations

import math
import os
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import circuits, qtnh
from .qtnh import IndexTuple, Tensor

_BIG_FIRST = os.environ.get("QTNH_NET_BIG_FIRST", "1") != "0"


class Network:
    """Labelled tensors on one rank, or -- in a world of P > 1 ranks (SURVEY.md 8(e)
    C3) -- replicated on every rank (DistParams(1, P, 0)): small contractions then
    run as replicas, and a contraction of at least `shard_flops` is M-sharded like
    C1: its first operand gets log2 P of its open qubit indices distributed
    (rebcast to one copy, permute with a new split), the other operand stays
    replicated, and the result stays sharded for the next steps (a contraction
    of two sharded operands replicates the smaller one first)."""

    def __init__(self, rank: qtnh.Rank, shard_flops: float = 1e11):
        self.rank = rank
        self.tensors: Dict[int, Tensor] = {}
        self.labels: Dict[int, List[str]] = {}
        self.dims: Dict[str, int] = {}
        self._next = 0
        self.world = rank.size()
        self.shard_flops = shard_flops
        self.rep = qtnh.DistParams(1, self.world, 0)
        self.n_sharded = 0      # contractions run M-sharded
        self.n_replicated = 0   # sharded operands gathered back to replicas

    def add(self, data: np.ndarray, labels: Sequence[str]) -> int:
        data = np.ascontiguousarray(data, dtype=np.complex128)
        shape = list(data.shape) if data.ndim else []
        assert len(shape) == len(labels)
        for lab, d in zip(labels, shape):
            if self.dims.setdefault(lab, d) != d:
                raise qtnh.InvalidArgument(f"bond {lab} has inconsistent dimensions")
        t = Tensor.from_global(self.rank, IndexTuple(shape, 0), self.rep, data.reshape(-1))
        i = self._next
        self._next += 1
        self.tensors[i] = t
        self.labels[i] = list(labels)
        return i

    # -- planning (host only) ------------------------------------------------------------
    @staticmethod
    def cost(labels: Dict[int, List[str]], dims: Dict[str, int], order) -> Tuple[float, int, float]:
        """(sum of 8MNK flops, largest intermediate, sum of 16(|A|+|B|+|C|) bytes)."""
        import math

        L = {k: list(v) for k, v in labels.items()}
        nxt = max(L) + 1
        fl, big, by = 0.0, 0, 0.0
        for s, (a, b) in enumerate(order):
            la, lb = L.pop(a), L.pop(b)
            sh = [x for x in la if x in lb]
            M = math.prod(dims[x] for x in la if x not in sh)
            N = math.prod(dims[x] for x in lb if x not in sh)
            K = math.prod(dims[x] for x in sh)
            fl += 8.0 * M * N * K
            by += 16.0 * (M * K + K * N + M * N)
            big = max(big, M * N)
            L[nxt + s] = [x for x in la if x not in sh] + [x for x in lb if x not in sh]
        return fl, big, by

    @staticmethod
    def plan(labels: Dict[int, List[str]], dims: Dict[str, int], seed: int = 0, trials: int = 64,
             keep_open: Sequence[str] = (), max_log2_size: float = 0.0) -> List[Tuple[int, int]]:
        """Seeded greedy contraction order, planned natively (csrc/plan.cpp via
        qtnh_plan_order): trial 0 is the plain smallest-result greedy (SURVEY.md
        8(d)), further trials seeded randomised greedy passes; the order with the
        smallest largest intermediate, then fewest flops, wins -- or, with a memory
        budget `max_log2_size`, the fewest flops among the orders whose largest
        intermediate has at most 2^max_log2_size elements. Deterministic per
        seed; tensor ids must be 0..n-1 and the result of step s gets id n + s."""
        import math

        from ._lib import i32_array

        ids = sorted(labels)
        if ids != list(range(len(ids))):
            raise qtnh.InvalidArgument("plan needs tensor ids 0..n-1")
        names = sorted({x for v in labels.values() for x in v})
        lid = {x: i for i, x in enumerate(names)}
        offs, flat = [0], []
        for t in ids:
            flat.extend(lid[x] for x in labels[t])
            offs.append(len(flat))
        lg = np.array([math.log2(dims[x]) for x in names], dtype=np.float64)
        out = np.zeros(2 * max(1, len(ids) - 1), dtype=np.int32)
        qtnh.check(qtnh.lib.qtnh_plan_order_capped(len(ids), i32_array(offs), i32_array(flat or [0]), len(names),
                                                   lg.ctypes.data, int(seed) & (2**64 - 1), int(trials),
                                                   float(max_log2_size),
                                                   out.ctypes.data_as(qtnh.C.POINTER(qtnh.C.c_int))))
        return [(int(out[2 * s]), int(out[2 * s + 1])) for s in range(len(ids) - 1)]

    # ---- multi-rank placement ---------------------------------------------------------
    def _replicate(self, t: Tensor) -> Tensor:
        """A copy of t on every rank (split 0, DistParams(1, P, 0))."""
        u = qtnh.ops.permute(t, list(range(t.shape().n_idx())), 0) if t.shape().split else t
        v = qtnh.ops.rebcast(u, self.rep)
        if u is not t:
            u.free()
        return v

    def _shard(self, t: Tensor, labels: List[str], avoid) -> Tuple[Optional[Tensor], List[str]]:
        """Distribute open indices of t (product = P) over the world; None if the
        labels do not allow it."""
        P, pick, prod = self.world, [], 1
        for i, lab in enumerate(labels):
            if lab in avoid or prod * self.dims[lab] > P:
                continue
            pick.append(i)
            prod *= self.dims[lab]
            if prod == P:
                break
        if prod != P:
            return None, labels
        perm = pick + [i for i in range(len(labels)) if i not in pick]
        one = qtnh.ops.rebcast(t, qtnh.DistParams(1, 1, 0))
        out = qtnh.ops.permute(one, perm, len(pick))
        one.free()
        return out, [labels[i] for i in perm]

    def _big_first(self, la: List[str], lb: List[str]) -> bool:
        """Operand order of one step: the larger tensor goes first. contract()
        reads its first operand through the gather GEMM (layout permutation fused
        into the operand loads) and permutes the second into a dense K x N panel,
        so the big one is never copied; the result labels follow the order."""
        if not _BIG_FIRST:
            return False
        return sum(math.log2(self.dims[x]) for x in lb) > sum(math.log2(self.dims[x]) for x in la)

    def contract_pair(self, a: int, b: int, new_id: Optional[int] = None) -> int:
        la, lb = self.labels[a], self.labels[b]
        ta, tb = self.tensors[a], self.tensors[b]
        temps = []
        if self.world > 1:
            sa, sb = ta.shape().split, tb.shape().split
            if sb > 0 and sa == 0:  # the sharded operand goes first (its open indices lead the result)
                la, lb, ta, tb = lb, la, tb, ta
                sa, sb = sb, sa
            if sa > 0 and sb > 0:  # replicate the smaller, keep the larger sharded
                if int(np.prod(tb.shape().dims)) > int(np.prod(ta.shape().dims)):
                    la, lb, ta, tb = lb, la, tb, ta
                tb = self._replicate(tb)
                temps.append(tb)
                self.n_replicated += 1
            elif sa == 0:
                shared = set(la) & set(lb)
                flops = 8.0 * float(np.prod([self.dims[x] for x in la if x not in shared] or [1])) * \
                    float(np.prod([self.dims[x] for x in lb] or [1]))
                if flops >= self.shard_flops:
                    s_t, s_l = self._shard(ta, la, shared)
                    if s_t is not None:
                        ta, la = s_t, s_l
                        temps.append(s_t)
            if ta.shape().split > 0:
                self.n_sharded += 1
        elif self._big_first(la, lb):
            la, lb, ta, tb = lb, la, tb, ta
        shared = [x for x in la if x in lb]
        apos = [la.index(x) for x in shared]
        bpos = [lb.index(x) for x in shared]
        c = qtnh.contract(ta, tb, apos, bpos)
        for t in temps:
            t.free()
        new = [x for x in la if x not in shared] + [x for x in lb if x not in shared]
        self.tensors.pop(a).free()
        self.tensors.pop(b).free()
        del self.labels[a], self.labels[b]
        i = new_id if new_id is not None else self._next
        self._next = max(self._next, i + 1)
        self.tensors[i] = c
        self.labels[i] = new
        return i

    def contract_order_native(self, order: Sequence[Tuple[int, int]]) -> int:
        """The whole order in one native call (qtnh_contract_chain): positions are
        derived on the host from the labels, the C++ runtime runs the contractions
        back to back (single-rank networks; multi-rank ones use contract_order)."""
        from ._lib import i32_array

        ids = sorted(self.tensors)
        if ids != list(range(len(ids))) or self.world > 1:
            raise qtnh.InvalidArgument("contract_order_native needs ids 0..n-1 on a single rank")
        L = {k: list(v) for k, v in self.labels.items()}
        n = len(ids)
        ab, npairs, ap, bp = [], [], [], []
        for s, (a, b) in enumerate(order):
            if a not in L or b not in L:
                raise qtnh.InvalidArgument("order references consumed ids")
            la, lb = L.pop(a), L.pop(b)
            if self._big_first(la, lb):
                a, b, la, lb = b, a, lb, la
            sh = [x for x in la if x in lb]
            ab += [a, b]
            npairs.append(len(sh))
            ap += [la.index(x) for x in sh]
            bp += [lb.index(x) for x in sh]
            L[n + s] = [x for x in la if x not in sh] + [x for x in lb if x not in sh]
        handles = (qtnh.C.c_void_p * n)(*[self.tensors[i]._h for i in ids])
        h = qtnh.C.c_void_p()
        qtnh.check(qtnh.lib.qtnh_contract_chain(n, handles, len(order), i32_array(ab or [0]),
                                                i32_array(npairs or [0]), i32_array(ap or [0]), i32_array(bp or [0]),
                                                qtnh.C.byref(h)))
        last = n + len(order) - 1
        result = Tensor(self.rank, h)
        for i in ids:
            self.tensors.pop(i).free()
        self.labels = {last: L[last]}
        self.tensors = {last: result}
        self._next = last + 1
        return last

    def contract_order(self, order: Sequence[Tuple[int, int]]) -> int:
        nxt = max(self.tensors) + 1
        last = None
        for s, (a, b) in enumerate(order):
            if a not in self.tensors or b not in self.tensors:
                raise qtnh.InvalidArgument("order references consumed ids")
            last = self.contract_pair(a, b, nxt + s)
        return last


# ---- config 3: random circuit on a grid as a tensor network ---------------------------------
def grid_pairs(pattern: str, rows: int, cols: int) -> List[Tuple[int, int]]:
    """Entangling patterns: A/B horizontal (row parity
    alternating), C/D vertical (column parity alternating); sites row-major."""
    out = []
    if pattern in "AB":
        for r in range(rows):
            c0 = (r + (0 if pattern == "A" else 1)) % 2
            for c in range(c0, cols - 1, 2):
                out.append((r * cols + c, r * cols + c + 1))
    else:
        for c in range(cols):
            r0 = (c + (0 if pattern == "C" else 1)) % 2
            for r in range(r0, rows - 1, 2):
                out.append((r * cols + c, (r + 1) * cols + c))
    return out


def rcs_grid_circuit(rows: int, cols: int, depth: int, seed: int):
    """Per layer: one of {sqrt X, sqrt Y, sqrt W} per qubit by
    hash_counter(seed, layer, qubit) % 3, then fSim on the layer's pattern in the
    cyclic order ABCDCDAB."""
    seq = "ABCDCDAB"
    gates = []
    for layer in range(depth):
        for q in range(rows * cols):
            gates.append(("1q", (q,), circuits.hash_counter(seed, layer, q) % 3))
        for a, b in grid_pairs(seq[layer % len(seq)], rows, cols):
            gates.append(("fsim", (a, b), None))
    return gates


def output_bits(n: int, n_open: int, seed: int):
    """Which qubits stay open (n_open of them, seeded) and the fixed bit of the rest."""
    order = circuits.fisher_yates(seed, 11, n)
    open_q = sorted(order[:n_open])
    fixed = {q: circuits.hash_counter(seed, 12, q) % 2 for q in range(n) if q not in open_q}
    return open_q, fixed


def rcs_network_spec(rows: int, cols: int, depth: int, seed: int, n_open: int = 6):
    """Host description of config 3's network: [(array, labels)] in insertion order,
    the open labels (ascending qubit), the open qubits and the fixed output bits."""
    from .mps import SINGLE_QUBIT

    n = rows * cols
    items = []
    wire = [f"q{q}.0" for q in range(n)]
    ver = [0] * n
    for q in range(n):
        items.append((np.array([1, 0], complex), [wire[q]]))
    for kind, qs, g in rcs_grid_circuit(rows, cols, depth, seed):
        if kind == "1q":
            q = qs[0]
            ver[q] += 1
            new = f"q{q}.{ver[q]}"
            items.append((SINGLE_QUBIT[g], [new, wire[q]]))  # (out, in)
            wire[q] = new
        else:
            a, b = qs
            ver[a] += 1
            ver[b] += 1
            na, nb = f"q{a}.{ver[a]}", f"q{b}.{ver[b]}"
            items.append((circuits.FSIM.reshape(2, 2, 2, 2), [na, nb, wire[a], wire[b]]))
            wire[a], wire[b] = na, nb
    open_q, fixed = output_bits(n, n_open, seed)
    for q, bit in fixed.items():
        v = np.zeros(2, complex)
        v[bit] = 1
        items.append((v, [wire[q]]))
    return items, [wire[q] for q in open_q], open_q, fixed


def build_rcs_network(rank: qtnh.Rank, rows: int, cols: int, depth: int, seed: int, n_open: int = 6,
                      shard_flops: float = 1e11):
    net = Network(rank, shard_flops)
    items, open_labels, open_q, fixed = rcs_network_spec(rows, cols, depth, seed, n_open)
    for arr, labs in items:
        net.add(arr, labs)
    return net, open_labels, open_q, fixed
