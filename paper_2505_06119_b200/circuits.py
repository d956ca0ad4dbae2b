"""Host-side workload generators for the benchmark configurations.

Gate matrices follow PAPER.md:95-151 (H, CZ(theta), sqrt X / sqrt Y / sqrt W, fSim);
the QFT gate order follows PAPER.md Fig. 1 / SPEC.md:597-608 (unitary 1/sqrt(2^n)
convention of SPEC.md:666). Seeded inputs use the reference's counter-based hash
and Box-Muller (common.hpp:83-146) through libqtnh_b200's host generators.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import List, Sequence, Tuple

import numpy as np

from ._lib import lib
from . import qtnh

R2 = 1.0 / np.sqrt(2.0)
H = np.array([[R2, R2], [R2, -R2]], dtype=np.complex128)
SQRT_X = R2 * np.array([[1, -1j], [-1j, 1]], dtype=np.complex128)
SQRT_Y = R2 * np.array([[1, -1], [1, 1]], dtype=np.complex128)
SQRT_W = R2 * np.array([[1, -np.sqrt(1j)], [np.sqrt(-1j), 1]], dtype=np.complex128)
FSIM = np.array([[1, 0, 0, 0], [0, 0, -1j, 0], [0, -1j, 0, 0], [0, 0, 0, np.exp(-1j * np.pi / 6)]],
                dtype=np.complex128)
SWAP = np.array([[1, 0, 0, 0], [0, 0, 1, 0], [0, 1, 0, 0], [0, 0, 0, 1]], dtype=np.complex128)


def cp_diag(theta: float) -> np.ndarray:
    """Diagonal of CZ(theta) = diag(1, 1, 1, e^{i theta})."""
    return np.array([1, 1, 1, np.exp(1j * theta)], dtype=np.complex128)


def qft_gates(n: int, swaps: bool = True) -> List[Tuple[str, tuple, np.ndarray]]:
    """QFT gate list: ('h', (j,), H), ('cp', (j+m-1, j), diag), ('swap', (j, n-1-j), None)."""
    gates = []
    for j in range(n):
        gates.append(("h", (j,), H))
        for m in range(2, n - j + 1):
            theta = 2.0 * np.pi / (2.0 ** m)
            gates.append(("cp", (j + m - 1, j), cp_diag(theta)))
    if swaps:
        for j in range(n // 2):
            gates.append(("swap", (j, n - 1 - j), None))
    return gates


def counter_state(seed: int, n_amp: int, start: int = 0, threads: int = 0) -> np.ndarray:
    """Counter-based complex normals (bit-identical to the reference's hash_counter
    + glibc Box-Muller), element j independent of the others."""
    out = np.empty(n_amp, dtype=np.complex128)
    threads = threads or min(32, os.cpu_count() or 1)
    lib.qtnh_counter_complex_normals(seed, start, n_amp, out.ctypes.data, threads)
    return out


def rng_normals(seed: int, count: int) -> np.ndarray:
    """One sequential Rng(seed).next_complex_normal() stream (common.hpp:109-140)."""
    out = np.empty(count, dtype=np.complex128)
    lib.qtnh_rng_complex_normals(seed, count, out.ctypes.data)
    return out


def hash_counter(seed: int, k0: int = 0, k1: int = 0, k2: int = 0) -> int:
    return int(lib.qtnh_hash_counter(seed, k0, k1, k2))


def u64_to_unit(u: int) -> float:
    """common.hpp:103-105: top 53 bits -> [0, 1)."""
    return float(u >> 11) * 2.0**-53


def fisher_yates(seed: int, tag: int, r: int) -> List[int]:
    """Seeded Fisher-Yates on hash_counter(seed, tag, i) (test_ops.cpp:124-129)."""
    p = list(range(r))
    for i in range(r - 1, 0, -1):
        j = hash_counter(seed, tag, i) % (i + 1)
        p[i], p[j] = p[j], p[i]
    return p


def contraction_positions(seed: int, rank_a: int, rank_b: int, k: int):
    """C1: the k contracted positions of A and of B by seeded Fisher-Yates, paired in
    sorted order."""
    ap = sorted(fisher_yates(seed, 8, rank_a)[:k])
    bp = sorted(fisher_yates(seed + 1, 8, rank_b)[:k])
    return ap, bp


def apply_qft(state: "qtnh.Tensor", n: int, swaps: bool = True) -> "qtnh.Tensor":
    """Run the QFT gate sequence on a state tensor (qubit j = tuple index j).
    H: dense 1-qubit gate kernel; CP: diagonal kernel (touches 1/4 of the state);
    final SWAPs: index permutations (contracting a swap tensor is a pure exchange of
    two indices, tensor.hpp:157-164)."""
    split = state.shape().split
    original = state
    for kind, q, g in qft_gates(n, swaps):
        if kind == "h":
            qtnh.apply_gate(state, q, g)
        elif kind == "cp":
            qtnh.apply_gate(state, q, g, diagonal=True)
        else:
            perm = list(range(n))
            perm[q[0]], perm[q[1]] = perm[q[1]], perm[q[0]]
            nxt = qtnh.ops.permute(state, perm, split)
            if state is not original:
                state.free()
            state = nxt
    return state


def apply_qft_fused(state: "qtnh.Tensor", n: int, swaps: bool = True) -> "qtnh.Tensor":
    """QFT with one fused pass per layer (H_j + all its controlled phases,
    qtnh.qft_layer) and in-place qubit swaps: n + n/2 passes instead of
    n(n+1)/2 + n/2. Same values as apply_qft up to rounding."""
    for j in range(n):
        qtnh.qft_layer(state, j)
    if swaps:
        for j in range(n // 2):
            qtnh.swap_indices(state, j, n - 1 - j)
    return state


# ---- gate fusion (grouping gates cuts state passes) -------------------
def _embed(block_qubits: List[int], gate_qubits: Sequence[int], g: np.ndarray) -> np.ndarray:
    """The 2^k x 2^k matrix of gate g (on gate_qubits, first most significant) acting on
    the block's qubits (sorted, first most significant)."""
    k, kg = len(block_qubits), len(gate_qubits)
    t = np.eye(2**k, dtype=np.complex128).reshape([2] * (2 * k))
    pos = [block_qubits.index(q) for q in gate_qubits]
    gt = np.asarray(g, dtype=np.complex128).reshape([2] * (2 * kg))
    # out[o..] = sum_i g[o_pos, i_pos] t[i_pos..]
    t = np.tensordot(gt, t, axes=(list(range(kg, 2 * kg)), pos))
    rest = [a for a in range(2 * k) if a not in pos]
    order = pos + rest  # current axis order of t in terms of original axes
    return np.transpose(t, np.argsort(order)).reshape(2**k, 2**k)


class FusedGate:
    __slots__ = ("qubits", "matrix", "diagonal", "count")

    def __init__(self, qubits, matrix, count):
        self.qubits = list(qubits)
        self.matrix = matrix
        self.count = count
        off = matrix - np.diag(np.diag(matrix))
        self.diagonal = not np.any(off)


def fuse_gates(gates: Sequence[Tuple[Sequence[int], np.ndarray]], max_qubits: int = 4) -> List[FusedGate]:
    """Group a gate sequence into blocks of at most `max_qubits` qubits (the dense gate
    kernel's D <= 16), preserving the circuit's action: every qubit belongs to at most
    one open block; a gate merges all open blocks it touches when the union fits,
    otherwise those blocks are emitted and the gate opens a new block. Blocks on
    disjoint qubits commute, so emission order only follows shared qubits. Each
    fused block costs one state pass instead of one per gate (diagonal blocks touch
    only their non-unit entries)."""
    out: List[FusedGate] = []
    open_of: dict = {}  # qubit -> block id
    blocks: dict = {}   # id -> [qubits(sorted), matrix, count]
    nid = 0

    def close(bid):
        qs, m, c = blocks.pop(bid)
        for q in qs:
            open_of.pop(q, None)
        out.append(FusedGate(qs, m, c))

    for qs, g in gates:
        qs = [int(q) for q in qs]
        if len(set(qs)) != len(qs):
            raise ValueError("gate with repeated qubits")
        touching = sorted({open_of[q] for q in qs if q in open_of})
        union = sorted(set(qs).union(*[blocks[b][0] for b in touching]))
        if len(qs) > max_qubits:
            for b in touching:
                close(b)
            out.append(FusedGate(qs, np.asarray(g, dtype=np.complex128).reshape(2 ** len(qs), -1), 1))
            continue
        if len(union) <= max_qubits:
            m = np.eye(2 ** len(union), dtype=np.complex128)
            c = 0
            for b in touching:  # disjoint open blocks commute: any order
                bq, bm, bc = blocks.pop(b)
                m = _embed(union, bq, bm) @ m
                c += bc
            m = _embed(union, qs, g) @ m
            blocks[nid] = [union, m, c + 1]
            for q in union:
                open_of[q] = nid
            nid += 1
        else:
            for b in touching:
                close(b)
            blocks[nid] = [sorted(qs), _embed(sorted(qs), qs, g), 1]
            for q in qs:
                open_of[q] = nid
            nid += 1
    for b in sorted(blocks):
        close(b)
    return out


def apply_fused(state: "qtnh.Tensor", fused: Sequence[FusedGate]) -> "qtnh.Tensor":
    """Apply fused blocks with the dense (D <= 16) or diagonal gate kernels."""
    for f in fused:
        if f.diagonal:
            qtnh.apply_gate(state, f.qubits, np.diag(f.matrix).copy(), diagonal=True)
        else:
            qtnh.apply_gate(state, f.qubits, f.matrix.reshape(-1))
    return state
