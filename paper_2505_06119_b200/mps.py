"""Config 4 driver: random-circuit evolution of a matrix product state with the
two-site update (contract two sites, apply the 2-qubit gate, truncated SVD with
the singular values absorbed into the left factor) -- SURVEY.md 3.3 / SPEC
apply_raw_gate, built only from the library's hot-path ops:
qtnh.contract (DMMA zgemm), qtnh.apply_gate, qtnh.svd (batched Jacobi SVD).

Sites are rank-3 tensors (chi_left, d, chi_right). Bond dimensions grow up to
chi and are then truncated to exactly chi; the reference's fixed-chi storage
(zero-padded to chi from the start, linalg.hpp:476-505) holds the same values
plus zeros, so amplitudes and fidelities are identical.
"""
from __future__ import annotations

import ctypes as C
from typing import List, Sequence, Tuple

import numpy as np

from . import circuits, qtnh
from .qtnh import ABSORB_LEFT, IndexTuple, Tensor

SINGLE_QUBIT = [circuits.SQRT_X, circuits.SQRT_Y, circuits.SQRT_W]


def rcs_1d_layers(n: int, depth: int, seed: int, no_repeat: bool = False):
    """1-D nearest-neighbour brickwork of the RCS gate set:
    per layer one of {sqrt X, sqrt Y, sqrt W} per qubit chosen by
    hash_counter(seed, layer, qubit) % 3, then fSim on pairs
    (0,1),(2,3),... on even layers and (1,2),(3,4),... on odd layers."""
    layers = []
    prev = [-1] * n
    for layer in range(depth):
        singles = []
        for q in range(n):
            g = circuits.hash_counter(seed, layer, q) % 3
            if no_repeat and g == prev[q]:
                g = (g + 1 + circuits.hash_counter(seed, layer, q, 1) % 2) % 3
            prev[q] = g
            singles.append(g)
        start = layer % 2
        pairs = [(q, q + 1) for q in range(start, n - 1, 2)]
        layers.append((singles, pairs))
    return layers


class MPS:
    def __init__(self, rank: qtnh.Rank, n: int, chi: int, d: int = 2):
        self.rank, self.n, self.chi, self.d = rank, n, chi, d
        self.sites: List[Tensor] = []
        self.log_fidelity = 0.0
        self.discarded = []
        for _ in range(n):  # |0...0>, bond dimension 1
            v = np.zeros(d, dtype=np.complex128)
            v[0] = 1.0
            self.sites.append(Tensor.from_global(rank, IndexTuple([1, d, 1], 0), None, v))

    def apply_1q(self, q: int, g: np.ndarray) -> None:
        qtnh.apply_gate(self.sites[q], [1], g)

    def apply_2q(self, q: int, g: np.ndarray) -> Tuple[np.ndarray, float]:
        """Two-site update on sites (q, q+1); returns (kept singular values, kept
        weight fraction)."""
        a, b = self.sites[q], self.sites[q + 1]
        theta = qtnh.contract(a, b, [2], [0])  # (l, d, d, r): open(a) then open(b)
        qtnh.apply_gate(theta, [1, 2], g)
        sh = theta.shape().dims
        k = min(sh[0] * sh[1], sh[2] * sh[3])
        keep = min(self.chi, k)
        # one full SVD; the kept weight comes from its spectrum, then slice to chi
        u, s, vh = qtnh.svd(theta, [0, 1], [2, 3], chi=k, absorb=ABSORB_LEFT)
        frac = 1.0
        if keep < k:
            tot = float(np.sum(s**2))
            frac = float(np.sum(s[:keep] ** 2)) / tot if tot > 0 else 1.0
            self.log_fidelity += np.log(frac)
            u2 = qtnh.ops.slice_local_dims(u, [sh[0], sh[1], keep])
            vh2 = qtnh.ops.slice_local_dims(vh, [keep, sh[2], sh[3]])
            u.free()
            vh.free()
            u, vh, s = u2, vh2, s[:keep]
        theta.free()
        a.free()
        b.free()
        self.sites[q], self.sites[q + 1] = u, vh
        return s, frac

    def apply_layer(self, pairs: Sequence[Tuple[int, int]], g: np.ndarray) -> List[Tuple[np.ndarray, float]]:
        """Two-site updates of disjoint pairs, with every group of equal-shape thetas
        factorised by ONE batched Jacobi SVD launch sequence (qtnh_svd_device)."""
        import torch

        thetas = []
        for (q, _) in pairs:
            th = qtnh.contract(self.sites[q], self.sites[q + 1], [2], [0])
            qtnh.apply_gate(th, [1, 2], g)
            thetas.append((q, th, th.shape().dims))
        groups: dict = {}
        for q, th, sh in thetas:
            groups.setdefault(tuple(sh), []).append((q, th))
        results = {}
        dev = torch.device("cuda")
        for sh, items in groups.items():
            l, d1, d2, r = sh
            m, n = l * d1, d2 * r
            k = min(m, n)
            keep = min(self.chi, k)
            bsz = len(items)
            a = torch.empty((bsz, m, n), dtype=torch.complex128, device=dev)
            for i, (q, th) in enumerate(items):
                src = torch.as_tensor(_DevView(th.device_ptr(), m * n), device=dev)
                a[i].view(-1).copy_(src)
            u = torch.empty((bsz, m, k), dtype=torch.complex128, device=dev)
            s = torch.empty((bsz, k), dtype=torch.float64, device=dev)
            vh = torch.empty((bsz, k, n), dtype=torch.complex128, device=dev)
            qtnh.check(qtnh.lib.qtnh_svd_device(self.rank._h, bsz, m, n, C.c_void_p(a.data_ptr()), k, ABSORB_LEFT,
                                                C.c_void_p(u.data_ptr()), C.c_void_p(s.data_ptr()),
                                                C.c_void_p(vh.data_ptr())))
            s_h = s.cpu().numpy()
            for i, (q, th) in enumerate(items):
                frac = 1.0
                if keep < k:
                    tot = float(np.sum(s_h[i] ** 2))
                    frac = float(np.sum(s_h[i][:keep] ** 2)) / tot if tot > 0 else 1.0
                    self.log_fidelity += np.log(frac)
                ui = u[i, :, :keep].contiguous()
                vi = vh[i, :keep, :].contiguous()
                nu = Tensor.from_device(self.rank, IndexTuple([l, d1, keep], 0), None, ui.data_ptr())
                nv = Tensor.from_device(self.rank, IndexTuple([keep, d2, r], 0), None, vi.data_ptr())
                self.rank.synchronize()  # the torch temporaries die at the end of the loop
                self.sites[q].free()
                self.sites[q + 1].free()
                self.sites[q], self.sites[q + 1] = nu, nv
                th.free()
                results[q] = (s_h[i][:keep], frac)
        return [results[q] for (q, _) in pairs]

    def bond_dims(self) -> List[int]:
        return [t.shape().dims[2] for t in self.sites[:-1]]

    def amplitudes(self, bitstrings: np.ndarray) -> np.ndarray:
        """<b|psi> for each row of `bitstrings` (n bits, qubit 0 first): a left-to-
        right chain of (batch x chi) x (chi x chi) products on the GPU, the batch
        split by the bit value at each site (two zgemms per site)."""
        import torch

        B = bitstrings.shape[0]
        dev = torch.device("cuda")
        env = torch.ones((B, 1), dtype=torch.complex128, device=dev)
        for q in range(self.n):
            t = self.sites[q]
            l, d, r = t.shape().dims
            site = torch.as_tensor(_DevView(t.device_ptr(), l * d * r), device=dev).reshape(l, d, r)
            new = torch.empty((B, r), dtype=torch.complex128, device=dev)
            for bit in range(d):
                idx = np.nonzero(bitstrings[:, q] == bit)[0]
                if idx.size == 0:
                    continue
                ti = torch.from_numpy(idx).to(dev)
                lhs = env.index_select(0, ti).contiguous()
                mat = site[:, bit, :].contiguous()
                out = torch.empty((idx.size, r), dtype=torch.complex128, device=dev)
                qtnh.check(qtnh.lib.qtnh_zgemm_device(self.rank._h, idx.size, r, l, C.c_void_p(lhs.data_ptr()),
                                                      C.c_void_p(mat.data_ptr()), C.c_void_p(out.data_ptr())))
                new.index_copy_(0, ti, out)
            env = new
        torch.cuda.synchronize()
        return env[:, 0].cpu().numpy()

    def free(self):
        for t in self.sites:
            t.free()


class _DevView:
    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<c16", "data": (ptr, False), "version": 3}


def run_rcs_mps(rank: qtnh.Rank, n: int, depth: int, chi: int, seed: int, layers=None, timer=None,
                batched: bool = True):
    """Evolve |0..0> through the 1-D RCS brickwork; returns the MPS and per-update
    records (layer, pair, kept fraction)."""
    import torch

    rank.set_stream(torch.cuda.current_stream().cuda_stream)
    m = MPS(rank, n, chi)
    layers = layers if layers is not None else rcs_1d_layers(n, depth, seed)
    recs = []
    for li, (singles, pairs) in enumerate(layers):
        for q, g in enumerate(singles):
            m.apply_1q(q, SINGLE_QUBIT[g])
        if batched:
            for (q, _), (s, frac) in zip(pairs, m.apply_layer(pairs, circuits.FSIM)):
                recs.append((li, q, frac, s))
        else:
            for (q, q1) in pairs:
                s, frac = m.apply_2q(q, circuits.FSIM)
                recs.append((li, q, frac, s))
    return m, recs
