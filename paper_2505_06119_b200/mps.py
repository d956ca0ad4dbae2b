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
import os
from typing import List, Sequence, Tuple

import numpy as np

from . import circuits, qtnh
from .qtnh import ABSORB_LEFT, ABSORB_RIGHT, IndexTuple, Tensor

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
        self.centre = None
        self.dist = None  # DistParams of the site tensors (DistMPS: the owning rank)
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
        """Two-site updates of disjoint pairs in ONE native call (qtnh_mps_apply_layer,
        csrc/mps.cu): thetas formed by zgemm straight into the batched-SVD buffer, the
        gate in place, every group of equal-shape thetas factorised by one batched
        Jacobi SVD whose outputs are the new site tensors; no torch, no per-update
        synchronisation. Returns (kept singular values, kept weight fraction) per pair."""
        n = len(pairs)
        if n == 0:
            return []
        left = (C.c_void_p * n)(*[self.sites[q]._h for q, _ in pairs])
        right = (C.c_void_p * n)(*[self.sites[q + 1]._h for q, _ in pairs])
        nl, nr = (C.c_void_p * n)(), (C.c_void_p * n)()
        gate = np.ascontiguousarray(g, dtype=np.complex128)
        s = np.zeros((n, self.chi), dtype=np.float64)
        keep = np.zeros(n, dtype=np.int64)
        nrm = np.zeros(n, dtype=np.float64)
        qtnh.check(qtnh.lib.qtnh_mps_apply_layer(n, left, right, gate.ctypes.data, self.chi, nl, nr, s.ctypes.data,
                                                 keep.ctypes.data, nrm.ctypes.data))
        out = []
        for i, (q, _) in enumerate(pairs):
            a, b = self.sites[q], self.sites[q + 1]
            l, d1, _ = a.shape().dims
            _, d2, r = b.shape().dims
            si = s[i, : keep[i]].copy()
            frac = 1.0
            if keep[i] < min(l * d1, d2 * r):  # truncated: kept weight of this update
                frac = float(np.sum(si**2)) / float(nrm[i]) if nrm[i] > 0 else 1.0
                self.log_fidelity += np.log(frac)
            a.free()
            b.free()
            self.sites[q], self.sites[q + 1] = Tensor(self.rank, C.c_void_p(nl[i])), Tensor(self.rank, C.c_void_p(nr[i]))
            out.append((si, frac))
        return out

    def bond_dims(self) -> List[int]:
        return [t.shape().dims[2] for t in self.sites[:-1]]

    # ---- SPEC mps operations either side of the two-site update ------------
    # All of them run on the device through the hot-path ops: qtnh.contract (DMMA zgemm),
    # qtnh.svd (Jacobi SVD), ops.conj / ops.scale. Bonds are stored at their effective
    # dimension; the reference's zero padding to chi adds only zeros, so
    # every quantity below is identical.

    @classmethod
    def bitstring(cls, rank: qtnh.Rank, bits: Sequence[int], chi: int, d: int = 2) -> "MPS":
        """mps_bitstring: amplitude 1 on `bits`, bond dimension 1."""
        m = cls(rank, len(bits), chi, d)
        for q, b in enumerate(bits):
            if not 0 <= int(b) < d:
                raise qtnh.InvalidArgument("bit value outside the physical dimension")
            v = np.zeros(d, dtype=np.complex128)
            v[int(b)] = 1.0
            m.sites[q].free()
            m.sites[q] = Tensor.from_global(rank, IndexTuple([1, d, 1], 0), None, v)
        return m

    @classmethod
    def random(cls, rank: qtnh.Rank, n: int, chi_eff: int, seed: int, chi: int = 0, d: int = 2) -> "MPS":
        """mps_random: seeded complex normal sites with effective bond
        dimension min(chi_eff, d^q, d^(n-q)) at bond q, normalised to norm2 = 1. Site q
        draws from the counter-based stream (seed, q) of common.hpp."""
        chi = chi or chi_eff
        if chi_eff > chi:
            raise qtnh.InvalidArgument("chi_eff exceeds chi")
        m = cls(rank, n, chi, d)
        bonds = [1] + [min(chi_eff, d ** (q + 1), d ** (n - q - 1)) for q in range(n - 1)] + [1]
        for q in range(n):
            l, r = bonds[q], bonds[q + 1]
            v = circuits.counter_state(circuits.hash_counter(seed, 31, q), l * d * r)
            m.sites[q].free()
            m.sites[q] = Tensor.from_global(rank, IndexTuple([l, d, r], 0), None, v)
        m.renormalise()
        return m

    def _set(self, q: int, t: Tensor) -> None:
        self.sites[q].free()
        self.sites[q] = t

    def canonicalize(self, centre: int) -> "MPS":
        """Mixed canonical form at `centre`: sites left of it are
        left-orthonormal (U of an SVD over (left, phys) x right, S Vh pushed right),
        sites right of it right-orthonormal (Vh, U S pushed left). No truncation, so
        the statevector is unchanged up to rounding."""
        if not 0 <= centre < self.n:
            raise qtnh.InvalidArgument("canonical centre outside the chain")
        for q in range(centre):
            u, sv, svh = qtnh.svd(self.sites[q], [0, 1], [2], absorb=ABSORB_RIGHT)
            u, svh = self._drop_null(u, svh, sv)
            nxt = qtnh.contract(svh, self.sites[q + 1], [1], [0])  # (k, d, r)
            svh.free()
            self._set(q, u)
            self._set(q + 1, nxt)
        for q in range(self.n - 1, centre, -1):
            us, sv, vh = qtnh.svd(self.sites[q], [0], [1, 2], absorb=ABSORB_LEFT)
            us, vh = self._drop_null(us, vh, sv)
            prv = qtnh.contract(self.sites[q - 1], us, [2], [0])  # (l, d, k)
            us.free()
            self._set(q, vh)
            self._set(q - 1, prv)
        self.centre = centre
        return self

    @staticmethod
    def _drop_null(u: Tensor, vh: Tensor, sv: np.ndarray) -> Tuple[Tensor, Tensor]:
        """Drop the singular triplets with sigma <= 1e-13 sigma_max from a split: the
        Jacobi SVD returns zero vectors for a null space (no orthonormal completion),
        so a rank-deficient site keeps its isometry (A A^H = I) only on
        the bond's effective rank. The dropped directions carry no weight."""
        k = sv.size
        keep = max(1, int(np.sum(sv > 1e-13 * sv[0]))) if k and sv[0] > 0 else max(1, k)
        if keep == k:
            return u, vh
        ud, vd = u.shape().dims, vh.shape().dims
        u2 = qtnh.ops.slice_local_dims(u, ud[:-1] + [keep])
        v2 = qtnh.ops.slice_local_dims(vh, [keep] + vd[1:])
        u.free()
        vh.free()
        return u2, v2

    def overlap(self, other: "MPS") -> complex:
        """<other|self> by the transfer-matrix contraction left to right:
        E(a, b) <- sum over (a, s, b) of E(a, b) A_s(a, a') conj(B_s(b, b'))."""
        if other.n != self.n or other.d != self.d:
            raise qtnh.InvalidArgument("overlap needs MPS of equal length and physical dimension")
        env = Tensor.from_global(self.rank, IndexTuple([1, 1], 0), self.dist, np.ones(1, dtype=np.complex128))
        for q in range(self.n):
            t1 = qtnh.contract(env, self.sites[q], [0], [0])  # (b, s, a')
            bc = qtnh.ops.conj(other.sites[q])
            env.free()
            env = qtnh.contract(t1, bc, [0, 1], [0, 1])  # (a', b')
            t1.free()
            bc.free()
        out = complex(env.to_global_vector()[0])
        env.free()
        return out

    def norm2(self) -> float:
        """overlap(m, m).real."""
        return float(self.overlap(self).real)

    def renormalise(self) -> "MPS":
        """Scale every site by the same factor so norm2 = 1;
        DegenerateStateError for a zero state."""
        n2 = self.norm2()
        if not n2 > 0.0:
            raise qtnh.DegenerateStateError("renormalise of a zero-norm MPS")
        f = n2 ** (-0.5 / self.n)
        for q in range(self.n):
            self._set(q, qtnh.ops.scale(self.sites[q], f))
        return self

    def effective_bond_dims(self, tol: float = 1e-12) -> List[int]:
        """Per-bond count of Schmidt values above tol: right-canonical
        form, then the centre walks right and each bond's SVD gives its spectrum."""
        self.canonicalize(0)
        out = []
        for q in range(self.n - 1):
            u, sv, svh = qtnh.svd(self.sites[q], [0, 1], [2], absorb=ABSORB_RIGHT)
            out.append(int(np.sum(sv > tol)))
            nxt = qtnh.contract(svh, self.sites[q + 1], [1], [0])
            svh.free()
            self._set(q, u)
            self._set(q + 1, nxt)
        self.centre = self.n - 1
        return out

    def sample(self, sites: Sequence[int], seed: int, draw: int = 0) -> List[int]:
        """One draw from the marginal on `sites`: right-canonical form,
        then sequential conditional sampling left to right over ALL sites (SPEC design
        decision), the requested subset projected from the full draw.
        Site q's uniform is u64_to_unit(hash_counter(seed, draw, q))."""
        n2 = self.norm2()
        if abs(n2 - 1.0) > 1e-8:
            raise qtnh.PreconditionError("sample needs a normalised MPS (norm2 = %.3e)" % n2)
        self.canonicalize(0)
        env = Tensor.from_global(self.rank, IndexTuple([1], 0), self.dist, np.ones(1, dtype=np.complex128))
        bits = []
        for q in range(self.n):
            v = qtnh.contract(env, self.sites[q], [0], [0])  # (d, r)
            d, r = v.shape().dims
            vh = v.to_global_vector().reshape(d, r)
            v.free()
            p = np.sum(np.abs(vh) ** 2, axis=1)
            tot = float(np.sum(p))
            u = circuits.u64_to_unit(circuits.hash_counter(seed, draw, q)) * tot
            s = int(min(np.searchsorted(np.cumsum(p), u, side="right"), d - 1))
            while p[s] == 0.0 and s > 0:  # never collapse onto a zero-probability outcome
                s -= 1
            bits.append(s)
            env.free()
            env = Tensor.from_global(self.rank, IndexTuple([r], 0), self.dist, vh[s] / np.sqrt(p[s]))
        env.free()
        return [bits[q] for q in sites]

    def _reshape(self, t: Tensor, dims: Sequence[int]) -> Tensor:
        """Same row-major values under new dims (one device copy)."""
        out = Tensor.from_device(self.rank, IndexTuple(list(dims), 0), self.dist, t.device_ptr())
        t.free()
        return out

    def _split_range(self, theta: Tensor, first: int, last: int, chi: int) -> None:
        """Write theta (l, d x (last-first+1), r) back as sites first..last by
        repeated SVDs truncated to chi (S pushed right, kept-weight into
        log_fidelity), then move the centre back to `first`."""
        for q in range(first, last):
            dims = theta.shape().dims
            m = dims[0] * dims[1]
            k = min(m, int(np.prod(dims[2:])))
            keep = min(chi, k)
            u, sv, rest = qtnh.svd(theta, [0, 1], list(range(2, len(dims))), chi=k, absorb=ABSORB_RIGHT)
            theta.free()
            if keep < k:
                tot = float(np.sum(sv**2))
                if tot > 0:
                    self.log_fidelity += np.log(float(np.sum(sv[:keep] ** 2)) / tot)
                u2 = qtnh.ops.slice_local_dims(u, [dims[0], dims[1], keep])
                r2 = qtnh.ops.slice_local_dims(rest, [keep] + list(dims[2:]))
                u.free()
                rest.free()
                u, rest = u2, r2
            self._set(q, u)
            theta = rest
        self._set(last, theta)
        for q in range(last, first, -1):
            us, _, vh = qtnh.svd(self.sites[q], [0], [1, 2], absorb=ABSORB_LEFT)
            prv = qtnh.contract(self.sites[q - 1], us, [2], [0])
            us.free()
            self._set(q, vh)
            self._set(q - 1, prv)
        self.centre = first

    def apply_gate_sites(self, targets: Sequence[int], gate: np.ndarray) -> "MPS":
        """apply_raw_gate: contract the inclusive site range of the
        sorted targets into one tensor, apply the gate there (identities on the
        intermediate sites), re-decompose by repeated SVD truncated to chi, and leave
        the canonical centre at the first target."""
        targets = [int(t) for t in targets]
        if targets != sorted(set(targets)) or not targets or targets[0] < 0 or targets[-1] >= self.n:
            raise qtnh.InvalidArgument("apply_raw_gate needs sorted distinct targets inside the chain")
        g = np.asarray(gate, dtype=np.complex128)
        D = self.d ** len(targets)
        if g.size != D * D:
            raise qtnh.InvalidArgument("gate dimension does not match the number of targets")
        first, last = targets[0], targets[-1]
        theta = qtnh.contract(self.sites[first], self.sites[first + 1], [2], [0]) if last > first else None
        if theta is None:
            theta = qtnh.ops.scale(self.sites[first], 1.0)
        for q in range(first + 2, last + 1):
            nxt = qtnh.contract(theta, self.sites[q], [theta.shape().n_idx() - 1], [0])
            theta.free()
            theta = nxt
        qtnh.apply_gate(theta, [1 + t - first for t in targets], g.reshape(-1))
        self._split_range(theta, first, last, self.chi)
        return self

    def apply_mpo(self, mpo: Sequence[np.ndarray], first: int = 0) -> "MPS":
        """apply_mpo: MPO sites W (wl, d_out, d_in, wr) on the
        contiguous support first..first+len-1; each MPS site becomes
        (l wl, d_out, r wr) = sum_{d_in} A(l, d_in, r) W(wl, d_out, d_in, wr), then one
        left-canonical sweep and a right-to-left compression sweep back to chi, centre
        restored at the first MPO site."""
        if first < 0 or first + len(mpo) > self.n:
            raise qtnh.InvalidArgument("MPO support outside the chain")
        for i, w in enumerate(mpo):
            w = np.asarray(w, dtype=np.complex128)
            if w.ndim != 4 or w.shape[1] != self.d or w.shape[2] != self.d:
                raise qtnh.InvalidArgument("MPO site needs shape (wl, d, d, wr) with the physical dimension")
            if (i == 0 and w.shape[0] != 1) or (i == len(mpo) - 1 and w.shape[3] != 1):
                raise qtnh.InvalidArgument("MPO boundary bonds must be 1")
            q = first + i
            a = self.sites[q]
            l, _, r = a.shape().dims
            wt = Tensor.from_global(self.rank, IndexTuple(list(w.shape), 0), self.dist, w.reshape(-1))
            c = qtnh.contract(a, wt, [1], [2])  # (l, r, wl, d_out, wr)
            wt.free()
            p = qtnh.ops.permute(c, [0, 2, 3, 1, 4], 0)  # (l, wl, d_out, r, wr)
            c.free()
            self._set(q, self._reshape(p, [l * w.shape[0], self.d, r * w.shape[3]]))
        # compression: left-canonical form, then truncating right-to-left sweep
        self.canonicalize(self.n - 1)
        for q in range(self.n - 1, 0, -1):
            dims = self.sites[q].shape().dims
            k = min(dims[0], dims[1] * dims[2])
            keep = min(self.chi, k)
            us, sv, vh = qtnh.svd(self.sites[q], [0], [1, 2], chi=k, absorb=ABSORB_LEFT)
            if keep < k:
                tot = float(np.sum(sv**2))
                if tot > 0:
                    self.log_fidelity += np.log(float(np.sum(sv[:keep] ** 2)) / tot)
                us2 = qtnh.ops.slice_local_dims(us, [dims[0], keep])
                vh2 = qtnh.ops.slice_local_dims(vh, [keep, dims[1], dims[2]])
                us.free()
                vh.free()
                us, vh = us2, vh2
            prv = qtnh.contract(self.sites[q - 1], us, [2], [0])
            us.free()
            self._set(q, vh)
            self._set(q - 1, prv)
        self.canonicalize(first)
        return self

    def to_statevector(self) -> np.ndarray:
        """mps_to_statevector, qubit 0 most significant; n <= 26."""
        if self.n > 26:
            raise qtnh.ResourceError("statevector of more than 26 sites", 0)
        acc = self.sites[0]
        owned = False
        for q in range(1, self.n):
            nxt = qtnh.contract(acc, self.sites[q], [acc.shape().n_idx() - 1], [0])
            if owned:
                acc.free()
            acc, owned = nxt, True
        out = acc.to_global_vector()
        if owned:
            acc.free()
        return out

    def amplitudes(self, bitstrings: np.ndarray) -> np.ndarray:
        """<b|psi> for each row of `bitstrings` (n bits, qubit 0 first): a left-to-
        right chain of (batch x chi) x (chi x chi) products on the GPU, the batch
        split by the bit value at each site (two zgemms per site)."""
        import torch

        B = bitstrings.shape[0]
        dev = torch.device("cuda")
        # The sites were written on the rank's stream; torch works on its current
        # stream. Drain the rank stream before torch reads, and launch the zgemms on
        # torch's stream for the duration (restored afterwards).
        self.rank.synchronize()
        prev = self.rank.stream_ptr()
        self.rank.set_stream(torch.cuda.current_stream().cuda_stream)
        try:
            return self._amplitudes_on_torch_stream(bitstrings, torch, dev, B)
        finally:
            torch.cuda.current_stream().synchronize()
            self.rank.set_stream(prev)

    def _amplitudes_on_torch_stream(self, bitstrings, torch, dev, B):
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


class DistMPS(MPS):
    """the chain's sites sharded over the world's ranks, rank r
    owning the contiguous range [lo, hi). A layer's two-site updates on pairs inside
    a range run as one batched SVD per rank; a pair straddling a boundary
    (q = hi - 1 here, q + 1 on rank r + 1) is computed here after one site exchange
    (Rank.exchange_tensors), and the new right site is sent back -- one exchange
    step per layer each way. Updates act on disjoint pairs, so the result equals the
    single-rank run (up to the batched SVD's rounding)."""

    def __init__(self, rank: qtnh.Rank, n: int, chi: int, d: int = 2):
        self.rank, self.n, self.chi, self.d = rank, n, chi, d
        P, r = rank.size(), rank.rank()
        if n < 2 * P:
            raise qtnh.InvalidArgument("DistMPS needs at least two sites per rank")
        self.lo, self.hi = (r * n) // P, ((r + 1) * n) // P
        self.log_fidelity = 0.0
        self.discarded = []
        self.centre = None
        self.dist = qtnh.DistParams(1, 1, r)  # every site lives on its owner alone
        self.sites = {}
        for q in range(self.lo, self.hi):
            v = np.zeros(d, dtype=np.complex128)
            v[0] = 1.0
            self.sites[q] = Tensor.from_global(rank, IndexTuple([1, d, 1], 0), self.dist, v)

    def apply_1q(self, q: int, g: np.ndarray) -> None:
        if self.lo <= q < self.hi:
            super().apply_1q(q, g)

    def apply_layer(self, pairs, g):
        r = self.rank.rank()
        qs = [q for (q, _) in pairs]
        inside = [(q, q + 1) for q in qs if self.lo <= q and q + 1 < self.hi]
        left = [(q, q + 1) for q in qs if q == self.hi - 1 and q + 1 < self.n]   # I compute
        right = [(q, q + 1) for q in qs if q + 1 == self.lo]                     # rank r-1 computes
        # pairwise collectives, the one with the left neighbour first: a rank that
        # meets both neighbours in one layer finishes with r - 1 before r + 1, so
        # the waits form a chain, never a cycle
        if right:
            self.rank.exchange_tensors({r - 1: self.sites[self.lo]}, [], self.dist)
        if left:
            self.sites[self.hi] = self.rank.exchange_tensors({}, [r + 1], self.dist)[r + 1]
        res = MPS.apply_layer(self, inside + left, g)
        if right:
            self.sites[self.lo].free()
            self.sites[self.lo] = self.rank.exchange_tensors({}, [r - 1], self.dist)[r - 1]
        if left:
            self.rank.exchange_tensors({r + 1: self.sites[self.hi]}, [], self.dist)
            self.sites.pop(self.hi).free()
        return res

    def bond_dims(self) -> List[int]:
        return [self.sites[q].shape().dims[2] for q in range(self.lo, self.hi) if q < self.n - 1]

    def local_sites(self):
        """{q: numpy array (l, d, r)} of the owned sites."""
        return {q: t.to_global_vector().reshape(t.shape().dims) for q, t in self.sites.items()}

    def free(self):
        for t in self.sites.values():
            t.free()


def mpo_from_operator(op: np.ndarray, k: int, d: int = 2) -> List[np.ndarray]:
    """Exact k-site MPO (wl, d_out, d_in, wr) of a d^k x d^k operator (row = output,
    site 0 most significant) by successive SVDs on the host (small operators)."""
    t = np.asarray(op, dtype=np.complex128).reshape([d] * (2 * k))
    # interleave (out_i, in_i) per site
    t = t.transpose([x for i in range(k) for x in (i, k + i)])
    sites, wl = [], 1
    rest = t.reshape(wl * d * d, -1)
    for i in range(k - 1):
        u, s, vh = np.linalg.svd(rest, full_matrices=False)
        r = int(np.sum(s > 1e-14 * s[0])) if s.size else 0
        sites.append(u[:, :r].reshape(wl, d, d, r))
        rest = (s[:r, None] * vh[:r]).reshape(r * d * d, -1)
        wl = r
    sites.append(rest.reshape(wl, d, d, 1))
    return sites


class _DevView:
    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<c16", "data": (ptr, False), "version": 3}


def run_rcs_mps(rank: qtnh.Rank, n: int, depth: int, chi: int, seed: int, layers=None, timer=None,
                batched: bool = True, distributed: bool = False):
    """Evolve |0..0> through the 1-D RCS brickwork; returns the MPS and per-update
    records (layer, pair, kept fraction). `distributed`: sites sharded over the
    world's ranks (DistMPS); records then cover the pairs this rank computed."""
    import torch

    rank.set_stream(torch.cuda.current_stream().cuda_stream)
    m = DistMPS(rank, n, chi) if distributed else MPS(rank, n, chi)
    layers = layers if layers is not None else rcs_1d_layers(n, depth, seed)
    recs = []
    for li, (singles, pairs) in enumerate(layers):
        for q, g in enumerate(singles):
            m.apply_1q(q, SINGLE_QUBIT[g])
        if distributed:
            qs = [q for (q, _) in pairs]
            mine = [q for q in qs if m.lo <= q and q + 1 < m.hi] + [q for q in qs if q == m.hi - 1 and q + 1 < n]
            for q, (s, frac) in zip(mine, m.apply_layer(pairs, circuits.FSIM)):
                recs.append((li, q, frac, s))
        elif batched:
            for (q, _), (s, frac) in zip(pairs, m.apply_layer(pairs, circuits.FSIM)):
                recs.append((li, q, frac, s))
        else:
            for (q, q1) in pairs:
                s, frac = m.apply_2q(q, circuits.FSIM)
                recs.append((li, q, frac, s))
    return m, recs
