// Tensor storage variants on the device (tensor.hpp:28-164, :209-337; ops.hpp:54-161).
//
// Reference: a Tensor is dense, symmetric (dense storage, half-split layout
// validated), diagonal (only elements with equal input and output coordinates
// stored), or computed (identity / swap: no storage, an element is 1 iff the
// paired coordinates agree). Structural ops either keep the variant (rebcast,
// conj, scale) or go through to_dense() first.
//
// Here the compact variants keep the same storage contract in HBM: a diagonal
// tensor holds one slice of the diagonal per on-diagonal block (nothing on the
// other blocks), identity / swap hold nothing. A diagonal tensor's storage is
// exactly a dense "shadow" tensor over (in_dist, out_dist; in_local) whose
// off-diagonal blocks are zero, so its rebcast is the dense remap of the shadow
// (same homes, same zero canonicalisation, one exchange) and never materialises
// the N_l-element blocks.
#include <numeric>

#include "ops.h"

namespace qtnhb {

void check_symmetric_shape(const Shape& s) {  // tensor.hpp:479-489
  const int split = s.split, nl = s.n_local();
  if (split % 2 != 0 || nl % 2 != 0) throw_invalid("symmetric tensors split both index groups in half");
  for (int i = 0; i < split / 2; ++i)
    if (s.dims[i] != s.dims[split / 2 + i]) throw_invalid("symmetric distributed dimensions differ");
  for (int i = 0; i < nl / 2; ++i)
    if (s.dims[split + i] != s.dims[split + nl / 2 + i]) throw_invalid("symmetric local dimensions differ");
}

Dim diag_local_count(const Shape& s) {
  Dim n = 1;
  for (int i = 0; i < s.n_local() / 2; ++i) n *= s.dims[s.split + i];
  return n;
}

bool diag_block_on_diagonal(const Shape& s, Dim block, Dim* in_block) {
  const int k = s.split / 2;
  auto dc = unflat(block, s.dist_dims());
  Dim b_in = 0;
  for (int i = 0; i < k; ++i) {
    if (dc[i] != dc[k + i]) return false;
    b_in = b_in * s.dims[i] + dc[i];
  }
  if (in_block) *in_block = b_in;
  return true;
}

Dim stored_count(const TensorImpl& t) {
  if (!t.in_span) return 0;
  switch (t.variant) {
    case kDense:
    case kSymmetric: return t.shape.local_size();
    case kDiagonal: return t.buf ? diag_local_count(t.shape) : 0;
    default: return 0;
  }
}

TP make_diagonal(RankCtx& r, Shape s, Dist d, const double* diag_global, Dim count) {
  check_symmetric_shape(s);
  Dim nd_in = 1;
  for (int i = 0; i < s.split / 2; ++i) nd_in *= s.dims[i];
  const Dim nl_in = diag_local_count(s);
  TP t = make_tensor(r, std::move(s), d, false);  // validation and ResourceError first (tensor.hpp:119)
  t->variant = kDiagonal;
  if (count != nd_in * nl_in) throw_invalid("diagonal payload has wrong length");
  Dim b_in = 0;
  if (t->in_span && diag_block_on_diagonal(t->shape, t->block, &b_in)) {
    t->buf = std::make_shared<DevBuf>(static_cast<size_t>(nl_in) * 16, r);
    if (diag_global) {
      QTNH_CUDA(cudaMemcpyAsync(t->data(), diag_global + 2 * b_in * nl_in, nl_in * 16, cudaMemcpyHostToDevice,
                                r.stream));
      QTNH_CUDA(cudaStreamSynchronize(r.stream));  // the host payload is the caller's
    } else {
      fill_zero(t->data(), nl_in, r.stream);
    }
  }
  return t;
}

namespace {
// Equality constraints of an identity / swap tensor (tensor.hpp:491-517): swap
// crosses the two outputs.
std::vector<int> equality_out(const TensorImpl& t) {
  std::vector<int> eq = t.pair_out;
  if (t.variant == kSwap) std::swap(eq[0], eq[1]);
  return eq;
}
}  // namespace

TP make_paired(RankCtx& r, Shape s, Dist d, const std::vector<int>& in_pos, const std::vector<int>& out_pos,
               bool crossed) {
  if (crossed && (in_pos.size() != 2 || out_pos.size() != 2)) throw_invalid("swap pairs exactly two indices");
  TP t = make_tensor(r, std::move(s), d, false);
  t->variant = crossed ? kSwap : kIdentity;
  const int n = t->shape.n_idx();
  if (in_pos.size() != out_pos.size()) throw_invalid("input/output position lists differ in length");
  std::vector<char> used(n, 0);
  auto chk = [&](int p) {
    if (p < 0 || p >= n || used[p]) throw_invalid("invalid index pairing");
    used[p] = 1;
  };
  for (int p : in_pos) chk(p);
  for (int p : out_pos) chk(p);
  if (static_cast<int>(in_pos.size() + out_pos.size()) != n)
    throw_invalid("every index must belong to exactly one pair");
  t->pair_in = in_pos;
  t->pair_out = out_pos;
  auto eq = equality_out(*t);
  for (size_t k = 0; k < in_pos.size(); ++k)
    if (t->shape.dims[in_pos[k]] != t->shape.dims[eq[k]]) throw_invalid("paired indices must have equal dimensions");
  return t;
}

TP variant_to_dense(const TP& t) {
  if (t->variant == kDense) return t;
  RankCtx& r = *t->rank;
  if (t->variant == kSymmetric) {  // same storage, dense tag (tensor.hpp:285-288)
    auto q = std::make_shared<TensorImpl>(*t);
    q->variant = kDense;
    return q;
  }
  TP out = make_tensor(r, t->shape, t->dist, true);
  if (!out->in_span) return out;
  const Dim nl = out->shape.local_size();
  if (t->variant == kDiagonal) {
    fill_zero(out->data(), nl, r.stream);
    if (t->buf) {  // local block (in_local, out_local) row-major: entry (j, j) at j (nl_in + 1)
      const Dim nl_in = diag_local_count(t->shape);
      CopyBox b;
      b.dims = {nl_in};
      b.in_stride = {1};
      b.out_stride = {nl_in + 1};
      strided_copy(t->data(), out->data(), b, false, r.stream);
    }
    return out;
  }
  fill_paired(out->data(), nl, out->block, out->shape.dims, out->shape.split, t->pair_in, equality_out(*t), r.stream);
  return out;
}

namespace {
// The dense tensor over (in_dist, out_dist; in_local) that a diagonal tensor's
// storage is: on-diagonal blocks share the slice, the others are zero.
TP diagonal_shadow(const TP& t) {
  const Shape& s = t->shape;
  std::vector<Dim> dims = s.dist_dims();
  for (int i = 0; i < s.n_local() / 2; ++i) dims.push_back(s.dims[s.split + i]);
  TP sh = make_tensor(*t->rank, Shape(dims, s.split), t->dist, false);
  if (!sh->in_span) return sh;
  if (t->buf) {
    sh->buf = t->buf;
  } else {
    const Dim n = sh->shape.local_size();
    sh->buf = std::make_shared<DevBuf>(static_cast<size_t>(n) * 16, *t->rank);
    fill_zero(sh->data(), n, t->rank->stream);
  }
  return sh;
}
}  // namespace

TP variant_rebcast(const TP& t, Dist d) {
  d.validate();
  RankCtx& r = *t->rank;
  switch (t->variant) {
    case kIdentity:
    case kSwap:  // metadata only (ops.hpp:57-62)
      return make_paired(r, t->shape, d, t->pair_in, t->pair_out, t->variant == kSwap);
    case kDiagonal: {  // same slices, new homes (ops.hpp:63-103)
      TP sh = diagonal_shadow(t);
      std::vector<int> ident(sh->shape.n_idx());
      std::iota(ident.begin(), ident.end(), 0);
      TP moved = remap(sh, sh->shape, d, ident);
      TP out = make_tensor(r, t->shape, d, false);
      out->variant = kDiagonal;
      if (out->in_span && diag_block_on_diagonal(out->shape, out->block)) out->buf = moved->buf;
      return out;
    }
    default: {
      TP out = op_rebcast(t, d);
      if (t->variant != kSymmetric) return out;
      auto q = std::make_shared<TensorImpl>(*out);  // same block, symmetric tag (ops.hpp:104-108)
      q->variant = kSymmetric;
      return q;
    }
  }
}

TP variant_scale(const TP& t, double re, double im, bool conj) {
  RankCtx& r = *t->rank;
  switch (t->variant) {
    case kIdentity:
    case kSwap:
      if (conj) return t;  // real entries (ops.hpp:148)
      return op_scale(variant_to_dense(t), re, im, false);  // ops.hpp:156-158
    case kDiagonal: {
      TP out = make_tensor(r, t->shape, t->dist, false);
      out->variant = kDiagonal;
      if (t->buf) {
        const Dim n = diag_local_count(t->shape);
        out->buf = std::make_shared<DevBuf>(static_cast<size_t>(n) * 16, r);
        scale_conj(t->data(), out->data(), n, re, im, conj, r.stream);
      }
      return out;
    }
    default: {
      TP out = op_scale(t, re, im, conj);
      out->variant = t->variant;
      return out;
    }
  }
}

void variant_local_element(const TensorImpl& t, const std::vector<Dim>& c, double* out2) {
  const Shape& s = t.shape;
  const int n = s.n_idx();
  if (static_cast<int>(c.size()) != n) throw_invalid("expected " + std::to_string(n) + " coordinates");
  for (int i = 0; i < n; ++i)
    if (c[i] < 0 || c[i] >= s.dims[i]) throw_invalid("coordinate out of bounds at index " + std::to_string(i));
  out2[0] = out2[1] = 0.0;
  auto fetch = [&](Dim off) {
    QTNH_CUDA(cudaMemcpyAsync(out2, static_cast<const char*>(t.data()) + off * 16, 16, cudaMemcpyDeviceToHost,
                              t.rank->stream));
    QTNH_CUDA(cudaStreamSynchronize(t.rank->stream));
  };
  auto hosted = [&] {
    Dim b = 0;
    for (int i = 0; i < s.split; ++i) b = b * s.dims[i] + c[i];
    if (!t.in_span || b != t.block) throw_invalid("rank does not host the requested element");
  };
  switch (t.variant) {
    case kDense:
    case kSymmetric: {
      hosted();
      Dim off = 0;
      for (int i = s.split; i < n; ++i) off = off * s.dims[i] + c[i];
      fetch(off);
      return;
    }
    case kDiagonal: {
      const int kd = s.split / 2, kl = s.n_local() / 2;
      for (int i = 0; i < kd; ++i)
        if (c[i] != c[kd + i]) return;
      for (int i = 0; i < kl; ++i)
        if (c[s.split + i] != c[s.split + kl + i]) return;
      hosted();
      Dim off = 0;
      for (int i = 0; i < kl; ++i) off = off * s.dims[s.split + i] + c[s.split + i];
      fetch(off);
      return;
    }
    default: {
      auto eq = equality_out(t);
      for (size_t k = 0; k < t.pair_in.size(); ++k)
        if (c[t.pair_in[k]] != c[eq[k]]) return;
      out2[0] = 1.0;
      return;
    }
  }
}

}  // namespace qtnhb
