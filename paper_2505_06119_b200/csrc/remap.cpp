// Redistribution engine and the structural ops built on it.
//
// Reference: remap::tensor_to_tensor (remap.hpp:106-161) packs one 24-byte
// (address, re, im) Item per element, exchanges the lists with all_to_all_v and
// scatters them into a zeroed destination. Here the destination address of every
// element is affine in its coordinates, so the whole redistribution is
//   pack   : one strided-copy launch that permutes this rank's canonical block
//            into contiguous per-destination-block chunks (zero canonicalised);
//   exchange: stream-ordered device/peer copies (local world) or grouped NCCL
//            send/recv (process per GPU) of raw 16-byte elements;
//   unpack : one strided-copy launch that embeds the received chunks into the
//            destination block.
// When no element changes rank, the permutation goes straight into the
// destination buffer (one launch, read once / write once).
#include <algorithm>
#include <numeric>

#include "ops.h"
#include "strided_copy.h"

namespace qtnhb {

namespace {

struct RemapPlan {
  // index classes (src positions), see file header of DESIGN.md section "remap"
  std::vector<int> V;  // src-local -> dst-dist   (ordered by dst position)
  std::vector<int> W;  // src-local -> dst-local  (ordered by dst position)
  std::vector<int> F;  // src-dist  -> dst-local  (ordered by src position)
  std::vector<int> G;  // src-dist  -> dst-dist
  Dim nV = 1, szW = 1, nF = 1;
};

Dim prod_dims(const std::vector<Dim>& dims, const std::vector<int>& idx) {
  Dim p = 1;
  for (int i : idx) p *= dims[i];
  return p;
}

}  // namespace

TP remap(const TP& src, Shape ds, Dist dd, const std::vector<int>& am) {
  const Shape& ss = src->shape;
  int n = ss.n_idx();
  if (static_cast<int>(am.size()) != n) throw_invalid("axis map size does not match tensor rank");
  std::vector<int> inv(ds.n_idx(), -1);
  for (int i = 0; i < n; ++i) {
    int p = am[i];
    if (p < 0 || p >= ds.n_idx() || inv[p] != -1) throw_invalid("axis map is not a bijection");
    inv[p] = i;
    if (ds.dims[p] != ss.dims[i]) throw_invalid("remap needs equal mapped dimensions");
  }
  if (ds.n_idx() != n) throw_invalid("axis map is not a bijection");
  RankCtx& r = *src->rank;
  TP dst = make_tensor(r, ds, dd, true);
  auto members = union_members({{src->dist.offset, src->span()}, {dd.offset, dst->span()}});
  if (!std::binary_search(members.begin(), members.end(), r.rank)) return dst;

  RemapPlan P;
  for (int p = 0; p < n; ++p) {
    int q = inv[p];
    bool sdist = q < ss.split, ddist = p < ds.split;
    if (!sdist && ddist) P.V.push_back(q);
    if (!sdist && !ddist) P.W.push_back(q);
    if (sdist && !ddist) P.F.push_back(q);
    if (sdist && ddist) P.G.push_back(q);
  }
  std::sort(P.F.begin(), P.F.end());
  P.nV = prod_dims(ss.dims, P.V);
  P.szW = prod_dims(ss.dims, P.W);
  P.nF = prod_dims(ss.dims, P.F);

  const Dim src_nd = ss.dist_size(), dst_nd = ds.dist_size();
  auto sdd = ss.dist_dims(), ddd = ds.dist_dims();
  auto dst_local_strides = row_major_strides(ds.local_dims());
  auto src_local_strides = row_major_strides(ss.local_dims());
  // dst local stride of a src index q that lands at a dst-local position
  auto dls = [&](int q) { return dst_local_strides[am[q] - ds.split]; };

  // dst block of src block bs, chunk v (row-major over V)
  auto dst_block = [&](Dim bs, Dim v) {
    auto cs = unflat(bs, sdd);
    std::vector<Dim> vd;
    for (int q : P.V) vd.push_back(ss.dims[q]);
    auto cv = unflat(v, vd);
    std::vector<Dim> cd(ds.split);
    for (int p = 0; p < ds.split; ++p) {
      int q = inv[p];
      if (q < ss.split) cd[p] = cs[q];
      else cd[p] = cv[std::find(P.V.begin(), P.V.end(), q) - P.V.begin()];
    }
    return flat(cd, ddd);
  };

  // Is any element moving between ranks (or copies needed)? Same answer on all members.
  bool local_only = P.V.empty() && P.F.empty() && dd.stretch * dd.cycles == 1;
  if (local_only) {
    for (Dim bs = 0; bs < src_nd && local_only; ++bs)
      if (src->dist.canonical(bs) != dd.canonical(dst_block(bs, 0))) local_only = false;
  }

  cudaStream_t st = r.stream;
  bool direct_layout = P.V.empty() && P.F.empty();  // pack layout == dst layout
  // Pack box over my local (src-local) indices.
  auto pack_box = [&](bool to_dst_layout) {
    CopyBox b;
    for (int q = ss.split; q < n; ++q) {
      b.dims.push_back(ss.dims[q]);
      b.in_stride.push_back(src_local_strides[q - ss.split]);
    }
    b.out_stride.assign(b.dims.size(), 0);
    if (to_dst_layout) {
      for (int q = ss.split; q < n; ++q) b.out_stride[q - ss.split] = dls(q);
    } else {
      Dim s = 1;
      for (int k = static_cast<int>(P.W.size()) - 1; k >= 0; --k) {
        b.out_stride[P.W[k] - ss.split] = s;
        s *= ss.dims[P.W[k]];
      }
      for (int k = static_cast<int>(P.V.size()) - 1; k >= 0; --k) {
        b.out_stride[P.V[k] - ss.split] = s;
        s *= ss.dims[P.V[k]];
      }
    }
    return b;
  };

  if (local_only) {
    if (src->canonical() && dst->in_span) strided_copy(src->data(), dst->data(), pack_box(true), true, st);
    return dst;
  }

  // ---- general path: sends ------------------------------------------------------
  std::vector<Xfer> sends, recvs;
  std::shared_ptr<DevBuf> packbuf, recvbuf;
  const void* send_ptr = nullptr;
  void* recv_ptr = nullptr;
  bool sent_into_dst = false;
  if (src->canonical()) {
    bool self_home_direct = false;
    if (direct_layout && dst->in_span && dst->block == dst_block(src->block, 0)) self_home_direct = true;
    if (self_home_direct) {
      strided_copy(src->data(), dst->data(), pack_box(true), true, st);
      send_ptr = dst->data();
      sent_into_dst = true;
    } else {
      packbuf = std::make_shared<DevBuf>(static_cast<size_t>(P.nV * P.szW) * 16, r);
      strided_copy(src->data(), packbuf->ptr, pack_box(direct_layout), true, st);
      send_ptr = packbuf->ptr;
    }
    for (Dim v = 0; v < P.nV; ++v) {
      Dim bd = dst_block(src->block, v);
      for (int h : dd.homes(bd, dst_nd)) {
        if (sent_into_dst && h == r.rank) continue;
        sends.push_back({h, v * P.szW, P.szW});
      }
    }
  }
  // ---- receives -----------------------------------------------------------------
  // Sources: src blocks agreeing with my dst dist coords on G; enumerated row-major
  // over the src dist dims, i.e. row-major over F (src order).
  std::vector<Dim> src_blocks;
  if (dst->in_span) {
    auto cd = unflat(dst->block, ddd);
    for (Dim bs = 0; bs < src_nd; ++bs) {
      auto cs = unflat(bs, sdd);
      bool ok = true;
      for (int p = 0; p < ds.split && ok; ++p)
        if (inv[p] < ss.split && cs[inv[p]] != cd[p]) ok = false;
      if (ok) src_blocks.push_back(bs);
    }
    // chunk index v of my block within each source's pack
    Dim off = 0;
    bool recv_into_dst = direct_layout;
    for (Dim bs : src_blocks) {
      int from = src->dist.canonical(bs);
      if (sent_into_dst && from == r.rank) continue;
      (void)recv_into_dst;
      recvs.push_back({from, off, P.szW});
      off += P.szW;
    }
    if (direct_layout) {
      recv_ptr = dst->data();  // single source, layout already final
    } else {
      recvbuf = std::make_shared<DevBuf>(static_cast<size_t>(off) * 16, r);
      recv_ptr = recvbuf->ptr;
    }
  }
  // chunk offsets within senders: sender list order is by v, then homes; the
  // receiver asks for the chunk by order, so fix up sender-side offsets: each send
  // entry already carries its own offset; receivers match in order per peer.
  exchange(r, members, send_ptr, sends, recv_ptr, recvs);

  if (dst->in_span && !direct_layout) {
    // Unpack: box [F (src order)][W (dst order)] -> dst local.
    CopyBox b;
    Dim s = P.szW;
    std::vector<Dim> fstr(P.F.size());
    for (int k = static_cast<int>(P.F.size()) - 1; k >= 0; --k) {
      fstr[k] = s;
      s *= ss.dims[P.F[k]];
    }
    for (size_t k = 0; k < P.F.size(); ++k) {
      b.dims.push_back(ss.dims[P.F[k]]);
      b.in_stride.push_back(fstr[k]);
      b.out_stride.push_back(dls(P.F[k]));
    }
    s = 1;
    std::vector<Dim> wstr(P.W.size());
    for (int k = static_cast<int>(P.W.size()) - 1; k >= 0; --k) {
      wstr[k] = s;
      s *= ss.dims[P.W[k]];
    }
    for (size_t k = 0; k < P.W.size(); ++k) {
      b.dims.push_back(ss.dims[P.W[k]]);
      b.in_stride.push_back(wstr[k]);
      b.out_stride.push_back(dls(P.W[k]));
    }
    // Sources not present (F coords of blocks outside...) cannot happen: every
    // src block exists, so the box covers the whole destination block.
    strided_copy(recv_ptr, dst->data(), b, false, st);
  }
  return dst;
}

TP op_permute(const TP& t, const std::vector<int>& perm, int new_split) {
  int r = t->shape.n_idx();
  if (static_cast<int>(perm.size()) != r) throw_invalid("permutation size does not match tensor rank");
  std::vector<int> inv(r, -1);
  for (int p = 0; p < r; ++p) {
    int o = perm[p];
    if (o < 0 || o >= r || inv[o] != -1) throw_invalid("invalid index permutation");
    inv[o] = p;
  }
  if (new_split < 0 || new_split > r) throw_invalid("invalid split for permuted tensor");
  bool identity = new_split == t->shape.split;
  for (int p = 0; p < r && identity; ++p) identity = perm[p] == p;
  if (identity) return t;
  std::vector<Dim> nd(r);
  for (int p = 0; p < r; ++p) nd[p] = t->shape.dims[perm[p]];
  return remap(t, Shape(nd, new_split), t->dist, inv);
}

TP op_rebcast(const TP& t, Dist d) {
  d.validate();
  std::vector<int> ident(t->shape.n_idx());
  std::iota(ident.begin(), ident.end(), 0);
  return remap(t, t->shape, d, ident);
}

TP op_scatter_index(const TP& t, int pos) {
  const Shape& s = t->shape;
  if (pos < s.split || pos >= s.n_idx()) throw_invalid("scatter_index position must name a local index");
  std::vector<int> perm;
  for (int i = 0; i < s.split; ++i) perm.push_back(i);
  perm.push_back(pos);
  for (int i = s.split; i < s.n_idx(); ++i)
    if (i != pos) perm.push_back(i);
  return op_permute(t, perm, s.split + 1);
}

TP op_gather_index(const TP& t, int pos) {
  const Shape& s = t->shape;
  if (pos < 0 || pos >= s.split) throw_invalid("gather_index position must name a distributed index");
  std::vector<int> perm;
  for (int i = 0; i < s.split; ++i)
    if (i != pos) perm.push_back(i);
  perm.push_back(pos);
  for (int i = s.split; i < s.n_idx(); ++i) perm.push_back(i);
  return op_permute(t, perm, s.split - 1);
}

TP op_slice_local(const TP& t, const std::vector<Dim>& nl) {
  auto ld = t->shape.local_dims();
  if (nl.size() != ld.size()) throw_invalid("local dimension count mismatch");
  bool same = true;
  for (size_t i = 0; i < ld.size(); ++i) {
    if (nl[i] > ld[i]) throw_invalid("slice cannot grow a dimension");
    same &= nl[i] == ld[i];
  }
  if (same) return t;
  std::vector<Dim> dims = t->shape.dist_dims();
  dims.insert(dims.end(), nl.begin(), nl.end());
  TP out = make_tensor(*t->rank, Shape(dims, t->shape.split), t->dist, true);
  if (out->in_span) {
    CopyBox b;
    b.dims = nl;
    b.in_stride = row_major_strides(ld);
    b.out_stride = row_major_strides(nl);
    strided_copy(t->data(), out->data(), b, false, t->rank->stream);
  }
  return out;
}

TP op_pad_local(const TP& t, const std::vector<Dim>& nl) {
  auto ld = t->shape.local_dims();
  if (nl.size() != ld.size()) throw_invalid("local dimension count mismatch");
  bool same = true;
  for (size_t i = 0; i < ld.size(); ++i) {
    if (nl[i] < ld[i]) throw_invalid("pad cannot shrink a dimension");
    same &= nl[i] == ld[i];
  }
  if (same) return t;
  std::vector<Dim> dims = t->shape.dist_dims();
  dims.insert(dims.end(), nl.begin(), nl.end());
  TP out = make_tensor(*t->rank, Shape(dims, t->shape.split), t->dist, true);
  if (out->in_span) {
    fill_zero(out->data(), out->shape.local_size(), t->rank->stream);
    CopyBox b;
    b.dims = ld;
    b.in_stride = row_major_strides(ld);
    b.out_stride = row_major_strides(nl);
    strided_copy(t->data(), out->data(), b, false, t->rank->stream);
  }
  return out;
}

TP op_scale(const TP& t, double re, double im, bool conj) {
  TP out = make_tensor(*t->rank, t->shape, t->dist, true);
  if (out->in_span) scale_conj(t->data(), out->data(), t->shape.local_size(), re, im, conj, t->rank->stream);
  return out;
}

void op_to_global(const TensorImpl& t, double* host) {
  if (!t.in_span) return;
  RankCtx& r = *t.rank;
  Dim nl = t.shape.local_size(), nd = t.shape.dist_size();
  if (t.span() == 1) {
    QTNH_CUDA(cudaMemcpyAsync(host, t.data(), nl * 16, cudaMemcpyDeviceToHost, r.stream));
    QTNH_CUDA(cudaStreamSynchronize(r.stream));
    return;
  }
  auto members = span_ranks(t);
  std::vector<Xfer> sends, recvs;
  if (t.canonical())
    for (int m : members) sends.push_back({m, 0, nl});
  for (Dim b = 0; b < nd; ++b) recvs.push_back({t.dist.canonical(b), b * nl, nl});
  DevBuf all(static_cast<size_t>(nd * nl) * 16, r);
  exchange(r, members, t.data(), sends, all.ptr, recvs);
  QTNH_CUDA(cudaMemcpyAsync(host, all.ptr, nd * nl * 16, cudaMemcpyDeviceToHost, r.stream));
  QTNH_CUDA(cudaStreamSynchronize(r.stream));
}

}  // namespace qtnhb
