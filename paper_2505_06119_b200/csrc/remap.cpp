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

Dim prod_dims(const std::vector<Dim>& dims, const std::vector<int>& idx) {
  Dim p = 1;
  for (int i : idx) p *= dims[i];
  return p;
}

}  // namespace

// Index classes (src positions) of a remap:
//   V src-local -> dst-dist   (ordered by dst position): chunk index
//   W src-local -> dst-local  (ordered by dst position): chunk payload
//   F src-dist  -> dst-local  (ordered by src position): chunk placement
//   G src-dist  -> dst-dist: routing only
RemapPlan plan_remap(const Shape& ss, const Dist& sd, const Shape& ds, const Dist& dd, const std::vector<int>& am,
                     int rank, int world_size) {
  int n = ss.n_idx();
  if (static_cast<int>(am.size()) != n) throw_invalid("axis map size does not match tensor rank");
  if (ds.n_idx() != n) throw_invalid("axis map is not a bijection");
  std::vector<int> inv(n, -1);
  for (int i = 0; i < n; ++i) {
    int p = am[i];
    if (p < 0 || p >= n || inv[p] != -1) throw_invalid("axis map is not a bijection");
    inv[p] = i;
    if (ds.dims[p] != ss.dims[i]) throw_invalid("remap needs equal mapped dimensions");
  }
  Dim need = dd.offset + dd.span(ds.dist_size());
  if (need > world_size) throw_resource("tensor span exceeds world size", need);
  RemapPlan R;
  Dim src_nd = ss.dist_size(), dst_nd = ds.dist_size();
  R.members = union_members({{sd.offset, sd.span(src_nd)}, {dd.offset, dd.span(dst_nd)}});
  R.member = std::binary_search(R.members.begin(), R.members.end(), rank);
  Dim blk = 0, cyc = 0, slot = 0;
  R.src_canonical = sd.locate(rank, src_nd, &blk, &cyc, &slot) && cyc == 0 && slot == 0;
  Dim src_block = blk;
  Dim dblk = 0, dcyc = 0, dslot = 0;
  R.dst_in_span = dd.locate(rank, dst_nd, &dblk, &dcyc, &dslot);
  Dim dst_block = dblk;
  if (!R.member) return R;

  std::vector<int> V, W, F;
  for (int p = 0; p < n; ++p) {
    int q = inv[p];
    bool sdist = q < ss.split, ddist = p < ds.split;
    if (!sdist && ddist) V.push_back(q);
    if (!sdist && !ddist) W.push_back(q);
    if (sdist && !ddist) F.push_back(q);
  }
  std::sort(F.begin(), F.end());
  const Dim nV = prod_dims(ss.dims, V), szW = prod_dims(ss.dims, W);
  auto sdd = ss.dist_dims(), ddd = ds.dist_dims();
  auto dst_local_strides = row_major_strides(ds.local_dims());
  auto src_local_strides = row_major_strides(ss.local_dims());
  auto dls = [&](int q) { return dst_local_strides[am[q] - ds.split]; };
  std::vector<Dim> vdims;
  for (int q : V) vdims.push_back(ss.dims[q]);
  // destination block of source block bs, chunk v (row-major over V)
  auto dst_block_of = [&](Dim bs, Dim v) {
    auto cs = unflat(bs, sdd);
    auto cv = unflat(v, vdims);
    std::vector<Dim> cd(ds.split);
    for (int p = 0; p < ds.split; ++p) {
      int q = inv[p];
      cd[p] = q < ss.split ? cs[q] : cv[std::find(V.begin(), V.end(), q) - V.begin()];
    }
    return flat(cd, ddd);
  };
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
      Dim st = 1;
      for (int k = static_cast<int>(W.size()) - 1; k >= 0; --k) {
        b.out_stride[W[k] - ss.split] = st;
        st *= ss.dims[W[k]];
      }
      for (int k = static_cast<int>(V.size()) - 1; k >= 0; --k) {
        b.out_stride[V[k] - ss.split] = st;
        st *= ss.dims[V[k]];
      }
    }
    return b;
  };

  // No element changes rank and there are no broadcast copies to feed: a plain
  // local permutation on every canonical holder. Same answer on all members.
  R.direct_layout = V.empty() && F.empty();
  R.local_only = R.direct_layout && dd.stretch * dd.cycles == 1;
  for (Dim bs = 0; bs < src_nd && R.local_only; ++bs)
    if (sd.canonical(bs) != dd.canonical(dst_block_of(bs, 0))) R.local_only = false;
  if (R.local_only) {
    R.pack_to_dst = true;
    R.pack = pack_box(true);
    return R;
  }
  // ---- pushes (peer-memory form) -------------------------------------------------------
  if (R.src_canonical) {
    for (int q : W) {
      R.push_box.dims.push_back(ss.dims[q]);
      R.push_box.in_stride.push_back(src_local_strides[q - ss.split]);
      R.push_box.out_stride.push_back(dls(q));
    }
    auto cs = unflat(src_block, sdd);
    Dim dst_off = 0;
    for (int q : F) dst_off += cs[q] * dls(q);
    for (Dim v = 0; v < nV; ++v) {
      auto cv = unflat(v, vdims);
      Dim src_off = 0;
      for (size_t k = 0; k < V.size(); ++k) src_off += cv[k] * src_local_strides[V[k] - ss.split];
      for (int h : dd.homes(dst_block_of(src_block, v), dst_nd)) R.pushes.push_back({h, src_off, dst_off});
    }
  }
  // ---- sends ------------------------------------------------------------------------
  if (R.src_canonical) {
    R.pack_to_dst = R.direct_layout && R.dst_in_span && dst_block == dst_block_of(src_block, 0);
    R.pack = pack_box(R.direct_layout);
    R.pack_elems = nV * szW;
    for (Dim v = 0; v < nV; ++v)
      for (int h : dd.homes(dst_block_of(src_block, v), dst_nd)) {
        if (R.pack_to_dst && h == rank) continue;
        R.sends.push_back({h, v * szW, szW});
      }
  }
  // ---- receives: every source block agreeing with my dst coords on G, row-major
  // over the src dist dims = row-major over F (src order) --------------------------------
  if (R.dst_in_span) {
    auto cd = unflat(dst_block, ddd);
    Dim off = 0;
    for (Dim bs = 0; bs < src_nd; ++bs) {
      auto cs = unflat(bs, sdd);
      bool ok = true;
      for (int p = 0; p < ds.split && ok; ++p)
        if (inv[p] < ss.split && cs[inv[p]] != cd[p]) ok = false;
      if (!ok) continue;
      int from = sd.canonical(bs);
      if (R.pack_to_dst && from == rank) continue;
      R.recvs.push_back({from, off, szW});
      off += szW;
    }
    R.recv_into_dst = R.direct_layout;
    R.recv_elems = off;
    if (!R.direct_layout) {
      // unpack box [F (src order)][W (dst order)] -> dst local
      R.unpack = true;
      CopyBox& b = R.unpack_box;
      Dim st = szW;
      std::vector<Dim> fstr(F.size()), wstr(W.size());
      for (int k = static_cast<int>(F.size()) - 1; k >= 0; --k) {
        fstr[k] = st;
        st *= ss.dims[F[k]];
      }
      st = 1;
      for (int k = static_cast<int>(W.size()) - 1; k >= 0; --k) {
        wstr[k] = st;
        st *= ss.dims[W[k]];
      }
      for (size_t k = 0; k < F.size(); ++k) {
        b.dims.push_back(ss.dims[F[k]]);
        b.in_stride.push_back(fstr[k]);
        b.out_stride.push_back(dls(F[k]));
      }
      for (size_t k = 0; k < W.size(); ++k) {
        b.dims.push_back(ss.dims[W[k]]);
        b.in_stride.push_back(wstr[k]);
        b.out_stride.push_back(dls(W[k]));
      }
    }
  }
  return R;
}

TP remap(const TP& src, Shape ds, Dist dd, const std::vector<int>& am) {
  QTNH_RANGE("qtnh::remap");
  RankCtx& r = *src->rank;
  RemapPlan P = plan_remap(src->shape, src->dist, ds, dd, am, r.rank, r.world->size);
  TP dst = make_tensor(r, ds, dd, true);
  if (!P.member) return dst;
  cudaStream_t st = r.stream;
  if (P.local_only) {
    if (P.src_canonical && dst->in_span) strided_copy(src->data(), dst->data(), P.pack, true, st);
    return dst;
  }
  if (peer_direct(r)) {
    // One pass: every canonical holder stores its chunks into the homes'
    // destination blocks over NVLink; the second all-gather is the fence.
    auto ptrs = peer_pointers(r, P.members, dst->in_span ? dst->data() : nullptr);
    for (const auto& p : P.pushes) {
      int j = static_cast<int>(std::lower_bound(P.members.begin(), P.members.end(), p.peer) - P.members.begin());
      if (j >= static_cast<int>(P.members.size()) || P.members[j] != p.peer || !ptrs[j])
        throw Status(QTNH_E_PROTOCOL, "peer remap target missing for pair (" + std::to_string(r.rank) + " -> " +
                                          std::to_string(p.peer) + ")");
      strided_copy(static_cast<const char*>(src->data()) + p.src_off * 16,
                   static_cast<char*>(ptrs[j]) + p.dst_off * 16, P.push_box, true, st);
    }
    peer_pointers(r, P.members, nullptr);
    return dst;
  }
  std::shared_ptr<DevBuf> packbuf, recvbuf;
  const void* send_ptr = nullptr;
  void* recv_ptr = nullptr;
  if (P.src_canonical) {
    if (P.pack_to_dst) {
      strided_copy(src->data(), dst->data(), P.pack, true, st);
      send_ptr = dst->data();
    } else {
      packbuf = std::make_shared<DevBuf>(static_cast<size_t>(P.pack_elems) * 16, r);
      strided_copy(src->data(), packbuf->ptr, P.pack, true, st);
      send_ptr = packbuf->ptr;
    }
  }
  if (dst->in_span) {
    if (P.recv_into_dst) {
      recv_ptr = dst->data();
    } else {
      recvbuf = std::make_shared<DevBuf>(static_cast<size_t>(P.recv_elems) * 16, r);
      recv_ptr = recvbuf->ptr;
    }
  }
  exchange(r, P.members, send_ptr, P.sends, recv_ptr, P.recvs);
  if (dst->in_span && P.unpack) strided_copy(recv_ptr, dst->data(), P.unpack_box, false, st);
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

TP op_scale_index(const TP& t, int pos, const std::vector<double>& f) {
  const Shape& sh = t->shape;
  if (pos < 0 || pos >= sh.n_idx()) throw_invalid("scale_index position out of range");
  if (static_cast<Dim>(f.size()) != sh.dims[pos]) throw_invalid("scale_index needs one factor per coordinate");
  TP out = make_tensor(*t->rank, sh, t->dist, true);
  if (!out->in_span) return out;
  RankCtx& r = *t->rank;
  const Dim nl = sh.local_size();
  if (pos < sh.split) {  // a distributed index: this rank's block has one coordinate
    const Dim c = unflat(t->block, sh.dist_dims())[pos];
    scale_conj(t->data(), out->data(), nl, f[c], 0.0, false, r.stream);
    return out;
  }
  Dim inner = 1;
  for (int i = pos + 1; i < sh.n_idx(); ++i) inner *= sh.dims[i];
  DevBuf fd(f.size() * sizeof(double), r);
  QTNH_CUDA(cudaMemcpyAsync(fd.ptr, f.data(), f.size() * sizeof(double), cudaMemcpyHostToDevice, r.stream));
  scale_index(t->data(), out->data(), nl, inner, sh.dims[pos], static_cast<const double*>(fd.ptr), r.stream);
  QTNH_CUDA(cudaStreamSynchronize(r.stream));  // the host factors are the caller's
  return out;
}

void op_to_global(const TensorImpl& t, double* host) {
  if (!t.in_span) return;
  RankCtx& r = *t.rank;
  Dim nl = t.shape.local_size(), nd = t.shape.dist_size();
  // raw values: the reference visits every dense element, zeros included
  // (visit_my_nonzeros, tensor.hpp:300-311), so signed zeros survive
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

// ---- in-place distributed <-> local index swap ------------------------------------------
namespace qtnhb {

// Exchange a distributed index a with a local index b of the same size d, in
// place: on the rank whose block has coordinate i at a, the local region b = j
// (j != i) is sent to the partner block (a = j) and replaced by the partner's
// region b = i. Only the (d-1)/d of each block that moves is touched, through a
// bounded staging buffer (chunks of the region's outer indices), so a 128 GiB
// shard swaps without a second copy of the tensor. Values equal ops::permute with
// a and b exchanged (zero canonicalisation included).
void op_swap_dist_local_inplace(TP& t, int a, int b, Dim chunk_bytes) {
  QTNH_RANGE("qtnh::swap_dist_local");
  const Shape& s = t->shape;
  if (!(a < s.split && b >= s.split)) throw_invalid("swap_dist_local needs a distributed a and a local b");
  const Dim d = s.dims[a];
  if (s.dims[b] != d) throw_invalid("swapped indices must have equal dimensions");
  RankCtx& r = *t->rank;
  auto members = span_ranks(*t);
  if (!t->in_span) return;
  const int lb = b - s.split;
  auto ld = s.local_dims();
  auto ls = row_major_strides(ld);
  const Dim nd = s.dist_size();
  auto ddims = s.dist_dims();
  auto cd = unflat(t->block, ddims);
  const Dim my_i = cd[a];
  // region (b fixed) dims / strides, outermost first
  std::vector<Dim> rdims, rstr;
  for (int q = 0; q < static_cast<int>(ld.size()); ++q)
    if (q != lb) {
      rdims.push_back(ld[q]);
      rstr.push_back(ls[q]);
    }
  Dim region = 1;
  for (Dim x : rdims) region *= x;
  // chunk the region over its outer dims: chunk = product of the innermost dims
  // that fit in chunk_bytes (at least one full innermost run)
  Dim per_chunk = 1;
  int split_at = static_cast<int>(rdims.size());
  while (split_at > 0 && per_chunk * rdims[split_at - 1] * 16 <= chunk_bytes) per_chunk *= rdims[--split_at];
  if (split_at == static_cast<int>(rdims.size()) && !rdims.empty()) {
    per_chunk = rdims.back();  // a run bigger than the budget: one run per chunk
    split_at = static_cast<int>(rdims.size()) - 1;
  }
  std::vector<Dim> odims(rdims.begin(), rdims.begin() + split_at), idims(rdims.begin() + split_at, rdims.end());
  std::vector<Dim> ostr(rstr.begin(), rstr.begin() + split_at), istr(rstr.begin() + split_at, rstr.end());
  Dim n_chunks = 1;
  for (Dim x : odims) n_chunks *= x;
  auto irow = row_major_strides(idims);
  const int partners = static_cast<int>(d - 1);
  DevBuf sbuf(static_cast<size_t>(per_chunk * std::max(1, partners)) * 16, r);
  DevBuf rbuf(static_cast<size_t>(per_chunk * std::max(1, partners)) * 16, r);
  if (peer_direct(r)) {
    // Peer-memory form: each pair of partner blocks exchanges its two regions
    // with one swap kernel over NVLink, no staging; the lower coordinate swaps
    // the first half of the pair's elements, the higher one the second half.
    // For d = 2 the same launch canonicalises both staying regions.
    Dim region_n = 1;
    for (Dim x : rdims) region_n *= x;
    char* keep = static_cast<char*>(t->data()) + my_i * ls[lb] * 16;
    if (d != 2) canon_region(keep, rdims, rstr, r.stream);
    auto ptrs = peer_pointers(r, members, t->data());
    for (Dim j = 0; j < d; ++j) {
      if (j == my_i) continue;
      auto pc = cd;
      pc[a] = j;
      int peer = t->dist.home(flat(pc, ddims), nd, t->cycle, t->slot);
      char* pb = static_cast<char*>(ptrs[peer - members.front()]);
      Dim half = region_n / 2;
      Dim lo = my_i < j ? 0 : half, hi = my_i < j ? half : region_n;
      swap_regions(static_cast<char*>(t->data()) + j * ls[lb] * 16, pb + my_i * ls[lb] * 16, rdims, rstr, lo, hi,
                   r.stream, d == 2 ? keep : nullptr, d == 2 ? pb + j * ls[lb] * 16 : nullptr);
    }
    peer_pointers(r, members, nullptr);
    return;
  }
  // Exchange form (NCCL world, or peer_direct off): a three-stage pipeline over
  // two staging pairs -- pack chunk c+1 (side stream 0) and unpack chunk c-1
  // (side stream 1) overlap the exchange of chunk c on the rank stream. Events
  // keep each staging buffer free until its previous user is done. Counts are
  // identical for every chunk, so the NCCL form verifies them once and waits for
  // completion once, at the end.
  canon_region(static_cast<char*>(t->data()) + my_i * ls[lb] * 16, rdims, rstr, r.stream);
  DevBuf sbuf2(static_cast<size_t>(per_chunk * std::max(1, partners)) * 16, r);
  DevBuf rbuf2(static_cast<size_t>(per_chunk * std::max(1, partners)) * 16, r);
  char* sb[2] = {static_cast<char*>(sbuf.ptr), static_cast<char*>(sbuf2.ptr)};
  char* rb[2] = {static_cast<char*>(rbuf.ptr), static_cast<char*>(rbuf2.ptr)};
  cudaStream_t pk_st = r.side_stream(0), up_st = r.side_stream(1);
  cudaEvent_t start, packed[2], xfered[2], unpacked[2];
  auto mk = [](cudaEvent_t& e) { QTNH_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming)); };
  mk(start);
  for (int k = 0; k < 2; ++k) {
    mk(packed[k]);
    mk(xfered[k]);
    mk(unpacked[k]);
  }
  QTNH_CUDA(cudaEventRecord(start, r.stream));
  QTNH_CUDA(cudaStreamWaitEvent(pk_st, start, 0));
  QTNH_CUDA(cudaStreamWaitEvent(up_st, start, 0));
  std::vector<Dim> peers;
  for (Dim j = 0; j < d; ++j)
    if (j != my_i) peers.push_back(j);
  auto peer_of = [&](Dim j) {
    auto pc = cd;
    pc[a] = j;
    return t->dist.home(flat(pc, ddims), nd, t->cycle, t->slot);
  };
  try {
    for (Dim ch = 0; ch < n_chunks; ++ch) {
      const int k = static_cast<int>(ch & 1);
      auto oc = unflat(ch, odims);
      Dim obase = 0;
      for (size_t q = 0; q < oc.size(); ++q) obase += oc[q] * ostr[q];
      // pack: sb[k] is free once the exchange of chunk ch-2 has read it
      if (ch >= 2) QTNH_CUDA(cudaStreamWaitEvent(pk_st, xfered[k], 0));
      std::vector<Xfer> sends, recvs;
      for (size_t sl = 0; sl < peers.size(); ++sl) {
        CopyBox pk;
        pk.dims = idims;
        pk.in_stride = istr;
        pk.out_stride = irow;
        const char* src = static_cast<const char*>(t->data()) + (obase + peers[sl] * ls[lb]) * 16;
        strided_copy(src, sb[k] + sl * per_chunk * 16, pk, true, pk_st);
        const int peer = peer_of(peers[sl]);
        sends.push_back({peer, static_cast<Dim>(sl) * per_chunk, per_chunk});
        recvs.push_back({peer, static_cast<Dim>(sl) * per_chunk, per_chunk});
      }
      QTNH_CUDA(cudaEventRecord(packed[k], pk_st));
      // exchange on the rank stream: rb[k] is free once chunk ch-2 is unpacked
      QTNH_CUDA(cudaStreamWaitEvent(r.stream, packed[k], 0));
      if (ch >= 2) QTNH_CUDA(cudaStreamWaitEvent(r.stream, unpacked[k], 0));
      exchange(r, members, sb[k], sends, rb[k], recvs, /*checked=*/ch == 0, /*wait=*/false);
      QTNH_CUDA(cudaEventRecord(xfered[k], r.stream));
      // unpack
      QTNH_CUDA(cudaStreamWaitEvent(up_st, xfered[k], 0));
      for (size_t sl = 0; sl < peers.size(); ++sl) {
        CopyBox up;
        up.dims = idims;
        up.in_stride = irow;
        up.out_stride = istr;
        char* dst = static_cast<char*>(t->data()) + (obase + peers[sl] * ls[lb]) * 16;
        strided_copy(rb[k] + sl * per_chunk * 16, dst, up, false, up_st);
      }
      QTNH_CUDA(cudaEventRecord(unpacked[k], up_st));
    }
  } catch (...) {
    QTNH_CUDA(cudaEventRecord(unpacked[0], up_st));
    cudaStreamWaitEvent(r.stream, unpacked[0], 0);
    cudaStreamWaitEvent(r.stream, packed[0], 0);
    throw;
  }
  // the rank stream continues after the last unpack (and the staging buffers,
  // freed stream-ordered on it, outlive every side-stream use)
  QTNH_CUDA(cudaEventRecord(unpacked[0], up_st));
  QTNH_CUDA(cudaEventRecord(packed[0], pk_st));
  QTNH_CUDA(cudaStreamWaitEvent(r.stream, unpacked[0], 0));
  QTNH_CUDA(cudaStreamWaitEvent(r.stream, packed[0], 0));
  cudaEventDestroy(start);
  for (int k = 0; k < 2; ++k) {
    cudaEventDestroy(packed[k]);
    cudaEventDestroy(xfered[k]);
    cudaEventDestroy(unpacked[k]);
  }
  nccl_wait(r);
}

}  // namespace qtnhb
