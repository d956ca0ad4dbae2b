// Pairwise contraction and gate application on sharded device tensors.
//
// Reference: SPEC network::contract realised with
// tensor_to_matrix -> pgemm -> matrix_to_tensor (linalg.hpp:208, :347, :273):
// every operand is redistributed into a 2-D block-cyclic matrix with one
// 24-byte Item per element and multiplied by SUMMA panel broadcasts.
//
// B200 design: no block-cyclic matrices. The contraction is made rank-local:
//   * the first operand keeps its sharding (its distributed indices select the
//     GPU; a contracted distributed index is first swapped with an open local
//     index of the same size -- one NVLink exchange);
//   * the second operand is replicated on the first operand's span (rebcast --
//     it is the small operand in every configuration: the 2^14 B of C1, gates);
//   * each GPU permutes its block into [open | contracted] and B into
//     [contracted | open] (skipped when already in that order) and runs one
//     FP64-tensor-core zgemm whose row-major output IS its block of the result in
//     the SPEC.md:408 order (open(a) then open(b)).
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <map>
#include <mutex>
#include <numeric>
#include <tuple>

#include "ops.h"
#include "strided_copy.h"

namespace qtnhb {

Dim swap_chunk_bytes();

namespace {

bool is_identity(const std::vector<int>& p) {
  for (size_t i = 0; i < p.size(); ++i)
    if (p[i] != static_cast<int>(i)) return false;
  return true;
}

// Local block of `t` permuted by perm (over local dims) into a fresh buffer, or
// the block itself when perm is the identity.
const void* local_permuted(const TensorImpl& t, const std::vector<Dim>& dims, const std::vector<int>& perm,
                           std::shared_ptr<DevBuf>& hold, RankCtx& r) {
  if (is_identity(perm)) return t.data();
  Dim n = 1;
  for (Dim d : dims) n *= d;
  hold = std::make_shared<DevBuf>(static_cast<size_t>(n) * 16, r);
  strided_copy(t.data(), hold->ptr, permute_box(dims, perm), false, r.stream);
  return hold->ptr;
}

// Offset tables of the fused-gather GEMM, cached per (device, dims, strides):
// a contraction repeated with the same layout (every bench step, every MPS
// update of a saturated bond) reuses them instead of regenerating 16 MB.
struct TableKey {
  int device;
  std::vector<Dim> dims, strides;
  bool operator<(const TableKey& o) const {
    return std::tie(device, dims, strides) < std::tie(o.device, o.dims, o.strides);
  }
};
using Table = std::shared_ptr<const int64_t>;
struct TableEntry {
  Table t;
  size_t bytes;
  cudaEvent_t ready;  // the table's generation; users on any stream wait on it
};
std::mutex g_tab_mu;
std::map<TableKey, TableEntry> g_tabs;
size_t g_tab_bytes = 0;

// Returns a reference-counted table: callers keep it alive until the GEMM that
// reads it is enqueued, so evicting the cache (or another rank thread on the
// same device evicting it) never frees a table a pending launch still names.
// The last holder frees it after the device drains.
Table gather_table(RankCtx& r, const std::vector<Dim>& dims, const std::vector<Dim>& strides) {
  TableKey key{r.device, dims, strides};
  std::lock_guard<std::mutex> lk(g_tab_mu);
  auto it = g_tabs.find(key);
  if (it != g_tabs.end()) {
    QTNH_CUDA(cudaStreamWaitEvent(r.stream, it->second.ready, 0));
    return it->second.t;
  }
  Dim count = 1;
  for (Dim d : dims) count *= d;
  if (g_tab_bytes > (size_t(1) << 30)) {  // bounded: drop the cache's references (tables are cheap to rebuild)
    g_tabs.clear();
    g_tab_bytes = 0;
  }
  const size_t bytes = static_cast<size_t>(std::max<Dim>(1, count)) * 8;
  int64_t* ptr = nullptr;
  QTNH_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&ptr), bytes, r.stream));  // pool hit, stream-ordered
  cudaEvent_t ready;
  QTNH_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
  const int dev = r.device;
  Table t(ptr, [dev, ready](const int64_t* p) {
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(dev);
    cudaDeviceSynchronize();  // launches that named the table have been enqueued by now: let them finish
    cudaFreeAsync(const_cast<int64_t*>(p), 0);
    cudaEventDestroy(ready);
    cudaSetDevice(cur);
  });
  index_offsets(ptr, count, dims, strides, r.stream);
  // other ranks (streams) on this device wait on the event instead of this
  // thread synchronising (a sync per new layout serialised C3's ~600 small steps)
  QTNH_CUDA(cudaEventRecord(ready, r.stream));
  g_tabs[key] = {t, bytes, ready};
  g_tab_bytes += bytes;
  return t;
}

}  // namespace

TP op_contract(const TP& a_in, const TP& b_in, const std::vector<int>& apos, const std::vector<int>& bpos) {
  QTNH_RANGE("qtnh::contract");
  if (apos.size() != bpos.size()) throw_invalid("contracted position lists differ in length");
  if (a_in->rank != b_in->rank) throw_invalid("operands belong to different ranks");
  RankCtx& r = *a_in->rank;
  const Shape& sa = a_in->shape;
  const Shape& sb = b_in->shape;
  std::vector<char> ca(sa.n_idx(), 0), cb(sb.n_idx(), 0);
  for (size_t i = 0; i < apos.size(); ++i) {
    int p = apos[i], q = bpos[i];
    if (p < 0 || p >= sa.n_idx() || ca[p] || q < 0 || q >= sb.n_idx() || cb[q])
      throw_invalid("invalid contracted index positions");
    if (sa.dims[p] != sb.dims[q]) throw_invalid("contracted dimensions differ");
    ca[p] = cb[q] = 1;
  }
  std::vector<int> a_open, b_open;
  for (int i = 0; i < sa.n_idx(); ++i)
    if (!ca[i]) a_open.push_back(i);
  for (int i = 0; i < sb.n_idx(); ++i)
    if (!cb[i]) b_open.push_back(i);
  std::vector<Dim> cdims;
  int csplit = 0;
  for (int p : a_open) {
    cdims.push_back(sa.dims[p]);
    if (p < sa.split) ++csplit;
  }
  for (int p : b_open) cdims.push_back(sb.dims[p]);

  // 1. Make every contracted index of `a` local: swap it with an open local index
  //    of equal size (keeps the span), else move it behind the split.
  TP a = a_in;
  std::vector<int> a_order(sa.n_idx());  // a2 position -> a position
  std::iota(a_order.begin(), a_order.end(), 0);
  int a2_split = sa.split;
  {
    std::vector<int> dist_contracted;
    for (int p = 0; p < sa.split; ++p)
      if (ca[p]) dist_contracted.push_back(p);
    if (!dist_contracted.empty()) {
      std::vector<char> used(sa.n_idx(), 0);
      std::vector<int> order = a_order;
      std::vector<int> demote;
      for (int p : dist_contracted) {
        int swap_with = -1;
        for (int q = sa.n_idx() - 1; q >= sa.split; --q)
          if (!ca[q] && !used[q] && sa.dims[q] == sa.dims[p]) {
            swap_with = q;
            break;
          }
        if (swap_with >= 0) {
          used[swap_with] = 1;
          std::swap(order[p], order[swap_with]);
        } else {
          demote.push_back(p);
        }
      }
      // Demoted contracted dist indices move to the front of the local group.
      std::vector<int> final_order;
      for (int p = 0; p < sa.split; ++p)
        if (std::find(demote.begin(), demote.end(), p) == demote.end()) final_order.push_back(order[p]);
      for (int p : demote) final_order.push_back(order[p]);
      for (int p = sa.split; p < sa.n_idx(); ++p) final_order.push_back(order[p]);
      a2_split = sa.split - static_cast<int>(demote.size());
      a_order = final_order;
      a = op_permute(a_in, a_order, a2_split);
    }
  }
  const Shape& s2 = a->shape;
  // positions in a2 of a's indices
  std::vector<int> pos_in_a2(sa.n_idx());
  for (int i = 0; i < sa.n_idx(); ++i) pos_in_a2[a_order[i]] = i;

  // 2. Replicate b over a2's span (skipped when it already is).
  TP b = b_in;
  Dist want{a->span(), 1, a->dist.offset};
  bool b_ok = b->shape.split == 0 && b->dist.offset <= a->dist.offset &&
              b->dist.offset + b->span() >= a->dist.offset + a->span();
  if (!b_ok) {
    if (b->shape.split != 0) {
      std::vector<int> ident(sb.n_idx());
      std::iota(ident.begin(), ident.end(), 0);
      b = op_permute(b, ident, 0);
    }
    b = op_rebcast(b, want);
  }

  // 3. Result of the local GEMMs: dims = open(a2 order) + open(b); dist of a.
  std::vector<int> a2_open;  // a2 positions that are open, in a2 order
  std::vector<int> a2_contr;  // a2 positions of the contracted indices, pair order
  for (int i = 0; i < s2.n_idx(); ++i)
    if (!ca[a_order[i]]) a2_open.push_back(i);
  for (int p : apos) a2_contr.push_back(pos_in_a2[p]);
  std::vector<Dim> c2dims;
  for (int i : a2_open) c2dims.push_back(s2.dims[i]);
  for (int p : b_open) c2dims.push_back(sb.dims[p]);
  int c2split = s2.split;  // all of a2's distributed indices are open
  TP c2 = make_tensor(r, Shape(c2dims, c2split), a->dist, true);
  if (c2->in_span) {
    // local permutation of a2's block: [open local][contracted]
    std::vector<Dim> ald = s2.local_dims();
    std::vector<int> ap;
    for (int i : a2_open)
      if (i >= s2.split) ap.push_back(i - s2.split);
    Dim M = 1, K = 1, N = 1;
    for (int i : ap) M *= ald[i];
    for (int i : a2_contr) {
      ap.push_back(i - s2.split);
      K *= s2.dims[i];
    }
    std::vector<int> bp;
    for (int q : bpos) bp.push_back(q);
    for (int q : b_open) {
      bp.push_back(q);
      N *= sb.dims[q];
    }
    std::shared_ptr<DevBuf> hb;
    const void* B = local_permuted(*b, sb.dims, bp, hb, r);
    if (is_identity(ap)) {
      zgemm(a->data(), B, c2->data(), M, N, K, r.stream);
    } else {
      // Fused layout permutation: A(m, k) = a[rowoff[m] + coloff[k]], read
      // straight from the tensor's block by the GEMM's operand loads.
      auto als = row_major_strides(ald);
      std::vector<Dim> rd, rs, cd, cs;
      size_t n_open_local = ap.size() - a2_contr.size();
      for (size_t i = 0; i < ap.size(); ++i) {
        (i < n_open_local ? rd : cd).push_back(ald[ap[i]]);
        (i < n_open_local ? rs : cs).push_back(als[ap[i]]);
      }
      auto min_stride = [](const std::vector<Dim>& d, const std::vector<Dim>& st) {
        Dim m = Dim(1) << 62;
        for (size_t i = 0; i < d.size(); ++i)
          if (d[i] > 1) m = std::min(m, st[i]);
        return m;
      };
      Dim min_r = min_stride(rd, rs), min_c = min_stride(cd, cs);
      // Row offsets: for a long M two small tables, rowoff(m) = hi[m >> sh] +
      // lo[m & (2^sh - 1)], instead of an M-entry table (16 MB at C1).
      Table ro, rohi;
      int ro_sh = 0;
      static const bool row_split = [] {
        const char* e = std::getenv("QTNH_ROW_SPLIT");
        return !(e && e[0] == '0');
      }();
      if (M > 4096 && row_split) {
        Dim best = 0;
        size_t best_sp = 0;
        for (size_t sp = 1; sp < rd.size(); ++sp) {
          Dim lo = 1, hi = 1;
          for (size_t i = 0; i < rd.size(); ++i) (i < sp ? hi : lo) *= rd[i];
          if ((lo & (lo - 1)) != 0) continue;
          Dim cost = std::max(lo, hi);
          if (!best || cost < best) {
            best = cost;
            best_sp = sp;
          }
        }
        if (best && best <= (Dim(1) << 16)) {
          const size_t sp = best_sp;
          ro = gather_table(r, {rd.begin() + sp, rd.end()}, {rs.begin() + sp, rs.end()});
          rohi = gather_table(r, {rd.begin(), rd.begin() + sp}, {rs.begin(), rs.begin() + sp});
          Dim lo = 1;
          for (size_t i = sp; i < rd.size(); ++i) lo *= rd[i];
          while ((Dim(1) << ro_sh) < lo) ++ro_sh;
        }
      }
      if (!ro) ro = gather_table(r, rd, rs);
      // A long K keeps its column offsets in shared memory as two small tables:
      // coloff(k) = hi[k >> sh] + lo[k & (2^sh - 1)] (inner digits -> lo).
      Table co, cohi;
      int co_sh = 0;
      if (K > 512) {
        for (size_t sp = 1; sp < cd.size() && !cohi; ++sp) {
          Dim lo = 1, hi = 1;
          for (size_t i = 0; i < cd.size(); ++i) (i < sp ? hi : lo) *= cd[i];
          if ((lo & (lo - 1)) == 0 && lo + hi <= 512) {
            co = gather_table(r, {cd.begin() + sp, cd.end()}, {cs.begin() + sp, cs.end()});
            cohi = gather_table(r, {cd.begin(), cd.begin() + sp}, {cs.begin(), cs.begin() + sp});
            while ((Dim(1) << co_sh) < lo) ++co_sh;
          }
        }
      }
      if (!co) co = gather_table(r, cd, cs);
      zgemm_gather_a(a->data(), ro.get(), co.get(), min_r <= min_c, B, c2->data(), M, N, K, r.stream, cohi.get(),
                     co_sh, rohi.get(), ro_sh);
    }
  }
  // 4. Restore the SPEC order / split when a was reshuffled.
  if (a == a_in) return c2;
  std::vector<int> perm;  // result position -> c2 position
  for (int p : a_open) perm.push_back(static_cast<int>(std::find(a2_open.begin(), a2_open.end(), pos_in_a2[p]) - a2_open.begin()));
  for (size_t j = 0; j < b_open.size(); ++j) perm.push_back(static_cast<int>(a2_open.size() + j));
  return op_permute(c2, perm, csplit);
}

void op_gate_apply(TP& t, const std::vector<int>& targets, const double* gate, bool diagonal) {
  QTNH_RANGE("qtnh::gate_apply");
  const Shape& s = t->shape;
  int k = static_cast<int>(targets.size());
  std::vector<char> is_t(s.n_idx(), 0);
  for (int q : targets) {
    if (q < 0 || q >= s.n_idx() || is_t[q]) throw_invalid("invalid gate targets");
    is_t[q] = 1;
  }
  std::vector<int> dist_t, local_t;
  for (int q : targets) (q < s.split ? dist_t : local_t).push_back(q);
  RankCtx& r = *t->rank;
  if (dist_t.empty()) {
    if (!t->in_span) return;
    std::vector<int> lt;
    for (int q : targets) lt.push_back(q - s.split);
    gate_local(t->data(), s.local_dims(), lt, gate, diagonal, r.stream);
    return;
  }
  std::vector<Dim> tdims;
  for (int q : targets) tdims.push_back(s.dims[q]);
  if (diagonal) {
    // Distributed target coordinates are fixed by this rank's block: apply the
    // slice of the diagonal that matches them, no communication.
    if (!t->in_span) return;
    auto cd = unflat(t->block, s.dist_dims());
    std::vector<Dim> ldims;
    for (int q : local_t) ldims.push_back(s.dims[q]);
    Dim nl = 1;
    for (Dim d : ldims) nl *= d;
    std::vector<double> sub(2 * nl);
    for (Dim j = 0; j < nl; ++j) {
      auto cl = unflat(j, ldims);
      std::vector<Dim> c(k);
      for (int i = 0, li = 0; i < k; ++i) c[i] = targets[i] < s.split ? cd[targets[i]] : cl[li++];
      Dim idx = flat(c, tdims);
      sub[2 * j] = gate[2 * idx];
      sub[2 * j + 1] = gate[2 * idx + 1];
    }
    if (local_t.empty()) {
      if (!(sub[0] == 1.0 && sub[1] == 0.0))
        scale_conj(t->data(), t->data(), s.local_size(), sub[0], sub[1], false, r.stream);
      return;
    }
    std::vector<int> lt;
    for (int q : local_t) lt.push_back(q - s.split);
    gate_local(t->data(), s.local_dims(), lt, sub.data(), true, r.stream);
    return;
  }
  if (dist_t.size() == 1 && s.dims[dist_t[0]] == 2 && peer_direct(r)) {
    // Gate fused with the exchange over peer memory: the two ranks whose blocks
    // differ only in the distributed target's bit see the pair as one virtual
    // tensor [2][local...] whose leading stride is the distance between their
    // buffers; each applies the gate to half of the fibers, loading and storing
    // the partner's amplitudes in place over NVLink. One pass instead of
    // swap -> apply -> swap back.
    auto members = span_ranks(*t);
    if (!t->in_span) return;
    const int q = dist_t[0];
    auto ddims = s.dist_dims();
    auto cd = unflat(t->block, ddims);
    const Dim nd = s.dist_size();
    auto ptrs = peer_pointers(r, members, t->data());
    char* grp[2];
    for (Dim j = 0; j < 2; ++j) {
      auto pc = cd;
      pc[q] = j;
      grp[j] = static_cast<char*>(ptrs[t->dist.home(flat(pc, ddims), nd, t->cycle, t->slot) - members.front()]);
    }
    auto ld = s.local_dims();
    std::vector<Dim> vdims{2}, vstr{(grp[1] - grp[0]) / 16};
    auto ls = row_major_strides(ld);
    vdims.insert(vdims.end(), ld.begin(), ld.end());
    vstr.insert(vstr.end(), ls.begin(), ls.end());
    std::vector<int> vt;
    Dim D = 1;
    for (int x : targets) {
      vt.push_back(x < s.split ? 0 : x - s.split + 1);
      D *= s.dims[x];
    }
    const Dim n_fib = 2 * s.local_size() / D, half = n_fib / 2;
    gate_strided(grp[0], vdims, vstr, vt, gate, false, r.stream, cd[q] == 0 ? 0 : half, cd[q] == 0 ? half : n_fib);
    peer_pointers(r, members, nullptr);
    return;
  }
  // Dense gate on distributed targets: swap each with a local non-target index of
  // the same size (dist<->local swap over NVLink), apply, swap back.
  std::vector<int> perm(s.n_idx());
  std::iota(perm.begin(), perm.end(), 0);
  std::vector<char> used(s.n_idx(), 0);
  std::vector<int> new_targets = targets;
  for (int i = 0; i < k; ++i) {
    int q = targets[i];
    if (q >= s.split) continue;
    // outermost free local index: the moving and staying regions are then
    // contiguous halves of the block (coalesced peer swap)
    int w = -1;
    for (int p = s.split; p < s.n_idx(); ++p)
      if (!is_t[p] && !used[p] && s.dims[p] == s.dims[q]) {
        w = p;
        break;
      }
    if (w < 0) throw_invalid("no local index to swap a distributed gate target with");
    used[w] = 1;
    std::swap(perm[q], perm[w]);
    new_targets[i] = w;
  }
  // in place: exchange each distributed target with its local partner, apply,
  // exchange back (no second copy of the state; only the moving halves travel)
  const int split = s.split;
  const std::vector<Dim> ldims = s.local_dims();
  std::vector<std::pair<int, int>> swaps;
  for (int i = 0; i < k; ++i)
    if (targets[i] < split) swaps.push_back({targets[i], new_targets[i]});
  for (auto& sw : swaps) op_swap_dist_local_inplace(t, sw.first, sw.second, swap_chunk_bytes());
  if (t->in_span) {
    std::vector<int> lt;
    for (int q : new_targets) lt.push_back(q - split);
    gate_local(t->data(), ldims, lt, gate, false, r.stream);
  }
  for (auto it = swaps.rbegin(); it != swaps.rend(); ++it)
    op_swap_dist_local_inplace(t, it->first, it->second, swap_chunk_bytes());
}

}  // namespace qtnhb

namespace qtnhb {

std::atomic<Dim> g_swap_chunk_bytes{[] {
  const char* e = std::getenv("QTNH_SWAP_CHUNK_BYTES");
  return e ? static_cast<Dim>(std::atoll(e)) : (Dim(1) << 31);
}()};
Dim swap_chunk_bytes() { return g_swap_chunk_bytes.load(); }
void set_swap_chunk_bytes(Dim v) { g_swap_chunk_bytes.store(std::max<Dim>(16, v)); }

void op_swap_indices(TP& t, int a, int b) {
  const Shape& s = t->shape;
  if (a < 0 || b < 0 || a >= s.n_idx() || b >= s.n_idx() || a == b) throw_invalid("invalid index pair to swap");
  if (s.dims[a] != s.dims[b]) throw_invalid("swapped indices must have equal dimensions");
  if (a >= s.split && b >= s.split) {
    if (t->in_span) swap_indices_local(t->data(), s.local_dims(), a - s.split, b - s.split, t->rank->stream);
    return;
  }
  if ((a < s.split) != (b < s.split)) {
    int da = a < s.split ? a : b, lb = a < s.split ? b : a;
    op_swap_dist_local_inplace(t, da, lb, swap_chunk_bytes());
    return;
  }
  std::vector<int> perm(s.n_idx());
  std::iota(perm.begin(), perm.end(), 0);
  std::swap(perm[a], perm[b]);
  t = op_permute(t, perm, s.split);
}

void op_qft_layer(TP& t, int j) {
  const Shape& s = t->shape;
  int n = s.n_idx();
  for (Dim d : s.dims)
    if (d != 2) throw_invalid("qft layer needs a qubit tensor (all dims 2)");
  if (j < 0 || j >= n) throw_invalid("qft layer qubit out of range");
  int lb = n - s.split;
  if (lb > 62) throw_invalid("too many local qubits");
  RankCtx& r = *t->rank;
  if (j >= s.split) {
    if (t->in_span) qft_layer_local(t->data(), lb, n - 1 - j, r.stream);
    return;
  }
  // distributed target: H through the dist<->local swap path, then the phases on
  // the ranks whose block has x_j = 1 (dist bits below j enter v as a constant).
  const double h[8] = {0.70710678118654752440, 0, 0.70710678118654752440, 0,
                       0.70710678118654752440, 0, -0.70710678118654752440, 0};
  const int split = s.split;  // s refers to the tensor op_gate_apply may replace
  op_gate_apply(t, {j}, h, false);
  if (!t->in_span) return;
  auto cd = unflat(t->block, t->shape.dist_dims());
  if (cd[j] == 0) return;
  int64_t v_off = 0;
  for (int l = j + 1; l < split; ++l) v_off = (v_off << 1) | cd[l];
  v_off <<= lb;
  qft_phase_local(t->data(), lb, v_off, n - 1 - j, r.stream);
}

void op_qft(TP& t, bool swaps) {
  QTNH_RANGE("qtnh::qft");
  // t may be replaced by the distributed-layer path: copy the metadata first
  const int n = t->shape.n_idx(), split = t->shape.split;
  for (Dim d : t->shape.dims)
    if (d != 2) throw_invalid("qft needs a qubit tensor (all dims 2)");
  int nb = n - split;
  if (nb > 62) throw_invalid("too many local qubits");
  RankCtx& r = *t->rank;
  // Peer-memory form: the layers of all distributed qubits in one pass, and the
  // distributed half of the bit reversal in another (see gate.cu).
  const bool fused = split >= 1 && split <= 4 && nb >= split && peer_direct(r);
  std::vector<void*> grp;
  Dim my_x = 0;
  if (fused && t->in_span) {
    auto members = span_ranks(*t);
    auto ptrs = peer_pointers(r, members, t->data());
    const Dim X = Dim(1) << split;
    for (Dim x = 0; x < X; ++x)
      grp.push_back(ptrs[t->dist.home(x, X, t->cycle, t->slot) - members.front()]);
    my_x = t->block;
    const Dim L = t->shape.local_size();
    qft_dist_layers(grp.data(), split, nb, my_x * L / X, (my_x + 1) * L / X, r.stream);
    peer_pointers(r, members, nullptr);
  } else if (!fused) {
    for (int j = 0; j < split; ++j) op_qft_layer(t, j);  // distributed targets
  }
  if (t->in_span && nb > 0) qft_local_fused(t->data(), nb, nb - 1, r.stream);
  if (!swaps) return;
  if (fused) {
    if (!t->in_span) return;
    auto members = span_ranks(*t);
    // the local layers of every member are done; pointers are valid until the
    // next peer_pointers call (IPC worlds re-import them), so regroup
    auto ptrs = peer_pointers(r, members, t->data());
    const Dim Xg = Dim(1) << split;
    for (Dim x = 0; x < Xg; ++x) grp[x] = ptrs[t->dist.home(x, Xg, t->cycle, t->slot) - members.front()];
    const Dim X = Dim(1) << split, M = t->shape.local_size() >> split;
    dist_bitrev(grp.data(), split, my_x * M / X, (my_x + 1) * M / X, r.stream);
    peer_pointers(r, members, nullptr);
    bitrev_hi_local(t->data(), n - 2 * split, split, r.stream);
    return;
  }
  if (t->shape.split == 0 && nb >= 10) {
    if (t->in_span) bitrev_local(t->data(), nb, t->rank->stream);
    return;
  }
  if (t->shape.split == split && 2 * split <= n) {
    // distributed qubit j <-> local qubit n-1-j (the k innermost), then one
    // in-place pass reversing the middle qubits [k, n-k) = the top n-2k local bits
    for (int j = 0; j < split; ++j) op_swap_indices(t, j, n - 1 - j);
    if (t->in_span) bitrev_hi_local(t->data(), n - 2 * split, split, t->rank->stream);
    return;
  }
  for (int j = 0; j < n / 2; ++j) op_swap_indices(t, j, n - 1 - j);
}

}  // namespace qtnhb

// ---- host-buffer contraction, streamed through the GPU --------------------------------
namespace qtnhb {

namespace {
struct PipeRes {
  cudaStream_t s[3] = {nullptr, nullptr, nullptr};
  cudaEvent_t ev[3][3];  // [slot][h2d, comp, d2h]
  int device = -1;
};
std::mutex g_pipe_mu;
std::map<const RankCtx*, PipeRes> g_pipes;  // per rank (ranks may share a device)

PipeRes& pipes(const RankCtx& r) {
  std::lock_guard<std::mutex> lk(g_pipe_mu);
  PipeRes& p = g_pipes[&r];
  if (p.device < 0) {
    p.device = r.device;
    for (int i = 0; i < 3; ++i) QTNH_CUDA(cudaStreamCreateWithFlags(&p.s[i], cudaStreamNonBlocking));
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) QTNH_CUDA(cudaEventCreateWithFlags(&p.ev[i][j], cudaEventDisableTiming));
  }
  return p;
}
}  // namespace

// C = contract(A, B) (SPEC.md:408 order) with A, B, C in host memory. A is cut
// along its leading open indices into chunks whose host memory is a few long
// runs and whose results are contiguous slices of C; three streams overlap the
// H2D of chunk i+1, the gather-GEMM of chunk i and the D2H of chunk i-1.
void contract_host(RankCtx& r, const std::vector<Dim>& da, const double* a, const std::vector<Dim>& db,
                   const double* b, const std::vector<int>& apos, const std::vector<int>& bpos, double* c,
                   std::vector<Dim>* c_dims, int target_chunks) {
  int na = static_cast<int>(da.size()), nb = static_cast<int>(db.size());
  std::vector<char> ca(na, 0), cb(nb, 0);
  if (apos.size() != bpos.size()) throw_invalid("contracted position lists differ in length");
  for (size_t i = 0; i < apos.size(); ++i) {
    int p = apos[i], q = bpos[i];
    if (p < 0 || p >= na || ca[p] || q < 0 || q >= nb || cb[q]) throw_invalid("invalid contracted index positions");
    if (da[p] != db[q]) throw_invalid("contracted dimensions differ");
    ca[p] = cb[q] = 1;
  }
  std::vector<int> a_open, b_open;
  for (int i = 0; i < na; ++i)
    if (!ca[i]) a_open.push_back(i);
  for (int i = 0; i < nb; ++i)
    if (!cb[i]) b_open.push_back(i);
  Dim M = 1, N = 1, K = 1;
  for (int p : a_open) M *= da[p];
  for (int q : b_open) N *= db[q];
  for (int p : apos) K *= da[p];
  if (c_dims) {
    c_dims->clear();
    for (int p : a_open) c_dims->push_back(da[p]);
    for (int q : b_open) c_dims->push_back(db[q]);
  }
  // chunk positions: leading positions 0..D-1; their open ones index the chunks
  int D = 0;
  Dim nchunks = 1, runs = 1;
  while (D < na && nchunks < target_chunks && runs <= 16) {
    if (ca[D]) runs *= da[D];
    else nchunks *= da[D];
    ++D;
  }
  auto sa = row_major_strides(da);
  std::vector<int> lead_open, lead_contr;
  for (int p = 0; p < D; ++p) (ca[p] ? lead_contr : lead_open).push_back(p);
  // chunk sub-tensor: dims [lead contracted..., da[D:]...]
  std::vector<Dim> sub_dims;
  std::vector<int> sub_pos_of(na, -1);
  for (int p : lead_contr) {
    sub_pos_of[p] = static_cast<int>(sub_dims.size());
    sub_dims.push_back(da[p]);
  }
  for (int p = D; p < na; ++p) {
    sub_pos_of[p] = static_cast<int>(sub_dims.size());
    sub_dims.push_back(da[p]);
  }
  Dim tail = 1;
  for (int p = D; p < na; ++p) tail *= da[p];
  const Dim chunk_elems = runs * tail, Mc = M / nchunks;
  auto sub_strides = row_major_strides(sub_dims);
  // gather tables of the chunk's A(m, k): rows = its open indices, cols = pairs
  std::vector<Dim> rd, rs, cd, cs;
  for (int p : a_open)
    if (p >= D) {
      rd.push_back(da[p]);
      rs.push_back(sub_strides[sub_pos_of[p]]);
    }
  for (int p : apos) {
    cd.push_back(da[p]);
    cs.push_back(sub_strides[sub_pos_of[p]]);
  }
  auto min_stride = [](const std::vector<Dim>& d, const std::vector<Dim>& st) {
    Dim m = Dim(1) << 62;
    for (size_t i = 0; i < d.size(); ++i)
      if (d[i] > 1) m = std::min(m, st[i]);
    return m;
  };
  bool rows_fastest = min_stride(rd, rs) <= min_stride(cd, cs);
  PipeRes& pr = pipes(r);
  cudaStream_t s_in = pr.s[0], s_cmp = pr.s[1], s_out = pr.s[2];
  // the caller's stream orders before us
  QTNH_CUDA(cudaEventRecord(pr.ev[0][0], r.stream));
  for (int i = 0; i < 3; ++i) QTNH_CUDA(cudaStreamWaitEvent(pr.s[i], pr.ev[0][0], 0));
  // resident B, permuted to [contracted (pair order) | open]
  DevBuf dB(static_cast<size_t>(K * N) * 16, r), dBp(static_cast<size_t>(K * N) * 16, r);
  DevBuf tabs(static_cast<size_t>(Mc + K) * 8, r);
  auto* ro = static_cast<int64_t*>(tabs.ptr);
  auto* co = ro + Mc;
  QTNH_CUDA(cudaMemcpyAsync(dB.ptr, b, K * N * 16, cudaMemcpyHostToDevice, r.stream));
  std::vector<int> bp(bpos.begin(), bpos.end());
  bp.insert(bp.end(), b_open.begin(), b_open.end());
  strided_copy(dB.ptr, dBp.ptr, permute_box(db, bp), false, r.stream);
  index_offsets(ro, Mc, rd, rs, r.stream);
  index_offsets(co, K, cd, cs, r.stream);
  QTNH_CUDA(cudaEventRecord(pr.ev[1][0], r.stream));
  QTNH_CUDA(cudaStreamWaitEvent(s_cmp, pr.ev[1][0], 0));
  const int slots = 3;
  std::vector<std::unique_ptr<DevBuf>> abuf, cbuf;
  for (int i = 0; i < slots && i < nchunks; ++i) {
    abuf.emplace_back(new DevBuf(static_cast<size_t>(chunk_elems) * 16, r));
    cbuf.emplace_back(new DevBuf(static_cast<size_t>(Mc * N) * 16, r));
  }
  // the slot buffers were allocated on r.stream: make the pipeline streams wait
  QTNH_CUDA(cudaEventRecord(pr.ev[2][0], r.stream));
  for (int i = 0; i < 3; ++i) QTNH_CUDA(cudaStreamWaitEvent(pr.s[i], pr.ev[2][0], 0));
  std::vector<Dim> lo_dims;
  for (int p : lead_open) lo_dims.push_back(da[p]);
  std::vector<Dim> lc_dims;
  for (int p : lead_contr) lc_dims.push_back(da[p]);
  std::vector<bool> used(slots, false);
  for (Dim ch = 0; ch < nchunks; ++ch) {
    int sl = static_cast<int>(ch % slots);
    auto co_open = unflat(ch, lo_dims);
    Dim base = 0;
    for (size_t i = 0; i < lead_open.size(); ++i) base += co_open[i] * sa[lead_open[i]];
    // H2D: after the compute that last read this slot
    if (used[sl]) QTNH_CUDA(cudaStreamWaitEvent(s_in, pr.ev[sl][1], 0));
    for (Dim rr = 0; rr < runs; ++rr) {
      auto cr = unflat(rr, lc_dims);
      Dim off = base;
      for (size_t i = 0; i < lead_contr.size(); ++i) off += cr[i] * sa[lead_contr[i]];
      QTNH_CUDA(cudaMemcpyAsync(static_cast<char*>(abuf[sl]->ptr) + rr * tail * 16, a + 2 * off, tail * 16,
                                cudaMemcpyHostToDevice, s_in));
    }
    QTNH_CUDA(cudaEventRecord(pr.ev[sl][0], s_in));
    // compute: after the H2D of this chunk and the D2H that last read the slot
    QTNH_CUDA(cudaStreamWaitEvent(s_cmp, pr.ev[sl][0], 0));
    if (used[sl]) QTNH_CUDA(cudaStreamWaitEvent(s_cmp, pr.ev[sl][2], 0));
    zgemm_gather_a(abuf[sl]->ptr, ro, co, rows_fastest, dBp.ptr, cbuf[sl]->ptr, Mc, N, K, s_cmp);
    QTNH_CUDA(cudaEventRecord(pr.ev[sl][1], s_cmp));
    // D2H of the contiguous C slice
    QTNH_CUDA(cudaStreamWaitEvent(s_out, pr.ev[sl][1], 0));
    QTNH_CUDA(cudaMemcpyAsync(c + 2 * ch * Mc * N, cbuf[sl]->ptr, Mc * N * 16, cudaMemcpyDeviceToHost, s_out));
    QTNH_CUDA(cudaEventRecord(pr.ev[sl][2], s_out));
    used[sl] = true;
  }
  // the caller's stream (and the buffers' release) come after the pipeline
  for (int i = 0; i < 3; ++i) {
    QTNH_CUDA(cudaEventRecord(pr.ev[i][0], pr.s[i]));
    QTNH_CUDA(cudaStreamWaitEvent(r.stream, pr.ev[i][0], 0));
  }
}

}  // namespace qtnhb
