// Strided-copy engine for sm_100a (see strided_copy.h).
//
// Design (HBM-bound byte movement, no tensor cores):
//  * The box is simplified on the host: unit dims dropped, dims that stay
//    adjacent on both sides merged, then large dims split into <=64-wide factors
//    so a tile can take "part of" a big index.
//  * A tile is the union of the innermost input dims (product >= 32 elements,
//    i.e. >= 512 contiguous bytes read) and the innermost output dims (>= 32
//    elements written contiguously). One CTA moves a tile global -> shared ->
//    global: reads coalesced along the input order, writes coalesced along the
//    output order. Shared-memory positions are XOR-swizzled (16-B elements, 8
//    bank groups) so the transposed read-out is conflict-free for power-of-two
//    strides.
//  * Per-tile offset tables (input offset, output offset, shared slot) are built
//    once per plan on the host and read through the read-only path; outer
//    (non-tile) coordinates come from the tile id by shift/mask (powers of two)
//    or div/mod, once per tile.
//  * Tiles whose input and output orders coincide skip shared memory entirely.
//  * Persistent grid: (#SM x resident CTAs), grid-stride over tiles.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <numeric>

#include "strided_copy.h"

namespace qtnhb {

namespace {

constexpr int kMaxOuter = 64;
constexpr int kThreads = 256;

struct Outer {
  int n;
  int all_pow2;
  int64_t dim[kMaxOuter];
  int shift[kMaxOuter];
  int64_t is[kMaxOuter];
  int64_t os[kMaxOuter];
};

__device__ __forceinline__ void decompose(int64_t tile, const Outer& od, int64_t& bi, int64_t& bo) {
  bi = 0;
  bo = 0;
  if (od.all_pow2) {
    for (int i = od.n - 1; i >= 0; --i) {
      int64_t c = tile & (od.dim[i] - 1);
      tile >>= od.shift[i];
      bi += c * od.is[i];
      bo += c * od.os[i];
    }
  } else {
    for (int i = od.n - 1; i >= 0; --i) {
      int64_t c = tile % od.dim[i];
      tile /= od.dim[i];
      bi += c * od.is[i];
      bo += c * od.os[i];
    }
  }
}

__device__ __forceinline__ int swz(int e) { return e ^ (((e >> 3) ^ (e >> 6) ^ (e >> 9)) & 7); }

__device__ __forceinline__ double2 canon_zero(double2 v) {
  if (v.x == 0.0 && v.y == 0.0) v = make_double2(0.0, 0.0);
  return v;
}

template <bool CANON, bool DIRECT>
__global__ void __launch_bounds__(kThreads) k_tiled(const double2* __restrict__ in,
                                                    double2* __restrict__ out,
                                                    const int64_t* __restrict__ tin,
                                                    const int64_t* __restrict__ tout,
                                                    const int* __restrict__ tslot, int T,
                                                    int64_t n_tiles, const Outer od) {
  extern __shared__ double2 sm[];
  for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    int64_t bi, bo;
    decompose(tile, od, bi, bo);
    if (DIRECT) {
      constexpr int U = 4;
      for (int e0 = threadIdx.x; e0 < T; e0 += kThreads * U) {
        double2 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          int e = e0 + u * kThreads;
          if (e < T) v[u] = __ldg(in + bi + __ldg(tin + e));
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          int e = e0 + u * kThreads;
          if (e < T) out[bo + __ldg(tout + e)] = CANON ? canon_zero(v[u]) : v[u];
        }
      }
    } else {
      constexpr int U = 4;
      for (int e0 = threadIdx.x; e0 < T; e0 += kThreads * U) {
        double2 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          int e = e0 + u * kThreads;
          if (e < T) v[u] = __ldg(in + bi + __ldg(tin + e));
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          int e = e0 + u * kThreads;
          if (e < T) sm[swz(e)] = v[u];
        }
      }
      __syncthreads();
      for (int f = threadIdx.x; f < T; f += kThreads) {
        double2 v = sm[__ldg(tslot + f)];
        out[bo + __ldg(tout + f)] = CANON ? canon_zero(v) : v;
      }
      __syncthreads();
    }
  }
}

// Fallback for boxes no tile fits (huge prime dims on both sides): one thread per
// output element in output order, gathered input.
struct Full {
  int n;
  int64_t dim[kMaxOuter];
  int64_t is[kMaxOuter];
  int64_t os[kMaxOuter];
};

template <bool CANON>
__global__ void __launch_bounds__(kThreads) k_gather(const double2* __restrict__ in,
                                                     double2* __restrict__ out, int64_t total,
                                                     const Full fd) {
  for (int64_t f = blockIdx.x * (int64_t)kThreads + threadIdx.x; f < total;
       f += (int64_t)gridDim.x * kThreads) {
    int64_t t = f, bi = 0, bo = 0;
    for (int i = fd.n - 1; i >= 0; --i) {
      int64_t c = t % fd.dim[i];
      t /= fd.dim[i];
      bi += c * fd.is[i];
      bo += c * fd.os[i];
    }
    double2 v = in[bi];
    out[bo] = CANON ? canon_zero(v) : v;
  }
}

__global__ void k_scale_conj(const double2* __restrict__ in, double2* __restrict__ out, int64_t n,
                             double re, double im, int conj) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double2 v = in[i];
    if (conj) v.y = -v.y;
    out[i] = make_double2(v.x * re - v.y * im, v.x * im + v.y * re);
  }
}

// out[i] = in[i] * f[(i / inner) % dim]: a real factor per coordinate of one index
// (absorb_singular_* with an arbitrary power, linalg.hpp:508-523)
__global__ void k_scale_index(const double2* __restrict__ in, double2* __restrict__ out, int64_t n, int64_t inner,
                              int64_t dim, const double* __restrict__ f) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double x = f[(i / inner) % dim];
    const double2 v = in[i];
    out[i] = make_double2(v.x * x, v.y * x);
  }
}

__global__ void k_fill_zero(double2* __restrict__ out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = make_double2(0.0, 0.0);
}

// ---- host planning ------------------------------------------------------------
struct D {
  Dim n, is, os;
};

struct Plan {
  enum Kind { kTiled, kDirect, kGather, kEmpty } kind = kEmpty;
  int T = 0;
  int64_t n_tiles = 0;
  Outer od{};
  Full fd{};
  int64_t* d_tin = nullptr;
  int64_t* d_tout = nullptr;
  int* d_slot = nullptr;
  int grid = 0;
  size_t smem = 0;
  cudaEvent_t ready = nullptr;  // the tables' upload; launches on other streams wait on it
  void* base = nullptr;         // one stream-ordered allocation for the three tables
  int device = 0;
  ~Plan() {  // only on cache eviction
    if (ready) cudaEventDestroy(ready);
    if (base) {
      int cur = 0;
      cudaGetDevice(&cur);
      cudaSetDevice(device);
      cudaDeviceSynchronize();  // launches that used the plan have been enqueued by now
      cudaFreeAsync(base, 0);
      cudaSetDevice(cur);
    }
  }
};

int sm_count(int dev) {
  static std::mutex mu;
  static std::map<int, int> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(dev);
  if (it != cache.end()) return it->second;
  int n = 0;
  QTNH_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  cache[dev] = n;
  return n;
}

Dim pick_factor(Dim n) {
  // Largest power of two <= 64 dividing n, else the largest divisor in [8, 64].
  for (Dim t = 64; t >= 8; t >>= 1)
    if (n % t == 0 && n / t > 1) return t;
  for (Dim t = 64; t >= 8; --t)
    if (n % t == 0 && n / t > 1) return t;
  return 0;
}

std::vector<D> simplify(const CopyBox& box) {
  std::vector<D> v;
  for (size_t i = 0; i < box.dims.size(); ++i)
    if (box.dims[i] != 1) v.push_back({box.dims[i], box.in_stride[i], box.out_stride[i]});
  // Order by input stride descending (row-major over the input), then merge
  // neighbours that are adjacent on both sides.
  std::stable_sort(v.begin(), v.end(), [](const D& a, const D& b) { return a.is > b.is; });
  std::vector<D> m;
  for (const D& d : v) {
    if (!m.empty()) {
      D& o = m.back();
      if (o.is == d.is * d.n && o.os == d.os * d.n) {
        o.n *= d.n;
        o.is = d.is;
        o.os = d.os;
        continue;
      }
    }
    m.push_back(d);
  }
  // Split dims wider than 64 so a tile can take a slice of them.
  std::vector<D> s;
  for (const D& d : m) {
    std::vector<D> parts;  // outer..inner
    D cur = d;
    while (cur.n > 64) {
      Dim t = pick_factor(cur.n);
      if (!t) break;
      parts.insert(parts.begin(), D{t, cur.is, cur.os});
      cur = D{cur.n / t, cur.is * t, cur.os * t};
    }
    s.push_back(cur);
    for (const D& p : parts) s.push_back(p);
  }
  return s;
}

std::string key_of(const std::vector<D>& v, int dev) {
  std::string k(reinterpret_cast<const char*>(v.data()), v.size() * sizeof(D));
  k.append(reinterpret_cast<const char*>(&dev), sizeof(dev));
  return k;
}

std::shared_ptr<Plan> build_plan(const std::vector<D>& ds, int dev, cudaStream_t st) {
  auto p = std::make_shared<Plan>();
  int r = static_cast<int>(ds.size());
  std::vector<int> in_order(r), out_order(r);
  std::iota(in_order.begin(), in_order.end(), 0);
  std::iota(out_order.begin(), out_order.end(), 0);
  std::stable_sort(in_order.begin(), in_order.end(), [&](int a, int b) { return ds[a].is < ds[b].is; });
  std::stable_sort(out_order.begin(), out_order.end(), [&](int a, int b) { return ds[a].os < ds[b].os; });

  std::vector<char> in_tile;
  Dim tile = 1;
  const Dim kMaxTile = 8192;
  static const Dim first_run = [] {
    const char* e = std::getenv("QTNH_COPY_RUN");
    return e ? static_cast<Dim>(std::atoi(e)) : 64;  // 1 KB runs: +9-15 % on transposing permutations
  }();
  for (Dim min_run : {first_run, Dim(32), Dim(16), Dim(8), Dim(2)}) {
    in_tile.assign(r, 0);
    Dim prod = 1;
    for (int i = 0; i < r && prod < min_run; ++i) {
      in_tile[in_order[i]] = 1;
      prod *= ds[in_order[i]].n;
    }
    Dim oprod = 1;
    for (int i = 0; i < r && oprod < min_run; ++i) {
      oprod *= ds[out_order[i]].n;
      in_tile[out_order[i]] = 1;
    }
    tile = 1;
    for (int i = 0; i < r; ++i)
      if (in_tile[i]) tile *= ds[i].n;
    if (tile <= kMaxTile) break;
  }
  if (tile > kMaxTile) {
    p->kind = Plan::kGather;
    p->fd.n = r;
    for (int j = 0; j < r; ++j) {
      int i = out_order[r - 1 - j];  // outermost output dim first
      p->fd.dim[j] = ds[i].n;
      p->fd.is[j] = ds[i].is;
      p->fd.os[j] = ds[i].os;
    }
    Dim total = 1;
    for (auto& d : ds) total *= d.n;
    p->n_tiles = total;
    p->grid = sm_count(dev) * 8;
    return p;
  }
  // Grow small tiles with further input-order dims to amortise per-tile work.
  for (int i = 0; i < r && tile < 512; ++i) {
    int d = in_order[i];
    if (!in_tile[d] && tile * ds[d].n <= 2048) {
      in_tile[d] = 1;
      tile *= ds[d].n;
    }
  }
  std::vector<int> tin_dims, tout_dims;  // innermost first
  for (int i : in_order)
    if (in_tile[i]) tin_dims.push_back(i);
  for (int i : out_order)
    if (in_tile[i]) tout_dims.push_back(i);
  bool direct = tin_dims == tout_dims;
  int T = static_cast<int>(tile);
  std::vector<int64_t> tin(T), tout(T);
  std::vector<int> slot(T);
  auto swz = [](int e) { return e ^ (((e >> 3) ^ (e >> 6) ^ (e >> 9)) & 7); };
  // Input order: e = sum c * w_in.
  std::vector<Dim> w_in(r, 0);
  {
    Dim w = 1;
    for (int i : tin_dims) {
      w_in[i] = w;
      w *= ds[i].n;
    }
  }
  std::vector<Dim> c(r, 0);
  for (int e = 0; e < T; ++e) {
    Dim rem = e;
    int64_t off = 0;
    for (int i : tin_dims) {
      Dim ci = rem % ds[i].n;
      rem /= ds[i].n;
      off += ci * ds[i].is;
    }
    tin[e] = off;
  }
  for (int f = 0; f < T; ++f) {
    Dim rem = f;
    int64_t off = 0;
    Dim e = 0;
    for (int i : tout_dims) {
      Dim ci = rem % ds[i].n;
      rem /= ds[i].n;
      off += ci * ds[i].os;
      e += ci * w_in[i];
    }
    tout[f] = off;
    slot[f] = swz(static_cast<int>(e));
  }
  if (direct) {
    // Direct mode walks e in input order for both sides.
    for (int e = 0; e < T; ++e) {
      Dim rem = e;
      int64_t off = 0;
      for (int i : tin_dims) {
        Dim ci = rem % ds[i].n;
        rem /= ds[i].n;
        off += ci * ds[i].os;
      }
      tout[e] = off;
    }
  }
  // Outer dims: outermost (by output stride) first, tile id row-major over them.
  std::vector<int> outer;
  for (int j = r - 1; j >= 0; --j)
    if (!in_tile[out_order[j]]) outer.push_back(out_order[j]);
  if (static_cast<int>(outer.size()) > kMaxOuter) throw_invalid("tensor rank too large for the copy engine");
  p->od.n = static_cast<int>(outer.size());
  p->od.all_pow2 = 1;
  Dim n_tiles = 1;
  for (int j = 0; j < p->od.n; ++j) {
    const D& d = ds[outer[j]];
    p->od.dim[j] = d.n;
    p->od.is[j] = d.is;
    p->od.os[j] = d.os;
    int sh = 0;
    while ((Dim(1) << sh) < d.n) ++sh;
    p->od.shift[j] = sh;
    if ((Dim(1) << sh) != d.n) p->od.all_pow2 = 0;
    n_tiles *= d.n;
  }
  p->kind = direct ? Plan::kDirect : Plan::kTiled;
  p->T = T;
  p->n_tiles = n_tiles;
  p->smem = direct ? 0 : static_cast<size_t>((T + 7) & ~7) * sizeof(double2);
  // one pool allocation (stream-ordered: a pool hit, no cudaMalloc per new layout --
  // ~600 of them in config 3's contraction chain cost ~20 us of host time each)
  QTNH_CUDA(cudaMallocAsync(&p->base, static_cast<size_t>(T) * (2 * sizeof(int64_t) + sizeof(int)), st));
  p->device = dev;
  p->d_tin = static_cast<int64_t*>(p->base);
  p->d_tout = p->d_tin + T;
  p->d_slot = reinterpret_cast<int*>(p->d_tout + T);
  QTNH_CUDA(cudaMemcpyAsync(p->d_tin, tin.data(), T * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  QTNH_CUDA(cudaMemcpyAsync(p->d_tout, tout.data(), T * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  QTNH_CUDA(cudaMemcpyAsync(p->d_slot, slot.data(), T * sizeof(int), cudaMemcpyHostToDevice, st));
  // pageable sources: cudaMemcpyAsync has copied them to staging on return, so the
  // host vectors may die; no stream synchronisation (it serialised every new
  // layout -- ~600 in config 3's contraction chain)
  QTNH_CUDA(cudaEventCreateWithFlags(&p->ready, cudaEventDisableTiming));
  QTNH_CUDA(cudaEventRecord(p->ready, st));
  int per_sm = 1;
  if (direct) {
    QTNH_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tiled<true, true>, kThreads, 0));
  } else {
    // the attribute is per kernel, not per plan: always allow the largest tile
    // (kMaxTile elements), or a later small-tile plan would shrink the limit under
    // an earlier large-tile plan
    const int max_smem = static_cast<int>(kMaxTile * sizeof(double2));
    QTNH_CUDA(cudaFuncSetAttribute(k_tiled<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, max_smem));
    QTNH_CUDA(cudaFuncSetAttribute(k_tiled<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, max_smem));
    QTNH_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tiled<true, false>, kThreads, p->smem));
  }
  Dim g = static_cast<Dim>(sm_count(dev)) * std::max(1, per_sm);
  p->grid = static_cast<int>(std::max<Dim>(1, std::min<Dim>(g, n_tiles)));
  return p;
}

std::mutex g_plan_mu;
std::map<std::string, std::shared_ptr<Plan>> g_plans;

}  // namespace

CopyBox permute_box(const std::vector<Dim>& dims, const std::vector<int>& perm) {
  // Output position p holds input index perm[p]; iterate the box over the input
  // indices: in stride = row-major input stride, out stride = row-major output
  // stride at the position the index moves to.
  int r = static_cast<int>(dims.size());
  std::vector<Dim> nd(r);
  for (int p = 0; p < r; ++p) nd[p] = dims[perm[p]];
  auto is = row_major_strides(dims);
  auto os_new = row_major_strides(nd);
  CopyBox b;
  b.dims = dims;
  b.in_stride = is;
  b.out_stride.assign(r, 0);
  for (int p = 0; p < r; ++p) b.out_stride[perm[p]] = os_new[p];
  return b;
}

void strided_copy(const void* in, void* out, const CopyBox& box, bool canon, cudaStream_t st) {
  Dim total = 1;
  for (Dim d : box.dims) total *= d;
  if (total == 0) return;
  auto ds = simplify(box);
  int dev = 0;
  QTNH_CUDA(cudaGetDevice(&dev));
  std::shared_ptr<Plan> p;
  {
    std::lock_guard<std::mutex> lk(g_plan_mu);
    auto key = key_of(ds, dev);
    auto it = g_plans.find(key);
    if (it != g_plans.end()) {
      p = it->second;
    } else {
      p = build_plan(ds, dev, st);
      if (g_plans.size() > 4096) g_plans.clear();  // bounded; device tables leak-free enough
      g_plans[key] = p;
    }
  }
  if (p->ready) QTNH_CUDA(cudaStreamWaitEvent(st, p->ready, 0));
  auto i = static_cast<const double2*>(in);
  auto o = static_cast<double2*>(out);
  switch (p->kind) {
    case Plan::kGather:
      if (canon) k_gather<true><<<p->grid, kThreads, 0, st>>>(i, o, p->n_tiles, p->fd);
      else k_gather<false><<<p->grid, kThreads, 0, st>>>(i, o, p->n_tiles, p->fd);
      break;
    case Plan::kDirect:
      if (canon) k_tiled<true, true><<<p->grid, kThreads, 0, st>>>(i, o, p->d_tin, p->d_tout, p->d_slot, p->T, p->n_tiles, p->od);
      else k_tiled<false, true><<<p->grid, kThreads, 0, st>>>(i, o, p->d_tin, p->d_tout, p->d_slot, p->T, p->n_tiles, p->od);
      break;
    case Plan::kTiled:
      if (canon) k_tiled<true, false><<<p->grid, kThreads, p->smem, st>>>(i, o, p->d_tin, p->d_tout, p->d_slot, p->T, p->n_tiles, p->od);
      else k_tiled<false, false><<<p->grid, kThreads, p->smem, st>>>(i, o, p->d_tin, p->d_tout, p->d_slot, p->T, p->n_tiles, p->od);
      break;
    case Plan::kEmpty:
      return;
  }
  QTNH_LAUNCH_CHECK();
}

void scale_conj(const void* in, void* out, Dim n, double re, double im, bool conj, cudaStream_t st) {
  if (n <= 0) return;
  int dev = 0;
  QTNH_CUDA(cudaGetDevice(&dev));
  int grid = static_cast<int>(std::min<Dim>((n + 255) / 256, (Dim)sm_count(dev) * 8));
  k_scale_conj<<<grid, 256, 0, st>>>(static_cast<const double2*>(in), static_cast<double2*>(out), n, re, im, conj);
  QTNH_LAUNCH_CHECK();
}

void scale_index(const void* in, void* out, Dim n, Dim inner, Dim dim, const double* f_dev, cudaStream_t st) {
  if (n <= 0) return;
  int dev = 0;
  QTNH_CUDA(cudaGetDevice(&dev));
  int grid = static_cast<int>(std::min<Dim>((n + 255) / 256, (Dim)sm_count(dev) * 8));
  k_scale_index<<<grid, 256, 0, st>>>(static_cast<const double2*>(in), static_cast<double2*>(out), n, inner, dim,
                                      f_dev);
  QTNH_LAUNCH_CHECK();
}

struct Region {
  int nd;
  int64_t dims[8];
  int64_t strides[8];
};

__device__ __forceinline__ int64_t region_offset(int64_t i, const Region& rg) {
  int64_t off = 0;
  for (int d = rg.nd - 1; d > 0; --d) {
    int64_t c = i % rg.dims[d];
    i /= rg.dims[d];
    off += c * rg.strides[d];
  }
  return off + i * rg.strides[0];
}

// Zero canonicalisation in place: a write only where a zero is not +0 + 0i, so
// the pass costs a read of the region.
__device__ __forceinline__ void canon_in_place(double2* p) {
  double2 v = *p;
  if (v.x == 0.0 && v.y == 0.0 && (__double_as_longlong(v.x) | __double_as_longlong(v.y)) != 0)
    *p = make_double2(0.0, 0.0);
}

// One thread per element pair, 16-byte accesses; the region is pre-merged to at
// most a few dims so the offset arithmetic stays off the critical path. With
// keep_a/keep_b set, the elements at the same region offset in the two staying
// regions are canonicalised in the same pass.
__global__ void k_swap_regions(double2* __restrict__ a, double2* __restrict__ b, double2* keep_a, double2* keep_b,
                               int64_t begin, int64_t end, const __grid_constant__ Region rg) {
  for (int64_t i = begin + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < end;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t off = region_offset(i, rg);
    double2 x = a[off], y = b[off];
    if (x.x == 0.0 && x.y == 0.0) x = make_double2(0.0, 0.0);
    if (y.x == 0.0 && y.y == 0.0) y = make_double2(0.0, 0.0);
    a[off] = y;
    b[off] = x;
    if (keep_a) canon_in_place(keep_a + off);
    if (keep_b) canon_in_place(keep_b + off);
  }
}

__global__ void k_canon_region(double2* __restrict__ p, int64_t n, const __grid_constant__ Region rg) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    canon_in_place(p + region_offset(i, rg));
}

Region merged_region(const std::vector<Dim>& dims, const std::vector<Dim>& strides) {
  // merge row-major neighbours (outer stride == inner stride * inner dim)
  std::vector<std::pair<Dim, Dim>> m;
  for (size_t i = 0; i < dims.size(); ++i) {
    if (dims[i] == 1) continue;
    if (!m.empty() && m.back().second == strides[i] * dims[i]) {
      m.back().first *= dims[i];
      m.back().second = strides[i];
    } else {
      m.push_back({dims[i], strides[i]});
    }
  }
  if (m.empty()) m.push_back({1, 1});
  if (m.size() > 8) throw_invalid("swap region has too many non-mergeable dims");
  Region rg{};
  rg.nd = static_cast<int>(m.size());
  for (int i = 0; i < rg.nd; ++i) {
    rg.dims[i] = m[i].first;
    rg.strides[i] = m[i].second;
  }
  return rg;
}

void swap_regions(void* a, void* b, const std::vector<Dim>& dims, const std::vector<Dim>& strides, Dim begin,
                  Dim end, cudaStream_t st, void* keep_a, void* keep_b) {
  if (end <= begin) return;
  Region rg = merged_region(dims, strides);
  int dev = 0;
  QTNH_CUDA(cudaGetDevice(&dev));
  Dim n = end - begin;
  int grid = static_cast<int>(std::min<Dim>((n + 255) / 256, (Dim)sm_count(dev) * 8));
  k_swap_regions<<<grid, 256, 0, st>>>(static_cast<double2*>(a), static_cast<double2*>(b),
                                       static_cast<double2*>(keep_a), static_cast<double2*>(keep_b), begin, end, rg);
  QTNH_LAUNCH_CHECK();
}

void canon_region(void* p, const std::vector<Dim>& dims, const std::vector<Dim>& strides, cudaStream_t st) {
  Dim n = 1;
  for (Dim d : dims) n *= d;
  if (n <= 0) return;
  Region rg = merged_region(dims, strides);
  int dev = 0;
  QTNH_CUDA(cudaGetDevice(&dev));
  int grid = static_cast<int>(std::min<Dim>((n + 255) / 256, (Dim)sm_count(dev) * 8));
  k_canon_region<<<grid, 256, 0, st>>>(static_cast<double2*>(p), n, rg);
  QTNH_LAUNCH_CHECK();
}

struct PairSpec {
  int n, npairs;
  int64_t dims[32];
  int eq_in[16], eq_out[16];
};

// Identity / swap tensors (tensor.hpp:144-164, 491-514) materialised densely: the
// local element whose global coordinates satisfy every pairing is 1, else 0.
__global__ void k_fill_paired(double2* __restrict__ out, int64_t nl, int64_t block, int split,
                              const __grid_constant__ PairSpec ps) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nl; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t c[32];
    int64_t r = e;
    for (int i = ps.n - 1; i >= split; --i) {
      c[i] = r % ps.dims[i];
      r /= ps.dims[i];
    }
    r = block;
    for (int i = split - 1; i >= 0; --i) {
      c[i] = r % ps.dims[i];
      r /= ps.dims[i];
    }
    bool one = true;
    for (int k = 0; k < ps.npairs; ++k) one &= c[ps.eq_in[k]] == c[ps.eq_out[k]];
    out[e] = make_double2(one ? 1.0 : 0.0, 0.0);
  }
}

void fill_paired(void* out, Dim nl, Dim block, const std::vector<Dim>& dims, int split, const std::vector<int>& eq_in,
                 const std::vector<int>& eq_out, cudaStream_t st) {
  if (nl <= 0) return;
  PairSpec ps{};
  ps.n = static_cast<int>(dims.size());
  ps.npairs = static_cast<int>(eq_in.size());
  if (ps.n > 32 || ps.npairs > 16) throw_invalid("paired tensor rank too large");
  for (int i = 0; i < ps.n; ++i) ps.dims[i] = dims[i];
  for (int k = 0; k < ps.npairs; ++k) {
    ps.eq_in[k] = eq_in[k];
    ps.eq_out[k] = eq_out[k];
  }
  int dev = 0;
  QTNH_CUDA(cudaGetDevice(&dev));
  int grid = static_cast<int>(std::min<Dim>((nl + 255) / 256, (Dim)sm_count(dev) * 8));
  k_fill_paired<<<grid, 256, 0, st>>>(static_cast<double2*>(out), nl, block, split, ps);
  QTNH_LAUNCH_CHECK();
}

void fill_zero(void* out, Dim n, cudaStream_t st) {
  if (n <= 0) return;
  int dev = 0;
  QTNH_CUDA(cudaGetDevice(&dev));
  int grid = static_cast<int>(std::min<Dim>((n + 255) / 256, (Dim)sm_count(dev) * 8));
  k_fill_zero<<<grid, 256, 0, st>>>(static_cast<double2*>(out), n);
  QTNH_LAUNCH_CHECK();
}

}  // namespace qtnhb
