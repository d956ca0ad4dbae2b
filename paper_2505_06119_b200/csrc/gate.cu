// In-place gate application on a dense local block (sm_100a, HBM-bound).
//
// Reference path: a gate is a separate tensor contracted with the state
// (PAPER.md III-E-1), i.e. tensor_to_matrix of both operands,
// a K = 2..4 zgemm and matrix_to_tensor (linalg.hpp:208-400), followed by a
// permute that puts the gate outputs back in place. For a D x D gate on a
// state of N elements that is the same arithmetic as y_f = G x_f on each of the
// N/D "fibers" x_f (the D elements that differ only in the target coordinates).
// Here one thread owns one fiber: D coalesced 16-byte loads (consecutive threads
// take consecutive non-target coordinates), D^2 complex FMAs from the gate held
// in the kernel parameter bank (warp-uniform broadcast), D stores. One read and
// one write of the state per gate: 32 B/element, the HBM roofline.
// Diagonal gates touch only the fibers' elements whose diagonal entry is not 1.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include <mutex>
#include <tuple>
#include <vector>

#include "ops.h"
#include "tma.h"

namespace qtnhb {

namespace {

constexpr int kMaxD = 16;
constexpr int kMaxSeg = 24;

struct GateArgs {
  int D;
  int nseg;
  int64_t seg_size[kMaxSeg];   // innermost segment last
  int64_t seg_stride[kMaxSeg];
  int seg_shift[kMaxSeg];
  int64_t off[kMaxD * 4];      // element offsets of the D (or listed diagonal) entries
  double2 g[kMaxD * kMaxD];    // row-major gate, or diagonal values
  int nd;                      // diagonal: number of listed entries
  int64_t f0;                  // first fiber of this launch
};

template <bool POW2>
__device__ __forceinline__ int64_t fiber_base(int64_t f, const GateArgs& a) {
  int64_t base = 0;
#pragma unroll 4
  for (int j = a.nseg - 1; j >= 0; --j) {
    int64_t c;
    if (POW2) {
      c = f & (a.seg_size[j] - 1);
      f >>= a.seg_shift[j];
    } else {
      c = f % a.seg_size[j];
      f /= a.seg_size[j];
    }
    base += c * a.seg_stride[j];
  }
  return base;
}

// F fibers per thread per iteration (strided by the grid size, so every load
// instruction stays coalesced): 2F..8 independent 16-byte loads in flight per
// thread for the small gates, which are otherwise latency- rather than
// bandwidth-limited.
template <int D, bool POW2>
__global__ void __launch_bounds__(256) k_gate_dense(double2* __restrict__ psi, int64_t n_fibers,
                                                    const __grid_constant__ GateArgs a) {
  constexpr int F = D <= 4 ? 4 : (D <= 8 ? 2 : 1);
  const int64_t S = (int64_t)gridDim.x * blockDim.x;
  for (int64_t f0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f0 < n_fibers; f0 += F * S) {
    int64_t base[F];
    double2 x[F][D];
#pragma unroll
    for (int u = 0; u < F; ++u) {
      const int64_t f = f0 + u * S;
      base[u] = f < n_fibers ? fiber_base<POW2>(f + a.f0, a) : -1;
      if (base[u] >= 0) {
#pragma unroll
        for (int d = 0; d < D; ++d) x[u][d] = psi[base[u] + a.off[d]];
      }
    }
#pragma unroll
    for (int u = 0; u < F; ++u) {
      if (base[u] < 0) continue;
      // D = 16: one output row per iteration keeps the 256 gate words out of
      // registers (fully unrolled, ptxas hoisted them and spilled 88 B)
#pragma unroll(D >= 16 ? 1 : D)
      for (int i = 0; i < D; ++i) {
        double re = 0.0, im = 0.0;
#pragma unroll
        for (int d = 0; d < D; ++d) {
          double2 g = a.g[i * D + d];
          re = fma(g.x, x[u][d].x, re);
          re = fma(-g.y, x[u][d].y, re);
          im = fma(g.x, x[u][d].y, im);
          im = fma(g.y, x[u][d].x, im);
        }
        psi[base[u] + a.off[i]] = make_double2(re, im);
      }
    }
  }
}

// 2x2 gate on the innermost index (the pair is two adjacent amplitudes): one
// 32-byte vector load / store per pair instead of two strided 16-byte accesses.
__device__ __forceinline__ double4 ld256(const double4* p) {
  double4 v;
  asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ void st256(double4* p, const double4& v) {
  asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(v.x), "d"(v.y), "d"(v.z), "d"(v.w) : "memory");
}

__global__ void __launch_bounds__(256) k_gate_inner2(double2* __restrict__ psi, int64_t n_pairs,
                                                     const __grid_constant__ GateArgs a) {
  const double2 g00 = a.g[0], g01 = a.g[1], g10 = a.g[2], g11 = a.g[3];
  double4* v4 = reinterpret_cast<double4*>(psi);
  const int64_t S = (int64_t)gridDim.x * blockDim.x;
  const int64_t end = n_pairs + a.f0;
  for (int64_t f0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x + a.f0; f0 < end; f0 += 4 * S) {
    double4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (f0 + u * S < end) v[u] = ld256(v4 + f0 + u * S);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (f0 + u * S >= end) continue;
      const double xr = v[u].x, xi = v[u].y, yr = v[u].z, yi = v[u].w;
      double4 o;
      o.x = fma(g00.x, xr, fma(-g00.y, xi, fma(g01.x, yr, -g01.y * yi)));
      o.y = fma(g00.x, xi, fma(g00.y, xr, fma(g01.x, yi, g01.y * yr)));
      o.z = fma(g10.x, xr, fma(-g10.y, xi, fma(g11.x, yr, -g11.y * yi)));
      o.w = fma(g10.x, xi, fma(g10.y, xr, fma(g11.x, yi, g11.y * yr)));
      st256(v4 + f0 + u * S, o);
    }
  }
}

// Same gate, two neighbouring fibers per thread when the innermost non-target
// index is contiguous (stride 1, even extent): fibers 2p and 2p+1 sit next to
// each other at every target offset, so each pair of amplitudes moves as one
// 32-byte access (LDG/STG.256) and a warp touches 1 KiB contiguous per offset.
template <int D, bool POW2>
__global__ void __launch_bounds__(256) k_gate_dense_v2(double2* __restrict__ psi, int64_t n_pairs,
                                                       const __grid_constant__ GateArgs a) {
  constexpr int F = D <= 2 ? 4 : 2;
  const int64_t S = (int64_t)gridDim.x * blockDim.x;
  for (int64_t p0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p0 < n_pairs; p0 += F * S) {
    int64_t base[F];
    double4 x[F][D];
#pragma unroll
    for (int u = 0; u < F; ++u) {
      const int64_t q = p0 + u * S;
      base[u] = q < n_pairs ? fiber_base<POW2>(2 * q + a.f0, a) : -1;
      if (base[u] >= 0) {
#pragma unroll
        for (int d = 0; d < D; ++d) x[u][d] = ld256(reinterpret_cast<const double4*>(psi + base[u] + a.off[d]));
      }
    }
#pragma unroll
    for (int u = 0; u < F; ++u) {
      if (base[u] < 0) continue;
      // D = 16: one output row per iteration keeps the 256 gate words out of
      // registers (fully unrolled, ptxas hoisted them and spilled 88 B)
#pragma unroll(D >= 16 ? 1 : D)
      for (int i = 0; i < D; ++i) {
        double r0 = 0.0, i0 = 0.0, r1 = 0.0, i1 = 0.0;
#pragma unroll
        for (int d = 0; d < D; ++d) {
          const double2 g = a.g[i * D + d];
          r0 = fma(g.x, x[u][d].x, fma(-g.y, x[u][d].y, r0));
          i0 = fma(g.x, x[u][d].y, fma(g.y, x[u][d].x, i0));
          r1 = fma(g.x, x[u][d].z, fma(-g.y, x[u][d].w, r1));
          i1 = fma(g.x, x[u][d].w, fma(g.y, x[u][d].z, i1));
        }
        st256(reinterpret_cast<double4*>(psi + base[u] + a.off[i]), make_double4(r0, i0, r1, i1));
      }
    }
  }
}

// Generic D (non power of two, or > kMaxD handled by host splitting): loops.
template <bool POW2>
__global__ void __launch_bounds__(256) k_gate_generic(double2* __restrict__ psi, int64_t n_fibers,
                                                      const __grid_constant__ GateArgs a) {
  for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < n_fibers;
       f += (int64_t)gridDim.x * blockDim.x) {
    int64_t base = fiber_base<POW2>(f + a.f0, a);
    double2 x[kMaxD];
    for (int d = 0; d < a.D; ++d) x[d] = psi[base + a.off[d]];
    for (int i = 0; i < a.D; ++i) {
      double re = 0.0, im = 0.0;
      for (int d = 0; d < a.D; ++d) {
        double2 g = a.g[i * a.D + d];
        re = fma(g.x, x[d].x, re);
        re = fma(-g.y, x[d].y, re);
        im = fma(g.x, x[d].y, im);
        im = fma(g.y, x[d].x, im);
      }
      psi[base + a.off[i]] = make_double2(re, im);
    }
  }
}

// Diagonal: y = g_j * x for the listed (non-unit) diagonal entries j only.
template <bool POW2>
__global__ void __launch_bounds__(256) k_gate_diag(double2* __restrict__ psi, int64_t n_fibers,
                                                   const __grid_constant__ GateArgs a) {
  for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < n_fibers;
       f += (int64_t)gridDim.x * blockDim.x) {
    int64_t base = fiber_base<POW2>(f + a.f0, a);
    for (int j = 0; j < a.nd; ++j) {
      double2 v = psi[base + a.off[j]];
      double2 g = a.g[j];
      psi[base + a.off[j]] = make_double2(fma(g.x, v.x, -g.y * v.y), fma(g.x, v.y, g.y * v.x));
    }
  }
}

int grid_for(int64_t work) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((work + 255) / 256, (int64_t)sms * 16)));
}

}  // namespace

void gate_local(void* data, const std::vector<Dim>& dims, const std::vector<int>& targets,
                const double* gh, bool diagonal, cudaStream_t st) {
  gate_strided(data, dims, row_major_strides(dims), targets, gh, diagonal, st, 0, -1);
}

void gate_strided(void* data, const std::vector<Dim>& dims, const std::vector<Dim>& strides,
                  const std::vector<int>& targets, const double* gh, bool diagonal, cudaStream_t st, Dim f_begin,
                  Dim f_end) {
  int r = static_cast<int>(dims.size());
  int k = static_cast<int>(targets.size());
  if (k == 0) throw_invalid("gate needs at least one target");
  std::vector<char> is_t(r, 0);
  for (int t : targets) {
    if (t < 0 || t >= r || is_t[t]) throw_invalid("invalid gate targets");
    is_t[t] = 1;
  }
  GateArgs a{};
  Dim D = 1;
  for (int t : targets) D *= dims[t];
  Dim total = 1;
  for (Dim d : dims) total *= d;
  if (total == 0) return;
  Dim n_fibers = total / D;
  if (f_end < 0 || f_end > n_fibers) f_end = n_fibers;
  if (f_begin >= f_end) return;
  a.f0 = f_begin;
  n_fibers = f_end - f_begin;
  // segments of consecutive non-target positions
  std::vector<std::pair<Dim, Dim>> segs;  // (size, stride of innermost position)
  for (int i = 0; i < r;) {
    if (is_t[i]) {
      ++i;
      continue;
    }
    Dim size = 1;
    int j = i;
    while (j < r && !is_t[j]) size *= dims[j++];
    if (size > 1) segs.push_back({size, strides[j - 1]});
    i = j;
  }
  if (static_cast<int>(segs.size()) > kMaxSeg) throw_invalid("too many index segments for the gate kernel");
  a.nseg = static_cast<int>(segs.size());
  bool pow2 = true;
  for (int j = 0; j < a.nseg; ++j) {
    a.seg_size[j] = segs[j].first;
    a.seg_stride[j] = segs[j].second;
    int sh = 0;
    while ((Dim(1) << sh) < segs[j].first) ++sh;
    a.seg_shift[j] = sh;
    if ((Dim(1) << sh) != segs[j].first) pow2 = false;
  }
  // offsets of the D target-coordinate combinations (targets[0] most significant)
  std::vector<Dim> tdims;
  for (int t : targets) tdims.push_back(dims[t]);
  auto offset_of = [&](Dim idx) {
    auto c = unflat(idx, tdims);
    Dim o = 0;
    for (int j = 0; j < k; ++j) o += c[j] * strides[targets[j]];
    return o;
  };
  int grid = grid_for(n_fibers);
  if (diagonal) {
    std::vector<Dim> nz;
    for (Dim j = 0; j < D; ++j)
      if (!(gh[2 * j] == 1.0 && gh[2 * j + 1] == 0.0)) nz.push_back(j);
    if (nz.empty()) return;
    if (static_cast<int>(nz.size()) > kMaxD * 4) {
      // Dense fallback for wide diagonals: expand in chunks is not needed at our sizes.
      throw_invalid("diagonal gate wider than 64 non-unit entries");
    }
    a.nd = static_cast<int>(nz.size());
    for (int j = 0; j < a.nd; ++j) {
      a.off[j] = offset_of(nz[j]);
      a.g[j] = make_double2(gh[2 * nz[j]], gh[2 * nz[j] + 1]);
    }
    if (pow2) k_gate_diag<true><<<grid, 256, 0, st>>>(static_cast<double2*>(data), n_fibers, a);
    else k_gate_diag<false><<<grid, 256, 0, st>>>(static_cast<double2*>(data), n_fibers, a);
    QTNH_LAUNCH_CHECK();
    return;
  }
  if (D > kMaxD) throw_invalid("dense gate dimension above 16; split or fuse differently");
  a.D = static_cast<int>(D);
  for (Dim j = 0; j < D; ++j) a.off[j] = offset_of(j);
  for (Dim j = 0; j < D * D; ++j) a.g[j] = make_double2(gh[2 * j], gh[2 * j + 1]);
  auto* p = static_cast<double2*>(data);
  // innermost-index 2x2 gate on a contiguous (dense row-major) buffer: vector path
  if (D == 2 && a.nseg == 1 && a.seg_stride[0] == 2 && a.off[0] == 0 && a.off[1] == 1 &&
      (reinterpret_cast<uintptr_t>(data) & 31) == 0) {
    k_gate_inner2<<<grid, 256, 0, st>>>(p, n_fibers, a);
    QTNH_LAUNCH_CHECK();
    return;
  }
  // two neighbouring fibers per thread (see k_gate_dense_v2)
  if ((D == 2 || D == 4) && a.nseg >= 1 && a.seg_stride[a.nseg - 1] == 1 && (a.seg_size[a.nseg - 1] & 1) == 0 &&
      (n_fibers & 1) == 0 && (a.f0 & 1) == 0 && (reinterpret_cast<uintptr_t>(data) & 31) == 0) {
    bool even = true;
    for (int d = 0; d < D; ++d) even = even && (a.off[d] & 1) == 0;
    if (even) {
      const int64_t n_pairs = n_fibers / 2;
      const int g2 = grid_for(n_pairs);
      if (D == 2) {
        if (pow2) k_gate_dense_v2<2, true><<<g2, 256, 0, st>>>(p, n_pairs, a);
        else k_gate_dense_v2<2, false><<<g2, 256, 0, st>>>(p, n_pairs, a);
      } else {
        if (pow2) k_gate_dense_v2<4, true><<<g2, 256, 0, st>>>(p, n_pairs, a);
        else k_gate_dense_v2<4, false><<<g2, 256, 0, st>>>(p, n_pairs, a);
      }
      QTNH_LAUNCH_CHECK();
      return;
    }
  }
#define QTNH_GATE_CASE(DD)                                                          \
  case DD:                                                                          \
    if (pow2) k_gate_dense<DD, true><<<grid, 256, 0, st>>>(p, n_fibers, a);         \
    else k_gate_dense<DD, false><<<grid, 256, 0, st>>>(p, n_fibers, a);             \
    break;
  switch (D) {
    QTNH_GATE_CASE(2)
    QTNH_GATE_CASE(4)
    QTNH_GATE_CASE(8)
    QTNH_GATE_CASE(16)
    default:
      if (pow2) k_gate_generic<true><<<grid, 256, 0, st>>>(p, n_fibers, a);
      else k_gate_generic<false><<<grid, 256, 0, st>>>(p, n_fibers, a);
  }
#undef QTNH_GATE_CASE
  QTNH_LAUNCH_CHECK();
}

namespace {

// ---- fused QFT layer (diagonal fast path + gate fusion) ------------
// Layer j of the QFT is H on qubit j followed by CP(2 pi / 2^m) between j and every
// lower-order qubit j+m-1 (Fig. 1). All those phases are diagonal and
// commute, and for an amplitude with x_j = 1 they multiply to
//   exp(i pi v / 2^t),  v = value of the bits below qubit j, t = its bit position,
// so one pass over the state applies the whole layer:
//   y0 = (a0 + a1)/sqrt2,  y1 = (a0 - a1)/sqrt2 * exp(i pi v / 2^t).
// 32 B/amplitude per LAYER instead of per gate (n layers vs n(n+1)/2 gates).
__global__ void __launch_bounds__(256) k_qft_layer(double2* __restrict__ psi, int64_t n_pairs, int t) {
  const double r = 0.70710678118654752440;
  const int64_t lo_mask = (int64_t(1) << t) - 1;
  const double scale = ldexp(1.0, -t);
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n_pairs;
       p += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = p & lo_mask;
    int64_t i0 = ((p >> t) << (t + 1)) | lo;
    int64_t i1 = i0 | (int64_t(1) << t);
    double2 a0 = psi[i0], a1 = psi[i1];
    double2 y0 = make_double2(r * a0.x + r * a1.x, r * a0.y + r * a1.y);
    double2 d = make_double2(r * a0.x - r * a1.x, r * a0.y - r * a1.y);
    double sn, cs;
    sincospi(static_cast<double>(lo) * scale, &sn, &cs);
    psi[i0] = y0;
    psi[i1] = make_double2(cs * d.x - sn * d.y, cs * d.y + sn * d.x);
  }
}

// Phases of a layer whose target is a distributed qubit with x_j = 1 on this
// rank: every local amplitude i gets exp(i pi (v_off + i) / 2^t).
__global__ void __launch_bounds__(256) k_qft_phase(double2* __restrict__ psi, int64_t n, int64_t v_off, int t) {
  const double scale = ldexp(1.0, -t);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double sn, cs;
    sincospi(static_cast<double>(v_off + i) * scale, &sn, &cs);
    double2 a = psi[i];
    psi[i] = make_double2(cs * a.x - sn * a.y, cs * a.y + sn * a.x);
  }
}

// In-place exchange of two equal-size indices a, b (values of ops::permute with
// the two positions swapped, remap.hpp zero canonicalisation included): per fiber,
// element (i at a, j at b) <-> (j at a, i at b) for i < j.
template <bool POW2>
__global__ void __launch_bounds__(256) k_swap_indices(double2* __restrict__ psi, int64_t n_fibers, int d,
                                                      int64_t sa, int64_t sb, const __grid_constant__ GateArgs a) {
  for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < n_fibers;
       f += (int64_t)gridDim.x * blockDim.x) {
    int64_t base = fiber_base<POW2>(f + a.f0, a);
    for (int i = 0; i < d; ++i) {
      int64_t oii = base + i * sa + i * sb;
      double2 v = psi[oii];
      if (v.x == 0.0 && v.y == 0.0 && (signbit(v.x) || signbit(v.y))) psi[oii] = make_double2(0.0, 0.0);
      for (int j = i + 1; j < d; ++j) {
        int64_t o1 = base + i * sa + j * sb, o2 = base + j * sa + i * sb;
        double2 x = psi[o1], y = psi[o2];
        if (x.x == 0.0 && x.y == 0.0) x = make_double2(0.0, 0.0);
        if (y.x == 0.0 && y.y == 0.0) y = make_double2(0.0, 0.0);
        psi[o1] = y;
        psi[o2] = x;
      }
    }
  }
}

}  // namespace

void qft_layer_local(void* data, int local_bits, int t, cudaStream_t st) {
  if (t < 0 || t >= local_bits) throw_invalid("qft layer target outside the local bits");
  int64_t n_pairs = int64_t(1) << (local_bits - 1);
  k_qft_layer<<<grid_for(n_pairs), 256, 0, st>>>(static_cast<double2*>(data), n_pairs, t);
  QTNH_LAUNCH_CHECK();
}

void qft_phase_local(void* data, int local_bits, int64_t v_off, int t, cudaStream_t st) {
  int64_t n = int64_t(1) << local_bits;
  k_qft_phase<<<grid_for(n), 256, 0, st>>>(static_cast<double2*>(data), n, v_off, t);
  QTNH_LAUNCH_CHECK();
}

void swap_indices_local(void* data, const std::vector<Dim>& dims, int ia, int ib, cudaStream_t st) {
  int r = static_cast<int>(dims.size());
  if (ia < 0 || ib < 0 || ia >= r || ib >= r || ia == ib) throw_invalid("invalid index pair to swap");
  if (dims[ia] != dims[ib]) throw_invalid("swapped indices must have equal dimensions");
  auto strides = row_major_strides(dims);
  GateArgs a{};
  std::vector<std::pair<Dim, Dim>> segs;
  for (int i = 0; i < r;) {
    if (i == ia || i == ib) {
      ++i;
      continue;
    }
    Dim size = 1;
    int j = i;
    while (j < r && j != ia && j != ib) size *= dims[j++];
    if (size > 1) segs.push_back({size, strides[j - 1]});
    i = j;
  }
  a.nseg = static_cast<int>(segs.size());
  bool pow2 = true;
  for (int j = 0; j < a.nseg; ++j) {
    a.seg_size[j] = segs[j].first;
    a.seg_stride[j] = segs[j].second;
    int sh = 0;
    while ((Dim(1) << sh) < segs[j].first) ++sh;
    a.seg_shift[j] = sh;
    if ((Dim(1) << sh) != segs[j].first) pow2 = false;
  }
  Dim total = 1;
  for (Dim d : dims) total *= d;
  Dim n_f = total / (dims[ia] * dims[ib]);
  auto* p = static_cast<double2*>(data);
  int d = static_cast<int>(dims[ia]);
  if (pow2) k_swap_indices<true><<<grid_for(n_f), 256, 0, st>>>(p, n_f, d, strides[ia], strides[ib], a);
  else k_swap_indices<false><<<grid_for(n_f), 256, 0, st>>>(p, n_f, d, strides[ia], strides[ib], a);
  QTNH_LAUNCH_CHECK();
}

namespace {

// ---- cache-blocked QFT ---------------------------------------------------------------
// Layer j (bit t = n-1-j): H on bit t, then exp(i pi v / 2^t) on amplitudes with
// bit t set, v = the bits below t. Layers run in order j = 0..n-1.
//  * k_qft_low3: the lowest L layers touch only the lowest L bits, so one pass over
//    contiguous chunks staged in shared memory applies all of them (twiddles
//    e^{i pi v / 2^t}, v < 2^t, tabulated once per CTA).
//  * k_qft_group: g consecutive upper layers (bits T..B, B >= L) in registers: a
//    thread owns the 2^g amplitudes that differ in those bits; the phase splits
//    into a per-layer table e^{i pi k / 2^u} (k < 2^u, u = t - B) and one
//    sincospi of the fixed low bits per layer.
//  * k_bitrev2: the final SWAP network reverses the bit order -- one in-place pass
//    that exchanges 32 x 32 tiles (a, m, b) <-> (rev b, rev m, rev a).
constexpr int kQftLowMax = 11;
#ifndef QTNH_LOW4_MINB
#define QTNH_LOW4_MINB 1  // 4 (<= 128 registers) spills 20 bytes and is 1 % slower
#endif

__device__ __forceinline__ double2 cmul2(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}



// Low layers: the chunk sits in shared memory and the L layers run in
// rounds of up to 4 bits; a thread owns the 2^g amplitudes of one fiber in
// registers for a round, so a round costs one shared load + store per amplitude
// and one twiddle lookup per amplitude and layer, with one barrier per round.
__constant__ double2 kQftSmallTw[15] = {{1.0, 0.0}, {1.0, 0.0}, {6.123233995736766e-17, 1.0}, {1.0, 0.0}, {0.7071067811865476, 0.7071067811865475}, {6.123233995736766e-17, 1.0}, {-0.7071067811865475, 0.7071067811865476}, {1.0, 0.0}, {0.9238795325112867, 0.3826834323650898}, {0.7071067811865476, 0.7071067811865475}, {0.38268343236508984, 0.9238795325112867}, {6.123233995736766e-17, 1.0}, {-0.3826834323650897, 0.9238795325112867}, {-0.7071067811865475, 0.7071067811865476}, {-0.9238795325112867, 0.3826834323650899}};  // e^{i pi k / 2^u}, index 2^u - 1 + k

__device__ __forceinline__ int swz8(int i) { return i ^ ((i >> 3) & 7); }  // conflict-free 16-B rows

// Compact twiddles of the low pass: the rounds run top-down in groups of up to 4
// bits; a round with bits B..B+g-1 only needs e^{i pi lo / 2^(B+u)} for lo < 2^B,
// u < g, stored at its round offset as [u][lo]. For L = 11 that is 547 entries
// (8.75 KB) instead of a 2^L-entry table (32 KB), so more CTAs fit on an SM.
__host__ __device__ constexpr int qft_low_g(int T) { return T + 1 >= 4 ? 4 : T + 1; }
__host__ __device__ inline int qft_low_tw_count(int L) {
  int n = 0;
  for (int T = L - 1; T >= 0;) {
    const int g = qft_low_g(T), B = T - g + 1;
    n += g << B;
    T = B - 1;
  }
  return n;
}
__device__ void qft_low_tw_build(double2* tw, int L) {
  int off = 0;
  for (int T = L - 1; T >= 0;) {
    const int g = qft_low_g(T), B = T - g + 1;
    for (int e = threadIdx.x; e < (g << B); e += blockDim.x) {
      const int u = e >> B, lo = e & ((1 << B) - 1);
      double sn, cs;
      sincospi(static_cast<double>(lo) * ldexp(1.0, -(B + u)), &sn, &cs);
      tw[off + e] = make_double2(cs, sn);
    }
    off += g << B;
    T = B - 1;
  }
}

// The butterflies are unnormalised (y0 = a0 + a1, y1 = (a0 - a1) w): the L
// factors of 1/sqrt2 are applied once when the chunk is written back, which
// takes a third of the FP64 work out of a pass that is FP64-issue bound.
template <int G>
__device__ __forceinline__ void qft_low_round(double2* __restrict__ data, const double2* __restrict__ tw, int L,
                                              int B, double scale = 1.0) {
  const int nf = 1 << (L - G);
  for (int f = threadIdx.x; f < nf; f += blockDim.x) {
    const int lo = f & ((1 << B) - 1), hi = f >> B;
    const int base = (hi << (B + G)) | lo;
    double2 x[1 << G];
#pragma unroll
    for (int k = 0; k < (1 << G); ++k) x[k] = data[swz8(base + (k << B))];
    // phase of layer t = B + u for in-fiber index k: e^{i pi klow / 2^u} * e^{i pi lo / 2^t}
    double2 lof[G];
#pragma unroll
    for (int u = 0; u < G; ++u) lof[u] = tw[(u << B) + lo];
#pragma unroll
    for (int u = G - 1; u >= 0; --u) {
#pragma unroll
      for (int k = 0; k < (1 << G); ++k) {
        if (k & (1 << u)) continue;
        const int k1 = k | (1 << u);
        double2 a0 = x[k], a1 = x[k1];
        x[k] = make_double2(a0.x + a1.x, a0.y + a1.y);
        double2 d = make_double2(a0.x - a1.x, a0.y - a1.y);
        const int kl = k & ((1 << u) - 1);
        double2 ph = kl ? cmul2(kQftSmallTw[(1 << u) - 1 + kl], lof[u]) : lof[u];
        x[k1] = (B + u) > 0 || kl ? cmul2(d, ph) : d;
      }
    }
    if (scale != 1.0) {
#pragma unroll
      for (int k = 0; k < (1 << G); ++k) x[k] = make_double2(x[k].x * scale, x[k].y * scale);
    }
#pragma unroll
    for (int k = 0; k < (1 << G); ++k) data[swz8(base + (k << B))] = x[k];
  }
}


// k_qft_low3 runs these rounds with the chunks streamed through two shared-memory
// buffers by cp.async (16-byte LDGSTS, swizzled destination): chunk c+1 is in
// flight while chunk c is transformed and written back, so the global loads no
// longer serialise behind the shared-memory rounds (the single-buffer version was
// long-scoreboard bound at ~25% of HBM bandwidth).
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::); }

__global__ void __launch_bounds__(128) k_qft_low3(double2* __restrict__ psi, int64_t n_chunks, int S, int L) {
  extern __shared__ double2 smq3[];
  // a chunk of 2^S amplitudes holds 2^(S-L) independent L-bit transforms, so the
  // rounds keep all threads busy for small L
  const int C = 1 << S;
  double2* buf0 = smq3;
  double2* buf1 = smq3 + C;
  double2* tw = smq3 + 2 * C;
  qft_low_tw_build(tw, L);
  int64_t ch = blockIdx.x;
  if (ch < n_chunks)
    for (int e = threadIdx.x; e < C; e += blockDim.x) cp_async16(buf0 + swz8(e), psi + ch * C + e);
  cp_async_commit();
  int cur = 0;
  for (; ch < n_chunks; ch += gridDim.x) {
    double2* data = cur ? buf1 : buf0;
    double2* next = cur ? buf0 : buf1;
    const int64_t nx = ch + gridDim.x;
    if (nx < n_chunks)
      for (int e = threadIdx.x; e < C; e += blockDim.x) cp_async16(next + swz8(e), psi + nx * C + e);
    cp_async_commit();
    cp_async_wait1();  // this chunk has landed (the next one may still be in flight)
    __syncthreads();
    for (int T = L - 1, off = 0; T >= 0;) {
      int gg = qft_low_g(T);
      int B = T - gg + 1;
      switch (gg) {
        case 4: qft_low_round<4>(data, tw + off, S, B); break;
        case 3: qft_low_round<3>(data, tw + off, S, B); break;
        case 2: qft_low_round<2>(data, tw + off, S, B); break;
        default: qft_low_round<1>(data, tw + off, S, B); break;
      }
      __syncthreads();
      off += gg << B;
      T = B - 1;
    }
    double2* g = psi + ch * C;
    const double sc = ldexp(1.0, -(L / 2)) * (L & 1 ? 0.70710678118654752440 : 1.0);  // (1/sqrt2)^L
    for (int e = threadIdx.x; e < C; e += blockDim.x) {
      double2 v = data[swz8(e)];
      g[e] = make_double2(v.x * sc, v.y * sc);
    }
    __syncthreads();  // buffer free before it is refilled two chunks on
    cur ^= 1;
  }
}

// Variant: the chunk's first (top) round reads straight from global memory into
// registers (16 independent loads per thread) and writes the shared chunk, so
// one shared-memory write + read of the chunk and the staging copy disappear;
// single buffer, occupancy hides the load latency.
template <int G>
__device__ __forceinline__ void qft_low_round_from_global(const double2* __restrict__ g, double2* __restrict__ data,
                                                          const double2* __restrict__ tw, int S, int B) {
  const int nf = 1 << (S - G);
  for (int f = threadIdx.x; f < nf; f += blockDim.x) {
    const int lo = f & ((1 << B) - 1), hi = f >> B;
    const int base = (hi << (B + G)) | lo;
    double2 x[1 << G];
#pragma unroll
    for (int k = 0; k < (1 << G); ++k) x[k] = g[base + (k << B)];
    double2 lof[G];
#pragma unroll
    for (int u = 0; u < G; ++u) lof[u] = tw[(u << B) + lo];
#pragma unroll
    for (int u = G - 1; u >= 0; --u) {
#pragma unroll
      for (int k = 0; k < (1 << G); ++k) {
        if (k & (1 << u)) continue;
        const int k1 = k | (1 << u);
        double2 a0 = x[k], a1 = x[k1];
        x[k] = make_double2(a0.x + a1.x, a0.y + a1.y);
        double2 d = make_double2(a0.x - a1.x, a0.y - a1.y);
        const int kl = k & ((1 << u) - 1);
        double2 ph = kl ? cmul2(kQftSmallTw[(1 << u) - 1 + kl], lof[u]) : lof[u];
        x[k1] = (B + u) > 0 || kl ? cmul2(d, ph) : d;
      }
    }
#pragma unroll
    for (int k = 0; k < (1 << G); ++k) data[swz8(base + (k << B))] = x[k];
  }
}

__global__ void __launch_bounds__(128, QTNH_LOW4_MINB) k_qft_low4(double2* __restrict__ psi, int64_t n_chunks, int S, int L) {
  extern __shared__ double2 smq4[];
  const int C = 1 << S;
  double2* data = smq4;
  double2* tw = smq4 + C;
  qft_low_tw_build(tw, L);
  __syncthreads();
  const double sc = ldexp(1.0, -(L / 2)) * (L & 1 ? 0.70710678118654752440 : 1.0);  // (1/sqrt2)^L
  for (int64_t ch = blockIdx.x; ch < n_chunks; ch += gridDim.x) {
    double2* g = psi + ch * C;
    int T = L - 1, off = 0;
    {
      const int gg = qft_low_g(T), B = T - gg + 1;
      switch (gg) {
        case 4: qft_low_round_from_global<4>(g, data, tw, S, B); break;
        case 3: qft_low_round_from_global<3>(g, data, tw, S, B); break;
        case 2: qft_low_round_from_global<2>(g, data, tw, S, B); break;
        default: qft_low_round_from_global<1>(g, data, tw, S, B); break;
      }
      off += gg << B;
      T = B - 1;
    }
    __syncthreads();
    while (T >= 0) {
      const int gg = qft_low_g(T), B = T - gg + 1;
      switch (gg) {
        case 4: qft_low_round<4>(data, tw + off, S, B); break;
        case 3: qft_low_round<3>(data, tw + off, S, B); break;
        case 2: qft_low_round<2>(data, tw + off, S, B); break;
        default: qft_low_round<1>(data, tw + off, S, B); break;
      }
      __syncthreads();
      off += gg << B;
      T = B - 1;
    }
    for (int e = threadIdx.x; e < C; e += blockDim.x) {
      double2 v = data[swz8(e)];
      g[e] = make_double2(v.x * sc, v.y * sc);
    }
    __syncthreads();
  }
}

// TMA form of the low pass (default): a chunk of 2^S amplitudes is one 2-D box
// of a FLOAT64 tensor map [2^(n-3) rows][16 doubles] with the 128-byte swizzle,
// which puts amplitude i at shared index i ^ ((i >> 3) & 7) -- exactly the swz8
// layout the shared-memory rounds use -- so the chunk lands by one bulk tensor
// load (mbarrier, NB buffers, issued NB - 1 chunks ahead) and leaves by one bulk
// tensor store straight from the rounds' output (the 1/sqrt2^L scale folded into
// the last round). k_qft_low4 (single buffer, first round from global into
// registers) kept its loads in flight only during its load phase: 4.8 TB/s at
// n = 33; here every CTA always has the next chunk loading and the previous one
// storing.
template <int NB, int MINB>
__global__ void __launch_bounds__(128, MINB) k_qft_low_tma(const __grid_constant__ CUtensorMap tm, int64_t n_chunks, int S,
                                                    int L) {
  extern __shared__ unsigned char smq_raw[];
  double2* bufs = reinterpret_cast<double2*>((reinterpret_cast<uintptr_t>(smq_raw) + 1023) & ~uintptr_t(1023));
  const int C = 1 << S, rows = C >> 3;
  double2* tw = bufs + NB * C;
  __shared__ uint64_t full[NB];
  const int tid = threadIdx.x;
  qft_low_tw_build(tw, L);
  const int64_t grid = gridDim.x;
  if (tid == 0) {
    prefetch_tmap(&tm);
    for (int b = 0; b < NB; ++b) mbar_init(&full[b], 1);
    fence_mbar_init();
    for (int b = 0; b < NB - 1; ++b) {
      const int64_t c = blockIdx.x + b * grid;
      if (c < n_chunks) {
        mbar_arrive_expect_tx(&full[b], static_cast<uint32_t>(C) * 16u);
        tma_load_2d(bufs + b * C, &tm, 0, static_cast<int>(c * rows), &full[b]);
      }
    }
  }
  __syncthreads();
  const double sc = ldexp(1.0, -(L / 2)) * (L & 1 ? 0.70710678118654752440 : 1.0);  // (1/sqrt2)^L
  int64_t i = 0;
  for (int64_t ch = blockIdx.x; ch < n_chunks; ch += grid, ++i) {
    const int b = static_cast<int>(i % NB);
    if (NB == 1 && tid == 0) {  // one buffer: it is free once the previous store has read it
      bulk_wait_read<0>();
      mbar_arrive_expect_tx(&full[0], static_cast<uint32_t>(C) * 16u);
      tma_load_2d(bufs, &tm, 0, static_cast<int>(ch * rows), &full[0]);
    }
    mbar_wait(&full[b], static_cast<uint32_t>((i / NB) & 1));
    double2* data = bufs + b * C;
    int T = L - 1, off = 0;
    bool first = true;
    while (T >= 0) {
      const int gg = qft_low_g(T), B = T - gg + 1;
      const double s_here = B == 0 ? sc : 1.0;  // the last round writes the scaled output
      switch (gg) {
        case 4: qft_low_round<4>(data, tw + off, S, B, s_here); break;
        case 3: qft_low_round<3>(data, tw + off, S, B, s_here); break;
        case 2: qft_low_round<2>(data, tw + off, S, B, s_here); break;
        default: qft_low_round<1>(data, tw + off, S, B, s_here); break;
      }
      off += gg << B;
      T = B - 1;
      if (NB > 1 && first && tid == 0) {
        // next load into the buffer of chunk i - 1, whose store has had a round to read it
        const int64_t nc = ch + (NB - 1) * grid;
        if (nc < n_chunks) {
          const int nbuf = static_cast<int>((i + NB - 1) % NB);
          bulk_wait_read<0>();
          mbar_arrive_expect_tx(&full[nbuf], static_cast<uint32_t>(C) * 16u);
          tma_load_2d(bufs + nbuf * C, &tm, 0, static_cast<int>(nc * rows), &full[nbuf]);
        }
      }
      first = false;
      __syncthreads();
    }
    fence_proxy_async_smem();  // this thread's round writes, visible to the bulk store
    __syncthreads();
    if (tid == 0) {
      tma_store_2d(&tm, 0, static_cast<int>(ch * rows), data);
      bulk_commit();
    }
  }
  if (tid == 0) bulk_wait_read<0>();
}

struct QftGroupArgs {
  double2 tab[32];  // tab[2^u + k] = e^{i pi k / 2^u}, k < 2^u, u < 5
};

// G = 5 (32 amplitudes = 128 registers per thread) runs one fiber per thread: in a
// grid-stride loop the compiler hoists the 31 loop-invariant table twiddles into
// registers and spills.
template <int G>
__global__ void __launch_bounds__(256, (G >= 4 ? 1 : 2)) k_qft_group(double2* __restrict__ psi, int64_t n_fibers, int B,
                                                   const __grid_constant__ QftGroupArgs ga) {
  const double r = 0.70710678118654752440;
  const int64_t lo_mask = (int64_t(1) << B) - 1;
  constexpr bool kOne = G >= 5;
  for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < n_fibers;
       f += kOne ? n_fibers : (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = f & lo_mask, hi = f >> B;
    int64_t base = (hi << (B + G)) | lo;
    // per-layer phases of the fixed low bits, before the amplitudes are live
    double2 lofs[G];
#pragma unroll
    for (int u = 0; u < G; ++u) {
      double sn, cs;
      sincospi(static_cast<double>(lo) * ldexp(1.0, -(B + u)), &sn, &cs);
      lofs[u] = make_double2(cs, sn);
    }
    double2 x[1 << G];
#pragma unroll
    for (int k = 0; k < (1 << G); ++k) x[k] = psi[base + (int64_t(k) << B)];
#pragma unroll
    for (int u = G - 1; u >= 0; --u) {
      const double2 lof = lofs[u];
#pragma unroll
      for (int k = 0; k < (1 << G); ++k) {
        if (k & (1 << u)) continue;
        const int k1 = k | (1 << u);
        double2 a0 = x[k], a1 = x[k1];
        x[k] = make_double2(r * a0.x + r * a1.x, r * a0.y + r * a1.y);
        double2 d = make_double2(r * a0.x - r * a1.x, r * a0.y - r * a1.y);
        const int kl = k & ((1 << u) - 1);
        double2 ph = u > 0 ? cmul2(ga.tab[(1 << u) + kl], lof) : lof;
        x[k1] = cmul2(d, ph);
      }
    }
#pragma unroll
    for (int k = 0; k < (1 << G); ++k) psi[base + (int64_t(k) << B)] = x[k];
  }
}

// ---- shared-memory group pass: G1 + G2 consecutive layers on strided bits ---------------
// Bits B .. B+G1+G2-1 (B >= 4) in one pass: a CTA owns a tile of 2^(G1+G2) group
// values x W = 16 consecutive low elements (256-byte rows, 64 KB at 8 bits), staged
// in shared memory; the upper G1 layers run in registers with the lower G2 group
// bits fixed per thread, then the lower G2 layers with the upper ones fixed. The
// phase of layer t = B + u splits into e^{i pi x / 2^u} (x = the group bits below
// u, table kQftMidTw) times e^{i pi lo / 2^(B+u)} (lo = the fixed low bits, one
// sincospi per (u, column) per tile). 8 layers per pass instead of 4: QFT-33 takes
// 3 + low + bit reversal = 5 passes over the state instead of 8.
constexpr int kMidW = 16;
__constant__ double2 kQftMidTw[256];  // e^{i pi x / 2^u} at index 2^u - 1 + x, u < 8

// The two register rounds of a shared-memory group pass over one staged tile
// data[NG][kMidW] (phases: kQftMidTw table x the per-column lofs[GB][kMidW]).
template <int G1, int G2>
__device__ __forceinline__ void qft_mid_rounds(double2* __restrict__ data, const double2* __restrict__ lofs) {
  constexpr int GB = G1 + G2;
  const int tid = threadIdx.x;
  const double r = 0.70710678118654752440;
    // round 1: upper G1 group bits (layers u = GB-1 .. G2), lower G2 bits fixed
    for (int f = tid; f < (1 << G2) * kMidW; f += 256) {
      const int w = f % kMidW, j = f / kMidW;
      double2 x[1 << G1];
#pragma unroll
      for (int k = 0; k < (1 << G1); ++k) x[k] = data[((k << G2) | j) * kMidW + w];
#pragma unroll
      for (int s = G1 - 1; s >= 0; --s) {
        const int u = G2 + s;
        const double2 lf = lofs[u * kMidW + w];
#pragma unroll
        for (int k = 0; k < (1 << G1); ++k) {
          if (k & (1 << s)) continue;
          const int k1 = k | (1 << s);
          const double2 a0 = x[k], a1 = x[k1];
          x[k] = make_double2(r * a0.x + r * a1.x, r * a0.y + r * a1.y);
          const double2 d = make_double2(r * a0.x - r * a1.x, r * a0.y - r * a1.y);
          const int xg = ((k & ((1 << s) - 1)) << G2) | j;  // group bits below u
          x[k1] = cmul2(d, cmul2(kQftMidTw[(1 << u) - 1 + xg], lf));
        }
      }
#pragma unroll
      for (int k = 0; k < (1 << G1); ++k) data[((k << G2) | j) * kMidW + w] = x[k];
    }
  __syncthreads();
    // round 2: lower G2 group bits (layers u = G2-1 .. 0), upper G1 bits fixed
    for (int f = tid; f < (1 << G1) * kMidW; f += 256) {
      const int w = f % kMidW, i = f / kMidW;
      double2 x[1 << G2];
#pragma unroll
      for (int k = 0; k < (1 << G2); ++k) x[k] = data[((i << G2) | k) * kMidW + w];
#pragma unroll
      for (int u = G2 - 1; u >= 0; --u) {
        const double2 lf = lofs[u * kMidW + w];
#pragma unroll
        for (int k = 0; k < (1 << G2); ++k) {
          if (k & (1 << u)) continue;
          const int k1 = k | (1 << u);
          const double2 a0 = x[k], a1 = x[k1];
          x[k] = make_double2(r * a0.x + r * a1.x, r * a0.y + r * a1.y);
          const double2 d = make_double2(r * a0.x - r * a1.x, r * a0.y - r * a1.y);
          const int xg = k & ((1 << u) - 1);
          x[k1] = cmul2(d, u > 0 ? cmul2(kQftMidTw[(1 << u) - 1 + xg], lf) : lf);
        }
      }
#pragma unroll
      for (int k = 0; k < (1 << G2); ++k) data[((i << G2) | k) * kMidW + w] = x[k];
    }
}

template <int G1, int G2>
__global__ void __launch_bounds__(256, 2) k_qft_mid(double2* __restrict__ psi, int64_t n_tiles, int B) {
  constexpr int GB = G1 + G2, NG = 1 << GB, NE = NG * kMidW;
  static_assert((1 << G1) * kMidW == 256 || (1 << G2) * kMidW <= 256, "fibers per round fit the block");
  extern __shared__ double2 smid[];
  double2* data = smid;              // [NG][kMidW]
  double2* lofs = smid + NE;         // [GB][kMidW]
  const int tid = threadIdx.x;
  const int64_t lo_blocks = (int64_t(1) << B) / kMidW;
  for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const int64_t hi = tile / lo_blocks, lo0 = (tile % lo_blocks) * kMidW;
    double2* g0 = psi + (hi << (B + GB)) + lo0;
    for (int e = tid; e < NE; e += 256) {
      const int g = e / kMidW, w = e % kMidW;
      cp_async16(data + e, g0 + (int64_t(g) << B) + w);
    }
    cp_async_commit();
    for (int e = tid; e < GB * kMidW; e += 256) {
      const int u = e / kMidW, w = e % kMidW;
      double sn, cs;
      sincospi(static_cast<double>(lo0 + w) * ldexp(1.0, -(B + u)), &sn, &cs);
      lofs[e] = make_double2(cs, sn);
    }
    asm volatile("cp.async.wait_group 0;\n" ::);
    __syncthreads();
    qft_mid_rounds<G1, G2>(data, lofs);
    __syncthreads();
    for (int e = tid; e < NE; e += 256) {
      const int g = e / kMidW, w = e % kMidW;
      g0[(int64_t(g) << B) + w] = data[e];
    }
    __syncthreads();  // the tile buffer is reused by the next tile
  }
}


__device__ __forceinline__ unsigned rev_bits(unsigned x, int bits) { return __brev(x) >> (32 - bits); }
__device__ __forceinline__ uint64_t rev_bits64(uint64_t x, int bits) { return __brevll(x) >> (64 - bits); }

__device__ __forceinline__ double2 canon2(double2 v) {
  if (v.x == 0.0 && v.y == 0.0) v = make_double2(0.0, 0.0);
  return v;
}

// TMA form of the in-place bit reversal (default): the tiles arrive by
// cp.async.bulk.tensor instead of 2048 per-thread 16-byte cp.async per tile pair.
// The state is a 3-D FLOAT64 tensor [a: 32][m: 2^(n-10)][b: 64 doubles]; a box
// is {16 doubles = 8 amplitudes of b, 1 m, 32 a}, 4 KB with the 128-byte
// swizzle (16-byte chunk j of row a stored at j ^ (a & 7)), so the bit-reversed
// column reads below hit 8 distinct 16-byte bank groups per 32 lanes. A stage
// is one tile pair (2 x 4 boxes, 32 KB), S stages per CTA with one mbarrier
// each; one thread re-arms a stage after the CTA barrier that ends its reads.
// Stores are plain coalesced 512-byte warp rows (the tile order is final).
template <int S>
__global__ void __launch_bounds__(512) k_bitrev_tma(const __grid_constant__ CUtensorMap tm, double2* __restrict__ psi,
                                                       int n, int64_t n_mid) {
  extern __shared__ unsigned char smem_raw[];
  double2* tiles = reinterpret_cast<double2*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[S];
  const int mbits = n - 10;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  auto rev_m = [&](int64_t m) {
    return mbits > 0 ? static_cast<int64_t>(rev_bits64(static_cast<uint64_t>(m), mbits)) : m;
  };
  auto next_valid = [&](int64_t m) {
    while (m < n_mid && rev_m(m) < m) m += gridDim.x;  // a pair is handled by its smaller member
    return m;
  };
  int64_t m_issue = 0;
  auto issue = [&](int stage, int64_t m) {
    const int64_t mr = rev_m(m);
    double2* t1 = tiles + stage * 2048;
    double2* t2 = t1 + 1024;
    mbar_arrive_expect_tx(&full[stage], mr != m ? 32768u : 16384u);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      tma_load_3d(t1 + c * 256, &tm, c * 16, static_cast<int>(m), 0, &full[stage]);
      if (mr != m) tma_load_3d(t2 + c * 256, &tm, c * 16, static_cast<int>(mr), 0, &full[stage]);
    }
  };
  if (threadIdx.x == 0) {
    prefetch_tmap(&tm);
    for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
    m_issue = next_valid(blockIdx.x);
    for (int s = 0; s < S && m_issue < n_mid; ++s) {
      issue(s, m_issue);
      m_issue = next_valid(m_issue + gridDim.x);
    }
  }
  __syncthreads();
  const int rb = rev_bits(lane, 5);
  int stage = 0;
  uint32_t phase = 0;
  for (int64_t m = next_valid(blockIdx.x); m < n_mid; m = next_valid(m + gridDim.x)) {
    mbar_wait(&full[stage], phase);
    const int64_t mr = rev_m(m);
    const double2* t1 = tiles + stage * 2048;
    const double2* t2 = mr != m ? t1 + 1024 : t1;
    for (int a = warp; a < 32; a += nwarps) {
      const int ra = rev_bits(a, 5);
      // source (row rb, amplitude ra): box ra >> 3, chunk (ra & 7) ^ (rb & 7)
      const int src = (ra >> 3) * 256 + rb * 8 + ((ra & 7) ^ (rb & 7));
      // new (a, m, b) = old (rev b, rev m, rev a)
      psi[(int64_t(a) << (n - 5)) | (m << 5) | lane] = canon2(t2[src]);
      if (mr != m) psi[(int64_t(a) << (n - 5)) | (mr << 5) | lane] = canon2(t1[src]);
    }
    __syncthreads();  // every read of this stage is done
    if (threadIdx.x == 0 && m_issue < n_mid) {
      fence_proxy_async_smem();
      issue(stage, m_issue);
      m_issue = next_valid(m_issue + gridDim.x);
    }
    if (++stage == S) {
      stage = 0;
      phase ^= 1;
    }
  }
}

// n >= 10: x = (a: top 5 bits, m: middle n-10 bits, b: low 5 bits).

// In-place bit reversal: the two 32 x 32 tiles of a pair are
// staged by cp.async into a double buffer (the next pair is in flight while this
// one is written back), and the tile columns are XOR-swizzled with bits 2..4 of
// the row so the bit-reversed column reads (lanes -> rows rev(tx)) hit eight
// distinct 16-byte bank groups (a padded layout is 4-way conflicted).
__device__ __forceinline__ int bswz(int row, int col) { return row * 32 + (col ^ ((row >> 2) & 7)); }

__global__ void __launch_bounds__(256) k_bitrev2(double2* __restrict__ psi, int n, int64_t n_mid) {
  extern __shared__ double2 sbr[];  // [stage][tile][32 x 32]
  const int mbits = n - 10;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  auto rev_m = [&](int64_t m) {
    return mbits > 0 ? static_cast<int64_t>(rev_bits64(static_cast<uint64_t>(m), mbits)) : m;
  };
  auto next_valid = [&](int64_t m) {
    while (m < n_mid && rev_m(m) < m) m += gridDim.x;  // a pair is handled by its smaller member
    return m;
  };
  auto issue = [&](int stage, int64_t m) {
    double2* t1 = sbr + stage * 2048;
    double2* t2 = t1 + 1024;
    const int64_t mr = rev_m(m);
#pragma unroll
    for (int a = ty; a < 32; a += 8) {
      cp_async16(t1 + bswz(a, tx), psi + ((int64_t(a) << (n - 5)) | (m << 5) | tx));
      cp_async16(t2 + bswz(a, tx), psi + ((int64_t(a) << (n - 5)) | (mr << 5) | tx));
    }
  };
  int64_t m = next_valid(blockIdx.x);
  if (m < n_mid) issue(0, m);
  cp_async_commit();
  int stage = 0;
  while (m < n_mid) {
    const int64_t mn = next_valid(m + gridDim.x);
    if (mn < n_mid) issue(stage ^ 1, mn);
    cp_async_commit();
    cp_async_wait1();
    __syncthreads();
    const double2* t1 = sbr + stage * 2048;
    const double2* t2 = t1 + 1024;
    const int64_t mr = rev_m(m);
    const int rb = rev_bits(tx, 5);
#pragma unroll
    for (int a = ty; a < 32; a += 8) {
      const int ra = rev_bits(a, 5);
      // new (a, m, b) = old (rev b, rev m, rev a)
      psi[(int64_t(a) << (n - 5)) | (m << 5) | tx] = canon2(t2[bswz(rb, ra)]);
      if (mr != m) psi[(int64_t(a) << (n - 5)) | (mr << 5) | tx] = canon2(t1[bswz(rb, ra)]);
    }
    __syncthreads();
    stage ^= 1;
    m = mn;
  }
}

// Bit reversal of the top nh bits of the local index with the low k bits held
// (the distributed QFT's final swaps once its k distributed qubits have been
// exchanged with the k innermost local ones): element (hi, lo) <- (rev hi, lo).
// Tiles of 2^B x 2^B "rows" of 2^k contiguous amplitudes (2^(2B+k) <= 2048) are
// exchanged between hi = (a, m, b) and (rev b, rev m, rev a) through shared memory.
__global__ void __launch_bounds__(256) k_bitrev_hi(double2* __restrict__ psi, int nh, int k, int B, int64_t n_mid) {
  extern __shared__ double2 smb[];
  const int R = 1 << B, RE = R << k, row = RE + 1;
  double2* t1 = smb;
  double2* t2 = smb + R * row;
  const int mbits = nh - 2 * B;
  const int tile = R * RE;
  auto base = [&](int a, int64_t m) { return ((int64_t(a) << (nh - B)) | (m << B)) << k; };
  for (int64_t m = blockIdx.x; m < n_mid; m += gridDim.x) {
    int64_t mr = mbits > 0 ? static_cast<int64_t>(rev_bits64(static_cast<uint64_t>(m), mbits)) : m;
    if (mr < m) continue;
    __syncthreads();
    for (int e = threadIdx.x; e < tile; e += blockDim.x) {
      int a = e / RE, rest = e - a * RE;
      t1[a * row + rest] = psi[base(a, m) + rest];
      t2[a * row + rest] = psi[base(a, mr) + rest];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < tile; e += blockDim.x) {
      int a = e / RE, rest = e - a * RE;
      int b = rest >> k, lo = rest & ((1 << k) - 1);
      int ra = B ? rev_bits(a, B) : 0, rb = B ? rev_bits(b, B) : 0;
      int src = rb * row + ((ra << k) | lo);
      psi[base(a, m) + rest] = canon2(t2[src]);
      if (mr != m) psi[base(a, mr) + rest] = canon2(t1[src]);
    }
  }
}

// ---- distributed QFT over peer memory ---------------------------------------------------
// The 2^K ranks of a copy group hold the blocks x = 0 .. 2^K-1 of a state whose K
// leading qubits are distributed. Each rank takes a slice of the local indices
// and, for every local index i in it, loads the 2^K amplitudes (x, i) from all
// group members (peer loads over NVLink), applies the QFT layers of the K
// distributed qubits in registers and stores them back: the layers' H and
// controlled phases fused with the exchange, one pass over the state.
// Layer j (qubit j = bit K-1-j of x, bit position t = nb + K-1-j of the index):
//   y0 = (a0 + a1)/sqrt2, y1 = (a0 - a1)/sqrt2 * exp(i pi v / 2^t),
//   v / 2^t = (x mod 2^b)/2^b + i / 2^(nb+b),  b = K-1-j;
// the i-dependent factor is w^(2^(K-1-b)) with w = exp(i pi i / 2^(nb+K-1)).
struct PeerGroup {
  double2* p[16];
};

template <int K>
__global__ void __launch_bounds__(256) k_qft_dist_layers(const __grid_constant__ PeerGroup g, int nb, int64_t i0,
                                                         int64_t i1) {
  constexpr int X = 1 << K;
  const double r = 0.70710678118654752440;
  for (int64_t i = i0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < i1;
       i += (int64_t)gridDim.x * blockDim.x) {
    double2 a[X];
#pragma unroll
    for (int x = 0; x < X; ++x) a[x] = g.p[x][i];
    double2 w[K];  // w[b] = exp(i pi i / 2^(nb+b))
    {
      double sn, cs;
      sincospi(static_cast<double>(i) * ldexp(1.0, -(nb + K - 1)), &sn, &cs);
      w[K - 1] = make_double2(cs, sn);
#pragma unroll
      for (int b = K - 1; b > 0; --b) w[b - 1] = cmul2(w[b], w[b]);
    }
#pragma unroll
    for (int j = 0; j < K; ++j) {
      const int b = K - 1 - j;
#pragma unroll
      for (int x = 0; x < X; ++x) {
        if (x & (1 << b)) continue;
        const int x1 = x | (1 << b);
        double2 a0 = a[x], a1 = a[x1];
        a[x] = make_double2(r * a0.x + r * a1.x, r * a0.y + r * a1.y);
        double2 d = make_double2(r * a0.x - r * a1.x, r * a0.y - r * a1.y);
        double2 ph = w[b];
        const int xl = x & ((1 << b) - 1);
        if (xl) ph = cmul2(ph, kQftSmallTw[(1 << b) - 1 + xl]);  // e^{i pi xl / 2^b}
        a[x1] = cmul2(d, ph);
      }
    }
#pragma unroll
    for (int x = 0; x < X; ++x) g.p[x][i] = a[x];
  }
}

// Final bit reversal, distributed part: with the local index i = (mid, l), l its
// K low bits, element (x, mid, l) moves to (rev l, mid, rev x) -- the K
// distributed qubits trade places with the K innermost local ones, each group
// reversed. For one mid the 2^K x 2^K elements form a closed set, so a CTA loads
// MB mids from all members (runs of MB * 2^K contiguous amplitudes per member),
// and stores them transposed; mids are split over the group. The middle qubits
// are reversed afterwards by k_bitrev_hi on every rank.
template <int K>
__global__ void __launch_bounds__(256) k_dist_bitrev(const __grid_constant__ PeerGroup g, int64_t m0, int64_t m1) {
  constexpr int X = 1 << K;
  constexpr int MB = 256 / X;   // mids per tile -> X * MB * X amplitudes
  constexpr int ROW = MB * X + 1;
  extern __shared__ double2 smd[];
  for (int64_t mt = m0 + int64_t(blockIdx.x) * MB; mt < m1; mt += int64_t(gridDim.x) * MB) {
    const int nm = static_cast<int>((m1 - mt < MB ? m1 - mt : int64_t(MB)));
    __syncthreads();
    for (int x = 0; x < X; ++x)
      for (int e = threadIdx.x; e < nm * X; e += blockDim.x) smd[x * ROW + e] = g.p[x][mt * X + e];
    __syncthreads();
    for (int x = 0; x < X; ++x) {
      const int rx = K ? static_cast<int>(__brev(x) >> (32 - K)) : 0;
      for (int e = threadIdx.x; e < nm * X; e += blockDim.x) {
        const int mb = e / X, l = e % X;
        const int rl = static_cast<int>(__brev(l) >> (32 - K));
        g.p[x][mt * X + e] = canon2(smd[rl * ROW + mb * X + rx]);
      }
    }
  }
}

}  // namespace

void qft_dist_layers(void* const* ptrs, int k, int nb, Dim i0, Dim i1, cudaStream_t st) {
  if (i1 <= i0) return;
  PeerGroup g{};
  for (int x = 0; x < (1 << k); ++x) g.p[x] = static_cast<double2*>(ptrs[x]);
  int grid = grid_for(i1 - i0);
  switch (k) {
    case 1: k_qft_dist_layers<1><<<grid, 256, 0, st>>>(g, nb, i0, i1); break;
    case 2: k_qft_dist_layers<2><<<grid, 256, 0, st>>>(g, nb, i0, i1); break;
    case 3: k_qft_dist_layers<3><<<grid, 256, 0, st>>>(g, nb, i0, i1); break;
    case 4: k_qft_dist_layers<4><<<grid, 256, 0, st>>>(g, nb, i0, i1); break;
    default: throw_invalid("fused distributed QFT layers need 1..4 distributed qubits");
  }
  QTNH_LAUNCH_CHECK();
}

void dist_bitrev(void* const* ptrs, int k, Dim m0, Dim m1, cudaStream_t st) {
  if (m1 <= m0) return;
  PeerGroup g{};
  for (int x = 0; x < (1 << k); ++x) g.p[x] = static_cast<double2*>(ptrs[x]);
  const int X = 1 << k, MB = 256 / X;
  size_t smem = size_t(X) * (MB * X + 1) * sizeof(double2);
  int grid = static_cast<int>(std::min<Dim>((m1 - m0 + MB - 1) / MB, 148 * 8));
  switch (k) {
#define QTNH_DBR(KK)                                                                                    \
  case KK: {                                                                                            \
    static bool attr = [] {                                                                             \
      cudaFuncSetAttribute(k_dist_bitrev<KK>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024); \
      return true;                                                                                      \
    }();                                                                                                \
    (void)attr;                                                                                         \
    k_dist_bitrev<KK><<<grid, 256, smem, st>>>(g, m0, m1);                                              \
    break;                                                                                              \
  }
    QTNH_DBR(1)
    QTNH_DBR(2)
    QTNH_DBR(3)
    QTNH_DBR(4)
#undef QTNH_DBR
    default: throw_invalid("distributed bit reversal needs 1..4 distributed qubits");
  }
  QTNH_LAUNCH_CHECK();
}

void bitrev_hi_local(void* data, int nh, int k, cudaStream_t st) {
  if (nh <= 1) return;
  int B = std::min((11 - k) / 2, nh / 2);
  if (B < 1) throw_invalid("bit reversal: too many held low bits");
  int64_t n_mid = int64_t(1) << (nh - 2 * B);
  size_t smem = size_t(2) * (size_t(1) << B) * ((size_t(1) << (B + k)) + 1) * sizeof(double2);
  static bool attr = [] {
    cudaFuncSetAttribute(k_bitrev_hi, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    return true;
  }();
  (void)attr;
  int grid = static_cast<int>(std::min<int64_t>(n_mid, 148 * 8));
  k_bitrev_hi<<<grid, 256, smem, st>>>(static_cast<double2*>(data), nh, k, B, n_mid);
  QTNH_LAUNCH_CHECK();
}

int qft_group_max() {
  static int v = [] {
    const char* e = std::getenv("QTNH_QFT_G");
    int g = e ? std::atoi(e) : 4;
    return std::max(1, std::min(5, g));
  }();
  return v;
}

void qft_local_fused(void* data, int nb, int first_layer_bit, cudaStream_t st) {
  // Layers with target bits first_layer_bit .. 0 (descending), all local.
  auto* p = static_cast<double2*>(data);
  static const int lmax = [] {
    const char* e = std::getenv("QTNH_QFT_L");
    int v = e ? std::atoi(e) : kQftLowMax;
    return std::max(4, std::min(kQftLowMax, v));
  }();
  // Low-chunk size: fewest strided group passes first, then fewest shared-memory
  // rounds in the low pass (e.g. 28 bits: L = 8 -> 5 group passes of 4 layers +
  // a 2-round low pass, instead of L = 11 -> 4 + 1 passes and 3 rounds).
  int top = first_layer_bit;
  const int layers = top + 1, gmax = qft_group_max();
  static const bool mid_on = [] {
    const char* e = std::getenv("QTNH_QFT_MID");
    return !(e && e[0] == '0');
  }();
  // passes over the state for R upper layers: shared-memory 6-8-layer passes
  // while at least 6 remain (their lowest bit must be >= 4), register groups after
  // (passes, shared-memory passes narrower than 8 layers): a 6- or 7-layer tile is
  // smaller and less efficient (QFT-33: 8 + 8 + 8 over a 9-layer low pass 0.256 s,
  // 8 + 8 + 6 over an 11-layer one 0.275 s)
  auto upper_passes = [&](int l) {
    int R = layers - l, n = 0, narrow = 0;
    while (R > 0) {
      if (mid_on && R >= 6 && l >= 4) {
        narrow += R < 8 ? 1 : 0;
        R -= std::min(R, 8);
      } else {
        R -= std::min(R, gmax);
      }
      ++n;
    }
    return std::make_pair(n, narrow);
  };
  int L = std::min(layers, lmax);
  {
    auto key = [&](int l) { return std::make_tuple(upper_passes(l).first, upper_passes(l).second, (l + 3) / 4); };
    for (int l = std::min(layers, lmax); l >= 1; --l)
      if (key(l) < key(L)) L = l;
  }
  if (mid_on && layers - L >= 6) {
    int dev = 0;
    QTNH_CUDA(cudaGetDevice(&dev));
    static std::mutex mu;
    static std::vector<char> ready(64, 0);
    std::lock_guard<std::mutex> lk(mu);
    if (dev < 64 && !ready[dev]) {
      double2 tw[256] = {};
      for (int u = 0; u < 8; ++u)
        for (int x = 0; x < (1 << u); ++x) {
          const double ang = M_PI * x / std::ldexp(1.0, u);
          tw[(1 << u) - 1 + x] = make_double2(std::cos(ang), std::sin(ang));
        }
      QTNH_CUDA(cudaMemcpyToSymbol(kQftMidTw, tw, sizeof(tw)));
      ready[dev] = 1;
    }
  }
  while (top >= L) {
    const int R = top - L + 1;
    if (mid_on && R >= 6 && L >= 4) {
      const int gb = std::min(R, 8), B = top - gb + 1;
      const int64_t n_tiles = int64_t(1) << (nb - gb - 4);
      const size_t smem = ((size_t(1) << gb) * kMidW + size_t(gb) * kMidW) * sizeof(double2);
      static bool attr = [] {
        const int mx = (256 * kMidW + 8 * kMidW) * 16;
        cudaFuncSetAttribute(k_qft_mid<4, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(k_qft_mid<4, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(k_qft_mid<3, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        return true;
      }();
      (void)attr;
      const int grid = static_cast<int>(std::min<int64_t>(n_tiles, int64_t(148) * 2));
      if (gb == 8) k_qft_mid<4, 4><<<grid, 256, smem, st>>>(p, n_tiles, B);
      else if (gb == 7) k_qft_mid<4, 3><<<grid, 256, smem, st>>>(p, n_tiles, B);
      else k_qft_mid<3, 3><<<grid, 256, smem, st>>>(p, n_tiles, B);
      QTNH_LAUNCH_CHECK();
      top = B - 1;
      continue;
    }
    int g = std::min(qft_group_max(), top - L + 1);  // 5 spills at 255 registers
    int B = top - g + 1;
    QftGroupArgs ga{};
    for (int u = 0; u < 5; ++u)
      for (int k = 0; k < (1 << u); ++k) {
        double ang = M_PI * k / std::ldexp(1.0, u);
        ga.tab[(1 << u) + k] = make_double2(std::cos(ang), std::sin(ang));
      }
    int64_t n_f = int64_t(1) << (nb - g);
    const int64_t one_grid = (n_f + 255) / 256;
    int grid = g == 5 ? static_cast<int>(one_grid) : grid_for(n_f);
    switch (g) {
      case 5: k_qft_group<5><<<grid, 256, 0, st>>>(p, n_f, B, ga); break;
      case 4: k_qft_group<4><<<grid, 256, 0, st>>>(p, n_f, B, ga); break;
      case 3: k_qft_group<3><<<grid, 256, 0, st>>>(p, n_f, B, ga); break;
      case 2: k_qft_group<2><<<grid, 256, 0, st>>>(p, n_f, B, ga); break;
      default: k_qft_group<1><<<grid, 256, 0, st>>>(p, n_f, B, ga); break;
    }
    QTNH_LAUNCH_CHECK();
    top = B - 1;
  }
  if (top >= 0) {
    // remaining layers: bits top..0 with top = L - 1 (all of the low chunk)
    int Lc = top + 1;
    static const int s_cap = [] {  // QTNH_QFT_LOW_S: largest low-pass chunk (bits), default 11
      const char* e = std::getenv("QTNH_QFT_LOW_S");
      return e ? std::max(6, std::min(kQftLowMax, std::atoi(e))) : kQftLowMax;
    }();
    const int S = std::max(Lc, std::min(nb, s_cap));
    const int64_t n_chunks = int64_t(1) << (nb - S);
    const size_t n_tw = static_cast<size_t>(qft_low_tw_count(Lc));
    size_t smem = ((static_cast<size_t>(2) << S) + n_tw) * sizeof(double2);  // 2 buffers + twiddles
    static bool attr = [] {
      cudaFuncSetAttribute(k_qft_low3, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 16 << kQftLowMax);
      return true;
    }();
    (void)attr;
    int dev = 0, occ = 0, sms = 0;
    QTNH_CUDA(cudaGetDevice(&dev));
    QTNH_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    QTNH_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_qft_low3, 128, smem));
    int grid = static_cast<int>(std::min<int64_t>(n_chunks, (int64_t)sms * std::max(1, occ)));
    static const int low_v = [] {  // QTNH_QFT_LOW: tma (default), 4 (registers-first form), 3 (cp.async staging)
      const char* e = std::getenv("QTNH_QFT_LOW");
      return e ? (e[0] == '3' ? 3 : e[0] == '4' ? 4 : 5) : 5;
    }();
    const bool v4 = low_v == 4;
    if (low_v == 5 && S >= 6 && (int64_t(1) << (nb - 3)) <= (int64_t(1) << 31)) {
      static const int nbuf = [] {
        const char* e = std::getenv("QTNH_QFT_LOW_NB");
        const int v = e ? std::atoi(e) : 2;
        return v == 1 || v == 3 ? v : 2;
      }();
      CUtensorMap tm;
      const uint64_t dims[2] = {16, uint64_t(1) << (nb - 3)};
      const uint64_t strides[1] = {128};
      const uint32_t box[2] = {16, static_cast<uint32_t>(1u << (S - 3))};
      make_tensor_map_f64(&tm, p, 2, dims, strides, box, true);
      const size_t smt = ((static_cast<size_t>(nbuf) << S) + n_tw) * sizeof(double2) + 1024;
      static const int minb = [] {  // CTAs per SM the register budget is cut for (3, 4 or 5)
        const char* e = std::getenv("QTNH_QFT_LOW_MINB");
        const int v = e ? std::atoi(e) : 3;
        return v == 4 || v == 5 ? v : 3;
      }();
      auto kern = nbuf == 3 ? k_qft_low_tma<3, 2> : nbuf == 1 ? k_qft_low_tma<1, 4> : k_qft_low_tma<2, 3>;
      if (nbuf == 2 && minb == 4) kern = k_qft_low_tma<2, 4>;
      if (nbuf == 2 && minb == 5) kern = k_qft_low_tma<2, 5>;
      QTNH_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smt)));
      int occt = 0;
      QTNH_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occt, kern, 128, smt));
      const int gridt = static_cast<int>(std::min<int64_t>(n_chunks, (int64_t)sms * std::max(1, occt)));
      kern<<<gridt, 128, smt, st>>>(tm, n_chunks, S, Lc);
    } else if (v4 || low_v == 5) {
      const size_t smem4 = ((size_t(1) << S) + n_tw) * sizeof(double2);
      static bool attr4 = [] {
        cudaFuncSetAttribute(k_qft_low4, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 16 << kQftLowMax);
        return true;
      }();
      (void)attr4;
      int occ4 = 0;
      QTNH_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ4, k_qft_low4, 128, smem4));
      int grid4 = static_cast<int>(std::min<int64_t>(n_chunks, (int64_t)sms * std::max(1, occ4)));
      k_qft_low4<<<grid4, 128, smem4, st>>>(p, n_chunks, S, Lc);
    } else {
      k_qft_low3<<<grid, 128, smem, st>>>(p, n_chunks, S, Lc);
    }
    QTNH_LAUNCH_CHECK();
  }
}

void bitrev_local(void* data, int nb, cudaStream_t st) {
  if (nb < 10) throw_invalid("in-place bit reversal needs at least 10 local qubits");
  int64_t n_mid = int64_t(1) << (nb - 10);
  int dev = 0, occ = 0, sms = 0;
  QTNH_CUDA(cudaGetDevice(&dev));
  QTNH_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  // QTNH_BITREV_TMA=1: the TMA form (read per call). Measured at n = 30 (ncu,
  // cold): 6.35 ms for k_bitrev2 vs 6.41 ms for the best TMA configuration (2
  // stages, 256 threads, 3 CTAs/SM) and 7.9 ms with 6 stages at 1 CTA/SM -- the
  // pass is bound by the DRAM traffic pattern (64 pages per tile pair), not by
  // load issue, so deeper TMA pipelines only add outstanding scattered requests.
  // TMA stores as well (tile pairs exchanged in place in the stage, 8 bulk tensor
  // stores per pair) measured 71-81 ms against 50.6 ms at n = 33: dropped.
  const char* tma_env = std::getenv("QTNH_BITREV_TMA");
  const bool use_tma = tma_env && tma_env[0] == '1';
  if (use_tma && n_mid <= (int64_t(1) << 31)) {
    // QTNH_BITREV_CFG = "stages,threads,ctas_per_sm" (stages 2, 3, 4 or 6)
    static int cfg[3] = {2, 256, 3};
    static bool parsed = [] {
      if (const char* e = std::getenv("QTNH_BITREV_CFG")) std::sscanf(e, "%d,%d,%d", &cfg[0], &cfg[1], &cfg[2]);
      return true;
    }();
    (void)parsed;
    CUtensorMap tm;
    const uint64_t dims[3] = {64, static_cast<uint64_t>(n_mid), 32};
    const uint64_t strides[2] = {512, static_cast<uint64_t>(16) << (nb - 5)};
    const uint32_t box[3] = {16, 1, 32};
    make_tensor_map_f64(&tm, data, 3, dims, strides, box, true);
    const int grid = static_cast<int>(std::min<int64_t>(n_mid, static_cast<int64_t>(sms) * cfg[2]));
    auto launch = [&](auto kern, int S) {
      const size_t smem = static_cast<size_t>(S) * 2048 * sizeof(double2) + 1024;
      QTNH_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
      kern<<<grid, cfg[1], smem, st>>>(tm, static_cast<double2*>(data), nb, n_mid);
    };
    switch (cfg[0]) {
      case 2: launch(k_bitrev_tma<2>, 2); break;
      case 3: launch(k_bitrev_tma<3>, 3); break;
      case 4: launch(k_bitrev_tma<4>, 4); break;
      default: launch(k_bitrev_tma<6>, 6); break;
    }
    QTNH_LAUNCH_CHECK();
    return;
  }
  const size_t smem = 4 * 1024 * sizeof(double2);  // 2 stages x 2 tiles
  static bool attr = [] {
    cudaFuncSetAttribute(k_bitrev2, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    return true;
  }();
  (void)attr;
  QTNH_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_bitrev2, 256, smem));
  int grid = static_cast<int>(std::min<int64_t>(n_mid, (int64_t)sms * std::max(1, occ)));
  k_bitrev2<<<grid, 256, smem, st>>>(static_cast<double2*>(data), nb, n_mid);
  QTNH_LAUNCH_CHECK();
}

}  // namespace qtnhb
