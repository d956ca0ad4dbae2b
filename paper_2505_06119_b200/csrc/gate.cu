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
#include <cstring>

#include "ops.h"

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

template <int D, bool POW2>
__global__ void __launch_bounds__(256) k_gate_dense(double2* __restrict__ psi, int64_t n_fibers,
                                                    const __grid_constant__ GateArgs a) {
  for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < n_fibers;
       f += (int64_t)gridDim.x * blockDim.x) {
    int64_t base = fiber_base<POW2>(f, a);
    double2 x[D];
#pragma unroll
    for (int d = 0; d < D; ++d) x[d] = psi[base + a.off[d]];
#pragma unroll
    for (int i = 0; i < D; ++i) {
      double re = 0.0, im = 0.0;
#pragma unroll
      for (int d = 0; d < D; ++d) {
        double2 g = a.g[i * D + d];
        re = fma(g.x, x[d].x, re);
        re = fma(-g.y, x[d].y, re);
        im = fma(g.x, x[d].y, im);
        im = fma(g.y, x[d].x, im);
      }
      psi[base + a.off[i]] = make_double2(re, im);
    }
  }
}

// Generic D (non power of two, or > kMaxD handled by host splitting): loops.
template <bool POW2>
__global__ void __launch_bounds__(256) k_gate_generic(double2* __restrict__ psi, int64_t n_fibers,
                                                      const __grid_constant__ GateArgs a) {
  for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < n_fibers;
       f += (int64_t)gridDim.x * blockDim.x) {
    int64_t base = fiber_base<POW2>(f, a);
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
    int64_t base = fiber_base<POW2>(f, a);
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
  int r = static_cast<int>(dims.size());
  int k = static_cast<int>(targets.size());
  if (k == 0) throw_invalid("gate needs at least one target");
  std::vector<char> is_t(r, 0);
  for (int t : targets) {
    if (t < 0 || t >= r || is_t[t]) throw_invalid("invalid gate targets");
    is_t[t] = 1;
  }
  auto strides = row_major_strides(dims);
  GateArgs a{};
  Dim D = 1;
  for (int t : targets) D *= dims[t];
  Dim total = 1;
  for (Dim d : dims) total *= d;
  if (total == 0) return;
  Dim n_fibers = total / D;
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

}  // namespace qtnhb
