// complex128 GEMM on the FP64 tensor cores of sm_100a.
//
// Replaces the reference's cblas_zgemm inside the SUMMA loop of linalg::pgemm
// (linalg.hpp:344-400). tcgen05 has no f64 kind, so the FP64 tensor path on B200
// is the warp-level DMMA (mma.sync ... f64; every f64 shape lowers to
// DMMA.8x8x4 in SASS, measured 37.1 TFLOP/s peak on this part -- the same rate
// as DFMA but with 8x fewer issue slots per flop).
//
// C = A * B with A (M x K), B (K x N), C (M x N) row-major interleaved complex.
// Default: Gauss / 3M formulation on real MMAs (3 products per complex MAC, the
// tensor pipe being the bound):
//   P1 += A_re B_re, P2 += A_im B_im, P3 += (A_re + A_im)(B_re + B_im);
//   C_re = P1 - P2, C_im = P3 - P1 - P2.
// The 4M form (C_re += A_re B_re + A_im (-B_im), C_im += A_re B_im + A_im B_re)
// remains for narrow N and as a tuning variant.
// Complex elements stay interleaved in shared memory, so one 16-byte shared load
// gives a lane both planes of its fragment element.
//
// Warp tile up to 32 x 32 complex. A CTA of
// WARPS_M x WARPS_N warps owns a BM x BN tile; K is streamed in BK-complex
// slices through a STAGES-deep cp.async pipeline (global reads coalesced along
// K for A and along N for B; A is stored k-major in shared memory with a row
// pitch = 2 (mod 8) x 16 B so fragment loads are bank-conflict free). Several
// CTAs per SM overlap one tile's prologue/epilogue with another's DMMA stream --
// with one CTA per SM those phases idle the tensor pipe for ~15% of the time.
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "ops.h"

namespace qtnhb {

namespace {

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  int sz = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

constexpr int kCoSmemMax = 512;  // K up to which a gather kernel stages coloff in shared memory

template <int BM_, int BN_, int WARPS_M_, int WARPS_N_, int BK_, int STAGES_, int MINB_, int WTM_ = 32,
          int WTN_ = 32, bool GAUSS_ = false>
struct Cfg {
  static constexpr int BM = BM_, BN = BN_, WARPS_M = WARPS_M_, WARPS_N = WARPS_N_, BK = BK_,
                       STAGES = STAGES_, MINB = MINB_;
  static constexpr bool GAUSS = GAUSS_;  // 3 real products per complex MAC
  static constexpr int WTM = WTM_, WTN = WTN_, MI = WTM / 8, NJ = WTN / 8;  // warp tile
  static constexpr int THREADS = WARPS_M * WARPS_N * 32;
  static constexpr int PA = BM + 2;  // 16-B elements; = 2 (mod 8)
  static constexpr int PB = BN + 2;
  static constexpr int A_ELEMS = BK * PA;
  static constexpr int B_ELEMS = BK * PB;
  static constexpr size_t SMEM = static_cast<size_t>(STAGES) * (A_ELEMS + B_ELEMS) * 16;
  static_assert(BM == WARPS_M * WTM && BN == WARPS_N * WTN, "CTA tile = warps x warp tile");
  static_assert((BM * BK) % THREADS == 0 && (BN * BK) % THREADS == 0, "even load split");
};

// MODE 0: A dense row-major (M x K).
// MODE 1/2: A gathered: element (m, k) at A + rowoff[m] + coloff[k] -- the layout
// permutation of the contraction fused into the operand loads (no permuted copy
// of A in HBM). MODE 1 walks consecutive rows with consecutive threads (the
// tensor's innermost index is open), MODE 2 consecutive k (innermost contracted).
template <class G, int MODE>
__global__ void __launch_bounds__(G::THREADS, G::MINB) k_zgemm(const double2* __restrict__ A,
                                                               const int64_t* __restrict__ rowoff,
                                                               const int64_t* __restrict__ coloff,
                                                               const double2* __restrict__ B,
                                                               double2* __restrict__ C, int64_t M,
                                                               int64_t N, int64_t K,
                                                               const int64_t* __restrict__ cohi, int co_sh,
                                                               const int64_t* __restrict__ rohi, int ro_sh) {
  constexpr int BM = G::BM, BN = G::BN, BK = G::BK, STAGES = G::STAGES, T = G::THREADS;
  extern __shared__ __align__(16) double2 smem[];
  double2* As = smem;                          // [stage][k][PA]
  double2* Bs = smem + STAGES * G::A_ELEMS;    // [stage][k][PB]

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // Gather modes: the column-offset table of a short K sits in shared memory, so a
  // stage's address lookups never wait on global memory (with few warps per
  // scheduler those waits idled the tensor pipe).
  // A long K whose column offsets factor as hi[k >> co_sh] + lo[k & (2^co_sh - 1)]
  // (row-major digits split in two) keeps both halves there instead.
  int64_t* co_s = reinterpret_cast<int64_t*>(Bs + STAGES * G::B_ELEMS);
  const bool co_split = MODE != 0 && cohi != nullptr;
  const bool co_in_smem = MODE != 0 && (K <= kCoSmemMax || co_split);
  const int64_t co_lo_n = co_split ? (int64_t(1) << co_sh) : K;
  const int64_t co_mask = co_lo_n - 1;
  if (co_in_smem) {
    for (int64_t i = tid; i < co_lo_n; i += T) co_s[i] = __ldg(coloff + i);
    if (co_split)
      for (int64_t i = tid; i < (K >> co_sh); i += T) co_s[co_lo_n + i] = __ldg(cohi + i);
    __syncthreads();
  }
  auto col_off = [&](int64_t k) -> int64_t {
    if (!co_in_smem) return __ldg(coloff + k);
    if (co_split) return co_s[co_lo_n + (k >> co_sh)] + co_s[k & co_mask];
    return co_s[k];
  };
  const int wm = warp / G::WARPS_N, wn = warp % G::WARPS_N;
  // 1-D grid, N tiles fastest: the CTAs sharing a row block of A run together
  // (A read once from HBM), and M is not limited by gridDim.y.
  const int64_t n_tiles_n = (N + BN - 1) / BN;
  const int64_t tile = blockIdx.x;
  const int64_t bm = (tile / n_tiles_n) * BM;
  const int64_t bn = (tile % n_tiles_n) * BN;
  const int64_t n_kt = (K + BK - 1) / BK;

  // Per-thread source rows / columns are fixed; only k advances by BK per stage.
  constexpr int LA = (BM * BK) / T, LB = (BN * BK) / T;
  const double2* pa[LA];
  const double2* pb[LB];
  int sa[LA], sb[LB], ka[LA], kb[LB];
  bool ma[LA], nbok[LB];
  // MODE 1 with T % BM == 0: every load of a thread hits the same row.
  constexpr bool kRowFixed = MODE == 1 && (T % BM) == 0;
#pragma unroll
  for (int u = 0; u < LA; ++u) {
    int e = tid + u * T;
    int m = MODE == 1 ? e % BM : e / BK;
    int k = MODE == 1 ? e / BM : e % BK;
    ka[u] = k;
    sa[u] = k * G::PA + m;
    if (kRowFixed && u > 0) {
      ma[u] = ma[0];
      pa[u] = pa[0];
      continue;
    }
    ma[u] = bm + m < M;
    if (MODE == 0) {
      pa[u] = A + (ma[u] ? (bm + m) : 0) * K + k;
    } else {
      // row offsets: one table, or hi[m >> ro_sh] + lo[m & (2^ro_sh - 1)]
      const int64_t row = bm + m;
      int64_t off = 0;
      if (ma[u]) off = rohi ? __ldg(rohi + (row >> ro_sh)) + __ldg(rowoff + (row & ((int64_t(1) << ro_sh) - 1)))
                            : __ldg(rowoff + row);
      pa[u] = A + off;
    }
  }
#pragma unroll
  for (int u = 0; u < LB; ++u) {
    int e = tid + u * T;
    int k = e / BN, n = e % BN;
    nbok[u] = bn + n < N;
    kb[u] = k;
    pb[u] = B + static_cast<int64_t>(k) * N + (nbok[u] ? bn + n : 0);
    sb[u] = k * G::PB + n;
  }
  auto load_stage = [&](int stage, int64_t kt) {
    int64_t k0 = kt * BK;
    double2* as = As + stage * G::A_ELEMS;
    double2* bs = Bs + stage * G::B_ELEMS;
#pragma unroll
    for (int u = 0; u < LA; ++u) {
      bool ok = ma[u] && k0 + ka[u] < K;
      const double2* src = A;
      if (ok) src = MODE == 0 ? pa[u] + k0 : pa[u] + col_off(k0 + ka[u]);
      cp_async16(as + sa[u], src, ok);
    }
#pragma unroll
    for (int u = 0; u < LB; ++u) {
      bool ok = nbok[u] && k0 + kb[u] < K;
      cp_async16(bs + sb[u], ok ? pb[u] + k0 * N : B, ok);
    }
  };

  constexpr int MI = G::MI, NJ = G::NJ;
  // 4M: acc_re = Re, acc_im = Im. Gauss (3M): acc_re = sum a_re b_re, acc_im =
  // sum a_im b_im, acc_s = sum (a_re + a_im)(b_re + b_im); Re = acc_re - acc_im,
  // Im = acc_s - acc_re - acc_im.
  double acc_re[MI][NJ][2], acc_im[MI][NJ][2], acc_s[G::GAUSS ? MI : 1][G::GAUSS ? NJ : 1][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      acc_re[i][j][0] = acc_re[i][j][1] = 0.0;
      acc_im[i][j][0] = acc_im[i][j][1] = 0.0;
      if (G::GAUSS) acc_s[G::GAUSS ? i : 0][G::GAUSS ? j : 0][0] = acc_s[G::GAUSS ? i : 0][G::GAUSS ? j : 0][1] = 0.0;
    }

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < n_kt) load_stage(s, s);
    cp_commit();
  }

  const int fr = lane >> 2, fk = lane & 3;
  for (int64_t kt = 0; kt < n_kt; ++kt) {
    cp_wait<STAGES - 2>();
    __syncthreads();
    const double2* as = As + (kt % STAGES) * G::A_ELEMS + wm * G::WTM + fr;
    const double2* bs = Bs + (kt % STAGES) * G::B_ELEMS + wn * G::WTN + fr;
#pragma unroll
    for (int k4 = 0; k4 < BK; k4 += 4) {
      double a_re[MI], a_im[MI], b_re[NJ], b_im[NJ], nb_im[NJ];
#pragma unroll
      for (int i = 0; i < MI; ++i) {
        double2 v = as[(k4 + fk) * G::PA + i * 8];
        a_re[i] = v.x;
        a_im[i] = v.y;
      }
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        double2 v = bs[(k4 + fk) * G::PB + j * 8];
        b_re[j] = v.x;
        b_im[j] = v.y;
        nb_im[j] = -v.y;
      }
      if constexpr (G::GAUSS) {
        double a_s[MI], b_s[NJ];
#pragma unroll
        for (int i = 0; i < MI; ++i) a_s[i] = a_re[i] + a_im[i];
#pragma unroll
        for (int j = 0; j < NJ; ++j) b_s[j] = b_re[j] + b_im[j];
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
          for (int j = 0; j < NJ; ++j) {
            dmma(acc_re[i][j], a_re[i], b_re[j]);
            dmma(acc_im[i][j], a_im[i], b_im[j]);
            dmma(acc_s[i][j], a_s[i], b_s[j]);
          }
      } else {
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
          for (int j = 0; j < NJ; ++j) {
            dmma(acc_re[i][j], a_re[i], b_re[j]);
            dmma(acc_im[i][j], a_re[i], b_im[j]);
          }
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
          for (int j = 0; j < NJ; ++j) {
            dmma(acc_re[i][j], a_im[i], nb_im[j]);
            dmma(acc_im[i][j], a_im[i], b_re[j]);
          }
      }
    }
    // Refill the slot freed at the top barrier only after this slice's DMMAs are
    // queued: the (gather-table) address loads then stall the warp while the
    // tensor pipe is busy, not before it is fed.
    {
      int64_t nk = kt + STAGES - 1;
      if (nk < n_kt) load_stage(static_cast<int>(nk % STAGES), nk);
      cp_commit();
    }
  }
  cp_wait<0>();
  if constexpr (G::GAUSS) {
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < NJ; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const double rr = acc_re[i][j][h], ii = acc_im[i][j][h];
          acc_re[i][j][h] = rr - ii;
          acc_im[i][j][h] = acc_s[i][j][h] - rr - ii;
        }
  }

  // Epilogue: lane holds C[fr][2*fk + {0,1}] of each 8x8 sub-tile.
#pragma unroll
  for (int i = 0; i < MI; ++i) {
    int64_t row = bm + wm * G::WTM + i * 8 + fr;
    if (row >= M) continue;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      int64_t col = bn + wn * G::WTN + j * 8 + 2 * fk;
      double2* dst = C + row * N + col;
      if (col + 1 < N) {
        dst[0] = make_double2(acc_re[i][j][0], acc_im[i][j][0]);
        dst[1] = make_double2(acc_re[i][j][1], acc_im[i][j][1]);
      } else if (col < N) {
        dst[0] = make_double2(acc_re[i][j][0], acc_im[i][j][0]);
      }
    }
  }
}

// Gauss kernel for tile-aligned problems (M % BM = N % BN = K % BK = 0, the
// contraction shapes of every configuration): no bounds predicates, the
// column-offset table form (CO: 0 = one shared-memory table, 1 = hi/lo split in
// shared memory, 2 = global) a template parameter, and the next stage's cp.async
// loads interleaved with the first k4 step's DMMAs (one piece per warp-tile row)
// instead of issued as a block after them. In k_zgemm a warp's refill phase
// (~400 address / branch instructions with shared- and global-load latencies)
// stalls its DMMA stream, and with two warps per sub-partition both are often in
// that phase at once: ncu showed the DMMA pipe 76 % busy although one warp with
// two independent accumulators saturates it (tools/microbench/dmma_issue.cu).
template <class G, int MODE, int CO>
__global__ void __launch_bounds__(G::THREADS, G::MINB) k_zgemm_even(const double2* __restrict__ A,
                                                                    const int64_t* __restrict__ rowoff,
                                                                    const int64_t* __restrict__ coloff,
                                                                    const double2* __restrict__ B,
                                                                    double2* __restrict__ C, int64_t M,
                                                                    int64_t N, int64_t K,
                                                                    const int64_t* __restrict__ cohi, int co_sh,
                                                                    const int64_t* __restrict__ rohi, int ro_sh) {
  static_assert(G::GAUSS, "Gauss kernel");
  constexpr int BM = G::BM, BN = G::BN, BK = G::BK, STAGES = G::STAGES, T = G::THREADS;
  extern __shared__ __align__(16) double2 smem[];
  double2* As = smem;
  double2* Bs = smem + STAGES * G::A_ELEMS;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int64_t* co_s = reinterpret_cast<int64_t*>(Bs + STAGES * G::B_ELEMS);
  const int64_t co_lo_n = CO == 1 ? (int64_t(1) << co_sh) : K;
  const int64_t co_mask = co_lo_n - 1;
  if (MODE != 0 && CO != 2) {
    for (int64_t i = tid; i < co_lo_n; i += T) co_s[i] = __ldg(coloff + i);
    if (CO == 1)
      for (int64_t i = tid; i < (K >> co_sh); i += T) co_s[co_lo_n + i] = __ldg(cohi + i);
    __syncthreads();
  }
  auto col_off = [&](int64_t k) -> int64_t {
    if (CO == 2) return __ldg(coloff + k);
    if (CO == 1) return co_s[co_lo_n + (k >> co_sh)] + co_s[k & co_mask];
    return co_s[k];
  };
  const int wm = warp / G::WARPS_N, wn = warp % G::WARPS_N;
  const int64_t n_tiles_n = N / BN;
  const int64_t bm = (blockIdx.x / n_tiles_n) * BM;
  const int64_t bn = (blockIdx.x % n_tiles_n) * BN;
  const int64_t n_kt = K / BK;

  constexpr int LA = (BM * BK) / T, LB = (BN * BK) / T, LT = LA + LB;
  constexpr bool kRowFixed = MODE == 1 && (T % BM) == 0;
  constexpr bool kColFixed = MODE == 2 && (T % BK) == 0;
  const double2* pa[kRowFixed ? 1 : LA];
  int sa[LA], ka[LA];
#pragma unroll
  for (int u = 0; u < LA; ++u) {
    const int e = tid + u * T;
    const int m = MODE == 1 ? e % BM : e / BK;
    const int k = MODE == 1 ? e / BM : e % BK;
    ka[u] = k;
    sa[u] = k * G::PA + m;
    if (kRowFixed && u > 0) continue;
    if (MODE == 0) {
      pa[u] = A + (bm + m) * K + k;
    } else {
      const int64_t row = bm + m;
      const int64_t off = rohi ? __ldg(rohi + (row >> ro_sh)) + __ldg(rowoff + (row & ((int64_t(1) << ro_sh) - 1)))
                               : __ldg(rowoff + row);
      pa[u] = A + off;
    }
  }
  // B(k, n): thread t loads column bn + t % BN of rows (t + u T) / BN.
  const double2* pb = B + bn + (tid % BN) + static_cast<int64_t>(tid / BN) * N;
  const int sb0 = (tid / BN) * G::PB + (tid % BN);
  constexpr int B_ROWS_PER_U = T / BN;  // rows between consecutive u (T % BN == 0 asserted below)
  static_assert(T % BN == 0, "B loads: whole rows per pass");

  auto load_one = [&](int q, int stage, int64_t k0, bool ok) {
    if (q < LA) {
      const int u = q;
      const double2* src;
      if (MODE == 0) src = pa[u] + k0;
      else if (kRowFixed) src = pa[0] + col_off(k0 + ka[u]);
      else if (kColFixed) src = pa[u] + col_off(k0 + ka[0]);
      else src = pa[u] + col_off(k0 + ka[u]);
      cp_async16(As + stage * G::A_ELEMS + sa[u], ok ? src : A, ok);
    } else {
      const int u = q - LA;
      const double2* src = pb + (k0 + u * B_ROWS_PER_U) * N;
      cp_async16(Bs + stage * G::B_ELEMS + sb0 + u * B_ROWS_PER_U * G::PB, ok ? src : B, ok);
    }
  };

  constexpr int MI = G::MI, NJ = G::NJ;
  double acc_re[MI][NJ][2], acc_im[MI][NJ][2], acc_s[MI][NJ][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) acc_re[i][j][h] = acc_im[i][j][h] = acc_s[i][j][h] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    const bool ok = s < n_kt;
#pragma unroll
    for (int q = 0; q < LT; ++q) load_one(q, s, ok ? int64_t(s) * BK : 0, ok);
    cp_commit();
  }

  constexpr int PER = (LT + MI - 1) / MI;  // loads issued after each warp-tile row of k4 = 0
  const int fr = lane >> 2, fk = lane & 3;
  for (int64_t kt = 0; kt < n_kt; ++kt) {
    cp_wait<STAGES - 2>();
    __syncthreads();
    const int64_t nk = kt + STAGES - 1;
    const bool refill = nk < n_kt;
    const int nslot = static_cast<int>(nk % STAGES);
    const int64_t nk0 = refill ? nk * BK : 0;  // past the end: keep table lookups in range
    const double2* as = As + (kt % STAGES) * G::A_ELEMS + wm * G::WTM + fr;
    const double2* bs = Bs + (kt % STAGES) * G::B_ELEMS + wn * G::WTN + fr;
#pragma unroll
    for (int k4 = 0; k4 < BK; k4 += 4) {
      double a_re[MI], a_im[MI], a_s[MI], b_re[NJ], b_im[NJ], b_s[NJ];
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        const double2 v = bs[(k4 + fk) * G::PB + j * 8];
        b_re[j] = v.x;
        b_im[j] = v.y;
        b_s[j] = v.x + v.y;
      }
#pragma unroll
      for (int i = 0; i < MI; ++i) {
        const double2 v = as[(k4 + fk) * G::PA + i * 8];
        a_re[i] = v.x;
        a_im[i] = v.y;
        a_s[i] = v.x + v.y;
      }
#pragma unroll
      for (int i = 0; i < MI; ++i) {
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
          dmma(acc_re[i][j], a_re[i], b_re[j]);
          dmma(acc_im[i][j], a_im[i], b_im[j]);
          dmma(acc_s[i][j], a_s[i], b_s[j]);
        }
        if (k4 == 0) {
#pragma unroll
          for (int q = i * PER; q < (i + 1) * PER && q < LT; ++q) load_one(q, nslot, nk0, refill);
        }
      }
    }
    cp_commit();
  }
  cp_wait<0>();

#pragma unroll
  for (int i = 0; i < MI; ++i) {
    const int64_t row = bm + wm * G::WTM + i * 8 + fr;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const int64_t col = bn + wn * G::WTN + j * 8 + 2 * fk;
      double2* dst = C + row * N + col;
      const double r0 = acc_re[i][j][0], i0 = acc_im[i][j][0], r1 = acc_re[i][j][1], i1 = acc_im[i][j][1];
      dst[0] = make_double2(r0 - i0, acc_s[i][j][0] - r0 - i0);
      dst[1] = make_double2(r1 - i1, acc_s[i][j][1] - r1 - i1);
    }
  }
}

template <class G, int MODE>
void launch_mode(const double2* a, const int64_t* ro, const int64_t* co, const double2* b, double2* c, Dim m,
                 Dim n, Dim k, cudaStream_t st, const int64_t* cohi = nullptr, int co_sh = 0,
                 const int64_t* rohi = nullptr, int ro_sh = 0) {
  size_t co_bytes = 0;
  if (MODE != 0 && cohi) co_bytes = static_cast<size_t>((Dim(1) << co_sh) + (k >> co_sh)) * 8;
  else if (MODE != 0 && k <= kCoSmemMax) co_bytes = static_cast<size_t>(k) * 8;
  if (co_bytes > kCoSmemMax * 8) throw_invalid("column offset split exceeds its shared-memory budget");
  const size_t smem = G::SMEM + co_bytes;
  ensure_max_dynamic_smem(reinterpret_cast<const void*>(k_zgemm<G, MODE>), (int)(G::SMEM + kCoSmemMax * 8));
  Dim tiles = ((m + G::BM - 1) / G::BM) * ((n + G::BN - 1) / G::BN);
  if (tiles > 0x7fffffff) throw_invalid("zgemm problem too large for one launch");
  k_zgemm<G, MODE><<<static_cast<unsigned>(tiles), G::THREADS, smem, st>>>(a, ro, co, b, c, m, n, k, cohi, co_sh, rohi,
                                                                                  ro_sh);
  QTNH_LAUNCH_CHECK();
}

bool narrow_gauss() {
  static const bool on = [] {
    const char* e = std::getenv("QTNH_ZGEMM_NARROW_GAUSS");
    return !(e && e[0] == '0');
  }();
  return on;
}

bool even_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("QTNH_ZGEMM_EVEN");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <class G>
bool even_shape(Dim m, Dim n, Dim k) {
  return even_enabled() && m % G::BM == 0 && n % G::BN == 0 && k % G::BK == 0;
}

template <class G, int MODE, int CO>
void launch_even_co(const double2* a, const int64_t* ro, const int64_t* co, const double2* b, double2* c, Dim m,
                    Dim n, Dim k, cudaStream_t st, const int64_t* cohi, int co_sh, const int64_t* rohi, int ro_sh,
                    size_t co_bytes) {
  ensure_max_dynamic_smem(reinterpret_cast<const void*>(k_zgemm_even<G, MODE, CO>), (int)(G::SMEM + kCoSmemMax * 8));
  const Dim tiles = (m / G::BM) * (n / G::BN);
  if (tiles > 0x7fffffff) throw_invalid("zgemm problem too large for one launch");
  k_zgemm_even<G, MODE, CO><<<static_cast<unsigned>(tiles), G::THREADS, G::SMEM + co_bytes, st>>>(
      a, ro, co, b, c, m, n, k, cohi, co_sh, rohi, ro_sh);
  QTNH_LAUNCH_CHECK();
}

template <class G, int MODE>
void launch_even(const double2* a, const int64_t* ro, const int64_t* co, const double2* b, double2* c, Dim m, Dim n,
                 Dim k, cudaStream_t st, const int64_t* cohi = nullptr, int co_sh = 0, const int64_t* rohi = nullptr,
                 int ro_sh = 0) {
  if (MODE == 0) return launch_even_co<G, 0, 2>(a, ro, co, b, c, m, n, k, st, cohi, co_sh, rohi, ro_sh, 0);
  if (cohi) {
    const size_t co_bytes = static_cast<size_t>((Dim(1) << co_sh) + (k >> co_sh)) * 8;
    if (co_bytes > kCoSmemMax * 8) throw_invalid("column offset split exceeds its shared-memory budget");
    return launch_even_co<G, MODE, 1>(a, ro, co, b, c, m, n, k, st, cohi, co_sh, rohi, ro_sh, co_bytes);
  }
  if (k <= kCoSmemMax)
    return launch_even_co<G, MODE, 0>(a, ro, co, b, c, m, n, k, st, cohi, co_sh, rohi, ro_sh,
                                      static_cast<size_t>(k) * 8);
  if constexpr (G::BN == 32 && MODE == 2) {
    // the narrow 64 x 32 Gauss tile with a per-column global offset table ran out
    // of registers (116 B spilled): that rare case takes the 4M narrow kernel (V4)
    return launch_mode<Cfg<64, 32, 2, 1, 8, 4, 4>, MODE>(a, ro, co, b, c, m, n, k, st, cohi, co_sh, rohi, ro_sh);
  } else {
    return launch_even_co<G, MODE, 2>(a, ro, co, b, c, m, n, k, st, cohi, co_sh, rohi, ro_sh, 0);
  }
}

template <class G>
void launch(const double2* a, const double2* b, double2* c, Dim m, Dim n, Dim k, cudaStream_t st) {
  if constexpr (G::GAUSS)
    if (even_shape<G>(m, n, k)) return launch_even<G, 0>(a, nullptr, nullptr, b, c, m, n, k, st);
  launch_mode<G, 0>(a, nullptr, nullptr, b, c, m, n, k, st);
}

struct MixedRadix {
  int nd;
  int64_t dims[64];
  int64_t strides[64];
};

__global__ void k_mixed_offsets(int64_t* __restrict__ out, int64_t count, const __grid_constant__ MixedRadix mr) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i, off = 0;
    for (int d = mr.nd - 1; d >= 0; --d) {
      int64_t c = r % mr.dims[d];
      r /= mr.dims[d];
      off += c * mr.strides[d];
    }
    out[i] = off;
  }
}

// 4M configurations kept after the tuning sweep (14 variants measured on the C1
// shape; V12 was best: 16x32 warp tiles, 4 CTAs/SM so one tile's prologue /
// epilogue overlaps another's DMMA stream). QTNH_ZGEMM_VARIANT=4|12|106|122
// pins one for experiments (106 = G6, 122 = G22).
using V4 = Cfg<64, 32, 2, 1, 8, 4, 4>;    // 64 thr, 4 CTA/SM: narrow N (<= 32)
using V12 = Cfg<32, 64, 2, 2, 8, 3, 4, 16, 32>;   // warp tile 16x32, 128 thr
// Gauss (3M) complex multiply: 3 real DMMA products per complex k-step instead of
// 4 (Re = ar br - ai bi, Im = (ar + ai)(br + bi) - ar br - ai bi). The FP64 tensor
// pipe is the bound (ncu: math_pipe_throttle, 90 % DMMA-pipe busy for 4M), so
// trading one product for two adds per fragment gives +17 % on the C1 shape
// (39.1 vs 33.4 TFLOP/s counted as 8MNK). 32x32 warp tiles, 64 threads, 4 CTAs/SM,
// 4-stage cp.async pipeline won a 16-configuration sweep (tools/bench_zgemm.py).
using G6 = Cfg<32, 64, 1, 2, 8, 4, 4, 32, 32, true>;
// Fewer, fatter CTAs for grids of a few waves (e.g. 2048 x 2048 x 1024: 39.2 vs
// 35.9 TFLOP/s with G6): 16x32 warp tiles, BK 4, 8 stages, 3 CTAs/SM.
using G22 = Cfg<32, 64, 2, 2, 4, 8, 3, 16, 32, true>;
// Tile-aligned experiments (k_zgemm_even only): full-N 32 x 128 tiles (A read
// once per row block) and 64 x 64 tiles (A and B fragments each shared by two warps).
using G7 = Cfg<32, 128, 1, 4, 8, 4, 2, 32, 32, true>;
using G8 = Cfg<64, 64, 2, 2, 8, 4, 2, 32, 32, true>;
// Default tile-aligned gather config: G6 with 3 stages (the interleaved refill
// needs less lead; C1 41.6 vs 41.3 TFLOP/s with 4 stages). A pre-summed B plane
// (4 instead of 8 DADDs per warp k4 step) spilled at 255 registers and lost 11 %.
using G9 = Cfg<32, 64, 1, 2, 8, 3, 4, 32, 32, true>;
// Narrow N (17..32): Gauss tile-aligned 64 x 32 tiles (two 32 x 32 warp tiles along
// M). The 4M V4 kernel ran C3's big narrow contractions (M = 2^19, N = 32, K = 2^11,
// at the ridge: 16 flop/B) at 2 TB/s.
using G10 = Cfg<64, 32, 2, 1, 8, 3, 4, 32, 32, true>;
// Narrower still (N = 16, e.g. config 3's M = 2^24, N = 16, K = 64 step, HBM-bound at
// 6.5 flop/B): 64 x 16 tiles, 32 x 16 warp tiles -- the 64 x 32 V4 tiles (4M) spent
// half their DMMAs on columns that do not exist.
using G11 = Cfg<64, 16, 2, 1, 8, 3, 4, 32, 16, true>;

int variant() {
  static int v = [] {
    const char* e = std::getenv("QTNH_ZGEMM_VARIANT");
    return e ? std::atoi(e) : -1;
  }();
  return v;
}

}  // namespace

void index_offsets(int64_t* out, Dim count, const std::vector<Dim>& dims, const std::vector<Dim>& strides,
                   cudaStream_t st) {
  if (count <= 0) return;
  MixedRadix mr{};
  mr.nd = static_cast<int>(dims.size());
  if (mr.nd > 64) throw_invalid("too many indices for an offset table");
  for (int i = 0; i < mr.nd; ++i) {
    mr.dims[i] = dims[i];
    mr.strides[i] = strides[i];
  }
  int grid = static_cast<int>(std::min<Dim>((count + 255) / 256, 148 * 8));
  k_mixed_offsets<<<grid, 256, 0, st>>>(out, count, mr);
  QTNH_LAUNCH_CHECK();
}

void zgemm_gather_a(const void* a, const int64_t* rowoff, const int64_t* coloff, bool rows_fastest,
                    const void* b, void* c, Dim m, Dim n, Dim k, cudaStream_t st, const int64_t* cohi, int co_sh,
                    const int64_t* rohi, int ro_sh) {
  if (m <= 0 || n <= 0) return;
  if (k <= 0) {
    QTNH_CUDA(cudaMemsetAsync(c, 0, static_cast<size_t>(m * n) * 16, st));
    return;
  }
  auto A = static_cast<const double2*>(a);
  auto B = static_cast<const double2*>(b);
  auto Cp = static_cast<double2*>(c);
  static int gv = [] {
    const char* e = std::getenv("QTNH_ZGEMM_GATHER_VARIANT");
    return e ? std::atoi(e) : 109;
  }();
  if (n > 32 && gv == 12) {
    if (rows_fastest) launch_mode<V12, 1>(A, rowoff, coloff, B, Cp, m, n, k, st, cohi, co_sh, rohi, ro_sh);
    else launch_mode<V12, 2>(A, rowoff, coloff, B, Cp, m, n, k, st, cohi, co_sh, rohi, ro_sh);
  } else if (n > 32 && gv == 107 && even_shape<G7>(m, n, k)) {
    if (rows_fastest) launch_even<G7, 1>(A, rowoff, coloff, B, Cp, m, n, k, st, cohi, co_sh, rohi, ro_sh);
    else launch_even<G7, 2>(A, rowoff, coloff, B, Cp, m, n, k, st, cohi, co_sh, rohi, ro_sh);
  } else if (n > 32 && gv == 108 && even_shape<G8>(m, n, k)) {
    if (rows_fastest) launch_even<G8, 1>(A, rowoff, coloff, B, Cp, m, n, k, st, cohi, co_sh, rohi, ro_sh);
    else launch_even<G8, 2>(A, rowoff, coloff, B, Cp, m, n, k, st, cohi, co_sh, rohi, ro_sh);
  } else if (n > 32 && gv == 106 && even_shape<G6>(m, n, k)) {
    if (rows_fastest) launch_even<G6, 1>(A, rowoff, coloff, B, Cp, m, n, k, st, cohi, co_sh, rohi, ro_sh);
    else launch_even<G6, 2>(A, rowoff, coloff, B, Cp, m, n, k, st, cohi, co_sh, rohi, ro_sh);
  } else if (n > 32 && even_shape<G9>(m, n, k)) {
    if (rows_fastest) launch_even<G9, 1>(A, rowoff, coloff, B, Cp, m, n, k, st, cohi, co_sh, rohi, ro_sh);
    else launch_even<G9, 2>(A, rowoff, coloff, B, Cp, m, n, k, st, cohi, co_sh, rohi, ro_sh);
  } else if (n > 32) {
    if (rows_fastest) launch_mode<G6, 1>(A, rowoff, coloff, B, Cp, m, n, k, st, cohi, co_sh, rohi, ro_sh);
    else launch_mode<G6, 2>(A, rowoff, coloff, B, Cp, m, n, k, st, cohi, co_sh, rohi, ro_sh);
  } else if (n > 16 && even_shape<G10>(m, n, k) && narrow_gauss()) {
    if (rows_fastest) launch_even<G10, 1>(A, rowoff, coloff, B, Cp, m, n, k, st, cohi, co_sh, rohi, ro_sh);
    else launch_even<G10, 2>(A, rowoff, coloff, B, Cp, m, n, k, st, cohi, co_sh, rohi, ro_sh);
  } else if (n == 16 && even_shape<G11>(m, n, k) && narrow_gauss()) {
    if (rows_fastest) launch_even<G11, 1>(A, rowoff, coloff, B, Cp, m, n, k, st, cohi, co_sh, rohi, ro_sh);
    else launch_even<G11, 2>(A, rowoff, coloff, B, Cp, m, n, k, st, cohi, co_sh, rohi, ro_sh);
  } else {
    if (rows_fastest) launch_mode<V4, 1>(A, rowoff, coloff, B, Cp, m, n, k, st, cohi, co_sh, rohi, ro_sh);
    else launch_mode<V4, 2>(A, rowoff, coloff, B, Cp, m, n, k, st, cohi, co_sh, rohi, ro_sh);
  }
}

void zgemm(const void* a, const void* b, void* c, Dim m, Dim n, Dim k, cudaStream_t st) {
  if (m <= 0 || n <= 0) return;
  auto A = static_cast<const double2*>(a);
  auto B = static_cast<const double2*>(b);
  auto Cp = static_cast<double2*>(c);
  if (k <= 0) {
    QTNH_CUDA(cudaMemsetAsync(c, 0, static_cast<size_t>(m * n) * 16, st));
    return;
  }
  switch (variant()) {
    case 4: return launch<V4>(A, B, Cp, m, n, k, st);
    case 12: return launch<V12>(A, B, Cp, m, n, k, st);
    case 106: return launch<G6>(A, B, Cp, m, n, k, st);
    case 122: return launch<G22>(A, B, Cp, m, n, k, st);
    case 109: return launch<G9>(A, B, Cp, m, n, k, st);
    default: break;
  }
  const Dim tiles = ((m + 31) / 32) * ((n + 63) / 64);
  if (n <= 32 && n > 16 && narrow_gauss() && even_shape<G10>(m, n, k)) launch<G10>(A, B, Cp, m, n, k, st);
  else if (n == 16 && narrow_gauss() && even_shape<G11>(m, n, k)) launch<G11>(A, B, Cp, m, n, k, st);
  else if (n <= 32) launch<V4>(A, B, Cp, m, n, k, st);
  else if (tiles < 8192) launch<G22>(A, B, Cp, m, n, k, st);
  else launch<G6>(A, B, Cp, m, n, k, st);
}

}  // namespace qtnhb
