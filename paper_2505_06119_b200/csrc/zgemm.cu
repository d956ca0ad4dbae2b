// complex128 GEMM on the FP64 tensor cores of sm_100a.
//
// Replaces the reference's cblas_zgemm inside the SUMMA loop of linalg::pgemm
// (linalg.hpp:344-400). tcgen05 has no f64 kind, so the FP64 tensor path on B200
// is the warp-level DMMA (mma.sync ... f64; every f64 shape lowers to
// DMMA.8x8x4 in SASS, measured 37.1 TFLOP/s peak on this part -- the same rate
// as DFMA but 8x fewer issue slots per flop).
//
// C = A * B with A (M x K), B (K x N), C (M x N) row-major interleaved complex.
// 4M formulation on real MMAs, keeping the algorithmic 8MNK flops:
//   C_re += A_re B_re + A_im (-B_im),   C_im += A_re B_im + A_im B_re.
// Complex elements stay interleaved in shared memory, so one 16-byte shared load
// gives a lane both planes of its fragment element.
//
// CTA: 256 threads (8 warps) own a BM x BN complex tile (warp tile 32 x 32, 64
// fp64 accumulators per lane); K is streamed in BK = 8 complex slices through a
// 4-stage cp.async pipeline (global reads coalesced 128 B per row; A is stored
// k-major in shared memory with a row pitch = 2 (mod 8) x 16 B so fragment loads
// are bank-conflict free).
#include <algorithm>

#include "ops.h"

namespace qtnhb {

namespace {

constexpr int kBK = 8;
constexpr int kStages = 4;

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
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

template <int BM, int BN>
struct Smem {
  static constexpr int PA = BM + 2;  // 16-B elements; = 2 (mod 8)
  static constexpr int PB = BN + 2;
  static constexpr int A_ELEMS = kBK * PA;
  static constexpr int B_ELEMS = kBK * PB;
  static constexpr size_t bytes = static_cast<size_t>(kStages) * (A_ELEMS + B_ELEMS) * 16;
};

template <int BM, int BN>
__global__ void __launch_bounds__(256, 1) k_zgemm(const double2* __restrict__ A,
                                                  const double2* __restrict__ B,
                                                  double2* __restrict__ C, int64_t M, int64_t N,
                                                  int64_t K) {
  constexpr int WM = 32, WN = 32;
  constexpr int WARPS_N = BN / WN;
  static_assert((BM / WM) * (BN / WN) == 8, "8 warps");
  using S = Smem<BM, BN>;
  extern __shared__ __align__(16) double2 smem[];
  double2* As = smem;                          // [stage][k][PA]
  double2* Bs = smem + kStages * S::A_ELEMS;   // [stage][k][PB]

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / WARPS_N, wn = warp % WARPS_N;
  const int64_t bm = static_cast<int64_t>(blockIdx.y) * BM;
  const int64_t bn = static_cast<int64_t>(blockIdx.x) * BN;
  const int64_t n_kt = (K + kBK - 1) / kBK;

  auto load_stage = [&](int stage, int64_t kt) {
    int64_t k0 = kt * kBK;
    double2* as = As + stage * S::A_ELEMS;
    double2* bs = Bs + stage * S::B_ELEMS;
#pragma unroll
    for (int u = 0; u < (BM * kBK) / 256; ++u) {
      int e = tid + u * 256;
      int m = e / kBK, k = e % kBK;
      int64_t gm = bm + m, gk = k0 + k;
      bool ok = gm < M && gk < K;
      cp_async16(as + k * S::PA + m, ok ? (A + gm * K + gk) : A, ok);
    }
#pragma unroll
    for (int u = 0; u < (BN * kBK) / 256; ++u) {
      int e = tid + u * 256;
      int k = e / BN, n = e % BN;
      int64_t gk = k0 + k, gn = bn + n;
      bool ok = gk < K && gn < N;
      cp_async16(bs + k * S::PB + n, ok ? (B + gk * N + gn) : B, ok);
    }
  };

  double acc_re[4][4][2], acc_im[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      acc_re[i][j][0] = acc_re[i][j][1] = 0.0;
      acc_im[i][j][0] = acc_im[i][j][1] = 0.0;
    }

#pragma unroll
  for (int s = 0; s < kStages - 1; ++s) {
    if (s < n_kt) load_stage(s, s);
    cp_commit();
  }

  const int fr = lane >> 2, fk = lane & 3;
  for (int64_t kt = 0; kt < n_kt; ++kt) {
    cp_wait<kStages - 2>();
    __syncthreads();
    // Prefetch the slice kStages-1 ahead into the slot freed last iteration.
    {
      int64_t nk = kt + kStages - 1;
      if (nk < n_kt) load_stage(static_cast<int>(nk % kStages), nk);
      cp_commit();
    }
    const double2* as = As + (kt % kStages) * S::A_ELEMS;
    const double2* bs = Bs + (kt % kStages) * S::B_ELEMS;
#pragma unroll
    for (int k4 = 0; k4 < kBK; k4 += 4) {
      double a_re[4], a_im[4], b_re[4], b_im[4], nb_im[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        double2 v = as[(k4 + fk) * S::PA + wm * WM + i * 8 + fr];
        a_re[i] = v.x;
        a_im[i] = v.y;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        double2 v = bs[(k4 + fk) * S::PB + wn * WN + j * 8 + fr];
        b_re[j] = v.x;
        b_im[j] = v.y;
        nb_im[j] = -v.y;
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          dmma(acc_re[i][j], a_re[i], b_re[j]);
          dmma(acc_im[i][j], a_re[i], b_im[j]);
          dmma(acc_re[i][j], a_im[i], nb_im[j]);
          dmma(acc_im[i][j], a_im[i], b_re[j]);
        }
    }
  }
  cp_wait<0>();

  // Epilogue: lane holds C[fr][2*fk + {0,1}] of each 8x8 sub-tile.
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int64_t row = bm + wm * WM + i * 8 + fr;
    if (row >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int64_t col = bn + wn * WN + j * 8 + 2 * fk;
      double2* dst = C + row * N + col;
      if (col < N) dst[0] = make_double2(acc_re[i][j][0], acc_im[i][j][0]);
      if (col + 1 < N) dst[1] = make_double2(acc_re[i][j][1], acc_im[i][j][1]);
    }
  }
}

template <int BM, int BN>
void launch(const double2* a, const double2* b, double2* c, Dim m, Dim n, Dim k, cudaStream_t st) {
  size_t smem = Smem<BM, BN>::bytes;
  QTNH_CUDA(cudaFuncSetAttribute(k_zgemm<BM, BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 grid(static_cast<unsigned>((n + BN - 1) / BN), static_cast<unsigned>((m + BM - 1) / BM));
  if (grid.y > 65535u) {
    // Split along M into chunks the grid can address.
    Dim rows = static_cast<Dim>(65535) * BM;
    for (Dim m0 = 0; m0 < m; m0 += rows) {
      Dim mm = std::min(rows, m - m0);
      launch<BM, BN>(a + m0 * k, b, c + m0 * n, mm, n, k, st);
    }
    return;
  }
  k_zgemm<BM, BN><<<grid, 256, smem, st>>>(a, b, c, m, n, k);
  QTNH_LAUNCH_CHECK();
}

}  // namespace

void zgemm(const void* a, const void* b, void* c, Dim m, Dim n, Dim k, cudaStream_t st) {
  if (m <= 0 || n <= 0) return;
  auto A = static_cast<const double2*>(a);
  auto B = static_cast<const double2*>(b);
  auto Cp = static_cast<double2*>(c);
  if (k <= 0) {
    QTNH_CUDA(cudaMemsetAsync(c, 0, static_cast<size_t>(m * n) * 16, st));
    return;
  }
  if (n > 64) launch<64, 128>(A, B, Cp, m, n, k, st);
  else if (n > 32) launch<128, 64>(A, B, Cp, m, n, k, st);
  else launch<256, 32>(A, B, Cp, m, n, k, st);
}

}  // namespace qtnhb
