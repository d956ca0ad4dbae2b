// Orthonormal completion of null singular directions.
//
// The reference's psvd returns LAPACK's zgesdd bases (linalg.hpp:441-471): U and
// Vh are isometries whatever the rank of the input, so after truncate_svd
// (linalg.hpp:476-505) a kept triplet with sigma = 0 still has unit vectors.
// The Jacobi SVD recovers one side as X / sigma (and, without the accumulated
// transform, the other as A Vh^H / sigma): for a numerically null sigma both are
// zero or noise. This pass, run by the public SVD entry points (qtnh_svd,
// qtnh_svd_device), replaces them with an orthonormal completion:
//   r   = #{c < k : sigma_c > max(m, n) eps sigma_0}   (k = min(m, n, chi))
//   Y   = (I - U_r U_r^H)^2 Omega      (seeded normals, classical Gram-Schmidt twice)
//   U_c = left singular vectors of Y   (Jacobi, all sigma ~ 1: a few sweeps)
// and the same for the rows of Vh; absorbed sides get sigma^p times the
// completion, so U S Vh is unchanged up to the null sigmas themselves. Columns
// c >= min(m, n) (truncate_svd's zero padding) stay zero. The scan costs one
// tiny kernel and one 4-byte-per-matrix read; nothing else runs unless a null
// direction exists.
#include <algorithm>
#include <cmath>
#include <vector>

#include "ops.h"
#include "qtnh_b200.h"

namespace qtnhb {

namespace {

// per matrix: number of non-null kept singular values
__global__ void k_null_scan(const double* __restrict__ s, int64_t chi, int64_t k, double rel, int* __restrict__ rank) {
  const int64_t b = blockIdx.x;
  const double* S = s + b * chi;
  const double thr = rel * S[0];
  int cnt = 0;
  for (int64_t c = threadIdx.x; c < k; c += blockDim.x) cnt += S[c] > thr ? 1 : 0;
  __shared__ int red[256];
  red[threadIdx.x] = cnt;
  __syncthreads();
  for (int h = blockDim.x / 2; h > 0; h >>= 1) {
    if (threadIdx.x < h) red[threadIdx.x] += red[threadIdx.x + h];
    __syncthreads();
  }
  if (threadIdx.x == 0) rank[b] = red[0];
}

// dst (rows x r) = the first r columns of src (rows x ld), column c divided by f[c] (f > 0)
__global__ void k_unit_columns(const double2* __restrict__ src, int64_t ld, double2* __restrict__ dst, int64_t rows,
                               int64_t r, const double* __restrict__ f) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < rows * r; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / r, c = e % r;
    const double2 v = src[i * ld + c];
    const double g = 1.0 / f[c];
    dst[e] = make_double2(v.x * g, v.y * g);
  }
}

// y -= p
__global__ void k_sub(double2* __restrict__ y, const double2* __restrict__ p, int64_t count) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count; e += (int64_t)gridDim.x * blockDim.x)
    y[e] = make_double2(y[e].x - p[e].x, y[e].y - p[e].y);
}

// column r0 + j of dst (rows x ld) = f_j * q[:, j] (q: rows x z)
__global__ void k_put_columns(double2* __restrict__ dst, int64_t ld, int64_t r0, const double2* __restrict__ q,
                              int64_t rows, int64_t z, const double* __restrict__ f) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < rows * z; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / z, j = e % z;
    const double g = f[j];
    dst[i * ld + r0 + j] = make_double2(q[e].x * g, q[e].y * g);
  }
}

// row r0 + j of dst (? x cols) = f_j * conj(q[:, j])^T (q: cols x z)
__global__ void k_put_rows_conj(double2* __restrict__ dst, int64_t cols, int64_t r0, const double2* __restrict__ q,
                                int64_t z, const double* __restrict__ f) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < cols * z; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t x = e / z, j = e % z;
    const double g = f[j];
    dst[(r0 + j) * cols + x] = make_double2(q[e].x * g, -q[e].y * g);
  }
}

int grid_for(int64_t n) { return static_cast<int>(std::min<int64_t>((n + 255) / 256, 148 * 8)); }

double absorb_factor(double sv, bool u_side, int absorb) {
  if (absorb == QTNH_ABSORB_SPLIT) return std::sqrt(sv);
  if (u_side && absorb == QTNH_ABSORB_LEFT) return sv;
  if (!u_side && absorb == QTNH_ABSORB_RIGHT) return sv;
  return 1.0;
}

// Orthonormal completion of a d-dimensional basis of r vectors by z more,
// written from vector r on: the basis is given as unit columns b (d x r).
// Output: columns of u (ld chi) or conjugated rows of vh (row length d), each
// scaled by fz[j].
void complete_side(RankCtx& rk, const double2* b, int64_t d, int64_t r, int64_t z, const std::vector<double>& fz,
                   double2* out, int64_t ld_out, bool columns, uint64_t seed) {
  cudaStream_t st = rk.stream;
  DevBuf om(static_cast<size_t>(d * z) * 16, rk);
  qtnh_counter_complex_normals_device(st, seed, 0, d * z, om.ptr);
  auto* y = static_cast<double2*>(om.ptr);
  if (r > 0) {
    DevBuf bh(static_cast<size_t>(r * d) * 16, rk), t(static_cast<size_t>(r * z) * 16, rk),
        p(static_cast<size_t>(d * z) * 16, rk);
    conj_transpose(b, static_cast<double2*>(bh.ptr), d, r, st);
    for (int pass = 0; pass < 2; ++pass) {  // classical Gram-Schmidt, twice
      zgemm(bh.ptr, y, t.ptr, r, z, d, st);
      zgemm(b, t.ptr, p.ptr, d, z, r, st);
      k_sub<<<grid_for(d * z), 256, 0, st>>>(y, static_cast<const double2*>(p.ptr), d * z);
      QTNH_LAUNCH_CHECK();
    }
  }
  // orthonormal basis of range(Y): its left singular vectors (sigma ~ 1)
  DevBuf uy(static_cast<size_t>(d * z) * 16, rk), sy(static_cast<size_t>(z) * 8, rk),
      vy(static_cast<size_t>(z * z) * 16, rk), f(static_cast<size_t>(z) * 8, rk);
  void* up = uy.ptr;
  void* vp = vy.ptr;
  int sweeps = 0;
  svd_jacobi_ptrs(rk, 1, d, z, y, z, QTNH_ABSORB_NONE, &up, sy.ptr, &vp, &sweeps);
  QTNH_CUDA(cudaMemcpyAsync(f.ptr, fz.data(), z * 8, cudaMemcpyHostToDevice, st));
  if (columns)
    k_put_columns<<<grid_for(d * z), 256, 0, st>>>(out, ld_out, r, static_cast<const double2*>(uy.ptr), d, z,
                                                   static_cast<const double*>(f.ptr));
  else
    k_put_rows_conj<<<grid_for(d * z), 256, 0, st>>>(out, d, r, static_cast<const double2*>(uy.ptr), z,
                                                     static_cast<const double*>(f.ptr));
  QTNH_LAUNCH_CHECK();
  // the host factor vectors and the scratch die with this call: finish first
  QTNH_CUDA(cudaStreamSynchronize(st));
}

}  // namespace

void svd_complete_null(RankCtx& rk, Dim batch, Dim m, Dim n, Dim chi, int absorb, void* const* u_ptrs, const void* s,
                       void* const* vh_ptrs) {
  if (chi <= 0) chi = std::min(m, n);
  const Dim k = std::min(std::min(m, n), chi);
  if (batch < 1 || k < 1) return;
  cudaStream_t st = rk.stream;
  DevBuf rank_d(static_cast<size_t>(batch) * 4, rk);
  const double rel = static_cast<double>(std::max(m, n)) * 2.220446049250313e-16;
  k_null_scan<<<static_cast<unsigned>(batch), 256, 0, st>>>(static_cast<const double*>(s), chi, k, rel,
                                                            static_cast<int*>(rank_d.ptr));
  QTNH_LAUNCH_CHECK();
  std::vector<int> rank(batch);
  QTNH_CUDA(cudaMemcpyAsync(rank.data(), rank_d.ptr, batch * 4, cudaMemcpyDeviceToHost, st));
  QTNH_CUDA(cudaStreamSynchronize(st));
  if (std::all_of(rank.begin(), rank.end(), [&](int v) { return v >= k; })) return;
  std::vector<double> sh(static_cast<size_t>(batch * chi));
  QTNH_CUDA(cudaMemcpyAsync(sh.data(), s, sh.size() * 8, cudaMemcpyDeviceToHost, st));
  QTNH_CUDA(cudaStreamSynchronize(st));
  for (Dim b = 0; b < batch; ++b) {
    const Dim r = rank[b], z = k - r;
    if (z <= 0) continue;
    const double* S = sh.data() + b * chi;
    auto* U = static_cast<double2*>(u_ptrs[b]);
    auto* VH = static_cast<double2*>(vh_ptrs[b]);
    for (int side = 0; side < 2; ++side) {
      const bool u_side = side == 0;
      const Dim d = u_side ? m : n;
      std::vector<double> fb(r), fz(z);
      for (Dim c = 0; c < r; ++c) fb[c] = absorb_factor(S[c], u_side, absorb);
      for (Dim j = 0; j < z; ++j) fz[j] = absorb_factor(S[r + j], u_side, absorb);
      DevBuf unit(static_cast<size_t>(std::max<Dim>(d * r, 1)) * 16, rk), f(static_cast<size_t>(std::max<Dim>(r, 1)) * 8, rk);
      if (r > 0) {
        QTNH_CUDA(cudaMemcpyAsync(f.ptr, fb.data(), r * 8, cudaMemcpyHostToDevice, st));
        if (u_side) {
          k_unit_columns<<<grid_for(d * r), 256, 0, st>>>(U, chi, static_cast<double2*>(unit.ptr), d, r,
                                                          static_cast<const double*>(f.ptr));
        } else {
          // V_r = conj(Vh_r)^T (n x r), then unit columns in place
          conj_transpose(VH, static_cast<double2*>(unit.ptr), r, d, st);
          k_unit_columns<<<grid_for(d * r), 256, 0, st>>>(static_cast<double2*>(unit.ptr), r,
                                                          static_cast<double2*>(unit.ptr), d, r,
                                                          static_cast<const double*>(f.ptr));
        }
        QTNH_LAUNCH_CHECK();
      }
      complete_side(rk, static_cast<const double2*>(unit.ptr), d, r, z, fz, u_side ? U : VH, chi, u_side,
                    0x9E3779B97F4A7C15ULL ^ (static_cast<uint64_t>(b) * 2 + side));
    }
  }
}

}  // namespace qtnhb
