// One brickwork layer of MPS two-site updates (config 4), entirely on the device.
//
// Reference composition (SPEC apply_raw_gate, SPEC.md:371-379 / :475-483, built
// from linalg.hpp): theta = contract(site_q, site_q+1) via t2m -> pgemm -> m2t
// (linalg.hpp:208-400); the 2-qubit gate as a second contraction + permute back;
// psvd = gather to the root + LAPACKE_zgesdd (linalg.hpp:441-471); truncate_svd
// to chi with zero padding (:476-505); absorb_singular_left (:508-514); the
// kept weight sum(s_kept^2) / ||theta||^2 for the truncation fidelity
// (SPEC.md:725-729).
//
// Here, per group of pairs whose thetas have equal shape:
//   * each theta is ONE zgemm straight into its slot of the SVD batch buffer
//     (site_q is (l d) x c row-major, site_q+1 is c x (d r): no permutation);
//   * the gate runs in place over the whole batch (one launch);
//   * ||theta||^2 per matrix by a fixed-order two-pass reduction (deterministic);
//   * the batched Jacobi SVD writes U S and Vh straight into the new site tensors
//     (per-matrix output pointers);
//   * the only host synchronisation is the download of the kept singular values
//     and norms, once per group;
//   * the largest group (the saturated thetas) runs on the rank's stream, the other
//     shapes concurrently on a side stream from a second host thread.
#include <algorithm>
#include <map>
#include <tuple>

#include <exception>
#include <thread>

#include "ops.h"

namespace qtnhb {

namespace {

constexpr int kFroParts = 256;

__global__ void k_fro2_partial(const double2* __restrict__ a, int64_t count, double* __restrict__ part) {
  const int64_t mat = blockIdx.y;
  const double2* A = a + mat * count;
  __shared__ double red[256];
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    s += A[i].x * A[i].x + A[i].y * A[i].y;
  red[threadIdx.x] = s;
  __syncthreads();
  for (int k = blockDim.x / 2; k > 0; k >>= 1) {
    if (threadIdx.x < k) red[threadIdx.x] += red[threadIdx.x + k];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[mat * gridDim.x + blockIdx.x] = red[0];
}

__global__ void k_fro2_final(const double* __restrict__ part, int parts, double* __restrict__ out) {
  const int mat = blockIdx.x;
  __shared__ double red[256];
  double s = 0.0;
  for (int i = threadIdx.x; i < parts; i += blockDim.x) s += part[mat * parts + i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int k = blockDim.x / 2; k > 0; k >>= 1) {
    if (threadIdx.x < k) red[threadIdx.x] += red[threadIdx.x + k];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[mat] = red[0];
}

}  // namespace

void mps_apply_layer(const std::vector<TP>& left, const std::vector<TP>& right, const double* gate, Dim chi,
                     std::vector<TP>& new_left, std::vector<TP>& new_right, double* s_out, int64_t* keep_out,
                     double* norm2_out) {
  QTNH_RANGE("qtnh::mps_layer");
  const size_t np = left.size();
  if (right.size() != np) throw_invalid("mps layer: left and right site lists differ in length");
  if (chi < 1) throw_invalid("mps layer: chi must be >= 1");
  new_left.assign(np, nullptr);
  new_right.assign(np, nullptr);
  if (np == 0) return;
  RankCtx& r = *left[0]->rank;
  using Key = std::tuple<Dim, Dim, Dim, Dim>;  // theta (l, d1, d2, r)
  std::map<Key, std::vector<size_t>> groups;
  for (size_t i = 0; i < np; ++i) {
    const TP& a = left[i];
    const TP& b = right[i];
    if (!a || !b) throw_invalid("mps layer: null site");
    if (a->rank != &r || b->rank != &r) throw_invalid("mps layer: sites belong to different ranks");
    if (a->shape.n_idx() != 3 || b->shape.n_idx() != 3) throw_invalid("mps layer: sites must be rank-3 (l, d, r)");
    if (a->shape.split || b->shape.split) throw_invalid("mps layer: sites must have no distributed indices");
    if (!a->in_span || !b->in_span) throw_invalid("mps layer: this rank holds no copy of a site");
    if (a->shape.dims[2] != b->shape.dims[0]) throw_invalid("mps layer: bond dimensions of a pair differ");
    groups[Key{a->shape.dims[0], a->shape.dims[1], b->shape.dims[1], b->shape.dims[2]}].push_back(i);
  }
  // Output sites first, on the caller's stream: the groups below may run on a second
  // stream from a second host thread.
  for (auto& [key, idx] : groups) {
    const auto [l, d1, d2, rr] = key;
    const Dim keep = std::min(chi, std::min(l * d1, d2 * rr));
    for (size_t i : idx) {
      new_left[i] = make_tensor(r, Shape({l, d1, keep}, 0), left[i]->dist, true);
      new_right[i] = make_tensor(r, Shape({keep, d2, rr}, 0), right[i]->dist, true);
    }
  }
  auto run_group = [&](RankCtx& rc, const Key& key, const std::vector<size_t>& idx) {
    const auto [l, d1, d2, rr] = key;
    const Dim bsz = static_cast<Dim>(idx.size());
    const Dim m = l * d1, n = d2 * rr, k = std::min(m, n), keep = std::min(chi, k);
    DevBuf theta(static_cast<size_t>(bsz * m * n) * 16, rc);
    double2* th = static_cast<double2*>(theta.ptr);
    for (Dim j = 0; j < bsz; ++j) {
      const TP& a = left[idx[j]];
      const TP& b = right[idx[j]];
      zgemm(a->data(), b->data(), th + j * m * n, m, n, a->shape.dims[2], rc.stream);
    }
    gate_local(th, {bsz * l, d1, d2, rr}, {1, 2}, gate, false, rc.stream);
    DevBuf part(static_cast<size_t>(bsz) * kFroParts * sizeof(double), rc);
    DevBuf nrm(static_cast<size_t>(bsz) * sizeof(double), rc);
    k_fro2_partial<<<dim3(kFroParts, static_cast<unsigned>(bsz)), 256, 0, rc.stream>>>(th, m * n,
                                                                                     static_cast<double*>(part.ptr));
    QTNH_LAUNCH_CHECK();
    k_fro2_final<<<static_cast<unsigned>(bsz), 256, 0, rc.stream>>>(static_cast<const double*>(part.ptr), kFroParts,
                                                                   static_cast<double*>(nrm.ptr));
    QTNH_LAUNCH_CHECK();
    std::vector<void*> up(bsz), vp(bsz);
    for (Dim j = 0; j < bsz; ++j) {
      const size_t i = idx[j];
      up[j] = new_left[i]->data();
      vp[j] = new_right[i]->data();
    }
    DevBuf s(static_cast<size_t>(bsz * keep) * sizeof(double), rc);
    int sweeps = 0;
    svd_batched_ptrs(rc, bsz, m, n, th, keep, QTNH_ABSORB_LEFT, up.data(), s.ptr, vp.data(), &sweeps);
    std::vector<double> sh(bsz * keep), nh(bsz);
    QTNH_CUDA(cudaMemcpyAsync(sh.data(), s.ptr, sh.size() * sizeof(double), cudaMemcpyDeviceToHost, rc.stream));
    QTNH_CUDA(cudaMemcpyAsync(nh.data(), nrm.ptr, nh.size() * sizeof(double), cudaMemcpyDeviceToHost, rc.stream));
    QTNH_CUDA(cudaStreamSynchronize(rc.stream));
    for (Dim j = 0; j < bsz; ++j) {
      const size_t i = idx[j];
      if (s_out) {
        std::fill(s_out + i * chi, s_out + (i + 1) * chi, 0.0);
        std::copy(sh.begin() + j * keep, sh.begin() + (j + 1) * keep, s_out + i * chi);
      }
      if (keep_out) keep_out[i] = keep;
      if (norm2_out) norm2_out[i] = nh[j];
    }
  };
  // The largest group (the saturated thetas: one batched SVD) runs here; the other
  // shapes (the unsaturated pairs towards the chain's ends: single-matrix, latency-
  // bound SVDs, ~20 % of a late config-4 layer when run one after the other) run
  // concurrently on a side stream from a second host thread -- the pairs of a layer
  // are disjoint, so the results do not depend on the interleaving
  // (QTNH_MPS_OVERLAP=0: one after the other).
  static const bool overlap = [] {
    const char* e = std::getenv("QTNH_MPS_OVERLAP");
    return !(e && e[0] == '0');
  }();
  const Key* big = nullptr;
  double big_work = -1.0;
  for (auto& [key, idx] : groups) {
    const auto [l, d1, d2, rr] = key;
    const double w = static_cast<double>(idx.size()) * double(l * d1) * double(d2 * rr) * double(std::min(l * d1, d2 * rr));
    if (w > big_work) {
      big_work = w;
      big = &key;
    }
  }
  if (!overlap || groups.size() < 2 || big_work < 1e9) {
    for (auto& [key, idx] : groups) run_group(r, key, idx);
    return;
  }
  RankCtx side;  // same rank and device, its own launch stream; owns nothing
  side.world = r.world;
  side.rank = r.rank;
  side.device = r.device;
  side.stream = r.side_stream(0);
  cudaEvent_t ev = nullptr;
  QTNH_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  QTNH_CUDA(cudaEventRecord(ev, r.stream));
  QTNH_CUDA(cudaStreamWaitEvent(side.stream, ev, 0));
  std::exception_ptr side_err;
  std::thread worker([&] {
    try {
      side.activate();
      for (auto& [key, idx] : groups)
        if (&key != big) run_group(side, key, idx);
    } catch (...) {
      side_err = std::current_exception();
    }
  });
  std::exception_ptr main_err;
  try {
    run_group(r, *big, groups.at(*big));
  } catch (...) {
    main_err = std::current_exception();
  }
  worker.join();
  cudaEventRecord(ev, side.stream);
  cudaStreamWaitEvent(r.stream, ev, 0);
  cudaEventDestroy(ev);
  side.stream = nullptr;
  if (main_err) std::rethrow_exception(main_err);
  if (side_err) std::rethrow_exception(side_err);
}

}  // namespace qtnhb
