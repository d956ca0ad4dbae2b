// Seeded synthetic inputs (common.hpp:83-146 semantics).
//
// Host generators are bit-identical to the reference's Rng / hash_counter (glibc
// log/sin/cos in Box-Muller). The device generator reproduces the counter-based
// stream with CUDA's double-precision log/sincos (correct to ~1 ulp, not
// bit-identical to glibc); it exists for states too large to build on the host
// (2^33 amplitudes), whose parity is checked through size-independent properties.
#include <cmath>
#include <thread>
#include <vector>

#include "common.h"
#include "qtnh_b200.h"

namespace qtnhb {

namespace {

__host__ __device__ inline uint64_t mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

__host__ __device__ inline uint64_t hash4(uint64_t seed, uint64_t k0, uint64_t k1, uint64_t k2) {
  uint64_t h = mix64(seed ^ 0x243f6a8885a308d3ULL);
  h = mix64(h ^ k0);
  h = mix64(h ^ k1);
  return mix64(h ^ k2);
}

__host__ __device__ inline double unit(uint64_t u) { return static_cast<double>(u >> 11) * 0x1.0p-53; }

constexpr double kTwoPi = 6.283185307179586476925286766559;

void host_counter(uint64_t seed, int64_t start, int64_t count, double* out) {
  for (int64_t i = 0; i < count; ++i) {
    uint64_t j = static_cast<uint64_t>(start + i);
    double u1 = 0.0;
    for (uint64_t k2 = 0; u1 <= 1e-300; ++k2) u1 = unit(hash4(seed, j, 0, k2));
    double u2 = unit(hash4(seed, j, 1, 0));
    double r = std::sqrt(-2.0 * std::log(u1));
    double a = kTwoPi * u2;
    out[2 * i] = r * std::cos(a);
    out[2 * i + 1] = r * std::sin(a);
  }
}

__global__ void k_counter(double2* out, uint64_t seed, int64_t start, int64_t count) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t j = static_cast<uint64_t>(start + i);
    double u1 = 0.0;
    for (uint64_t k2 = 0; u1 <= 1e-300; ++k2) u1 = unit(hash4(seed, j, 0, k2));
    double u2 = unit(hash4(seed, j, 1, 0));
    double r = sqrt(-2.0 * log(u1));
    double s, c;
    sincos(kTwoPi * u2, &s, &c);
    out[i] = make_double2(r * c, r * s);
  }
}

}  // namespace
}  // namespace qtnhb

extern "C" {

uint64_t qtnh_hash_counter(uint64_t seed, uint64_t k0, uint64_t k1, uint64_t k2) {
  return qtnhb::hash4(seed, k0, k1, k2);
}

void qtnh_rng_complex_normals(uint64_t seed, int64_t count, double* out) {
  uint64_t state = qtnhb::mix64(seed);
  bool have = false;
  double spare = 0.0;
  for (int64_t i = 0; i < 2 * count; ++i) {
    if (have) {
      have = false;
      out[i] = spare;
      continue;
    }
    double u1 = 0.0;
    while (u1 <= 1e-300) {
      state = qtnhb::mix64(state);
      u1 = qtnhb::unit(state);
    }
    state = qtnhb::mix64(state);
    double u2 = qtnhb::unit(state);
    double r = std::sqrt(-2.0 * std::log(u1));
    double a = qtnhb::kTwoPi * u2;
    spare = r * std::sin(a);
    have = true;
    out[i] = r * std::cos(a);
  }
}

void qtnh_counter_complex_normals(uint64_t seed, int64_t start, int64_t count, double* out, int threads) {
  if (threads <= 1 || count < (1 << 16)) {
    qtnhb::host_counter(seed, start, count, out);
    return;
  }
  std::vector<std::thread> ts;
  int64_t chunk = (count + threads - 1) / threads;
  for (int t = 0; t < threads; ++t) {
    int64_t s = t * chunk, e = std::min<int64_t>(count, s + chunk);
    if (s >= e) break;
    ts.emplace_back([=] { qtnhb::host_counter(seed, start + s, e - s, out + 2 * s); });
  }
  for (auto& t : ts) t.join();
}

int qtnh_counter_complex_normals_device(void* stream, uint64_t seed, int64_t start, int64_t count, void* out) {
  if (count <= 0) return 0;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t g = std::min<int64_t>((count + 255) / 256, (int64_t)sms * 16);
  qtnhb::k_counter<<<static_cast<int>(g), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<double2*>(out), seed, start, count);
  qtnhb::note_launch();
  return cudaGetLastError() == cudaSuccess ? 0 : QTNH_E_RUNTIME;
}

}  // extern "C"
