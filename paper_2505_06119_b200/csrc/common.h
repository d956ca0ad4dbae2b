// Shared infrastructure of libqtnh_b200: error classes, CUDA checks, layout
// metadata of the sharded (distributed-index) tensor layout.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "qtnh_b200.h"

namespace qtnhb {

// NVTX range over one library operation (nsys / ncu --nvtx show them nested in
// the caller's ranges). Header-only NVTX v3: without an attached tool the push /
// pop are a function-pointer check.
struct NvtxRange {
  explicit NvtxRange(const char* n) { nvtxRangePushA(n); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
#define QTNH_CAT2_(a, b) a##b
#define QTNH_CAT_(a, b) QTNH_CAT2_(a, b)
#define QTNH_RANGE(name) ::qtnhb::NvtxRange QTNH_CAT_(qtnh_nvtx_, __LINE__)(name)

using Dim = int64_t;

// One exception type carrying the qtnh error class (common.hpp:31-74); the C
// ABI turns it into a QTNH_E_* status plus thread-local message/info.
struct Status : std::runtime_error {
  int code;
  int64_t info;
  Status(int c, const std::string& msg, int64_t inf = 0)
      : std::runtime_error(msg), code(c), info(inf) {}
};

[[noreturn]] inline void throw_invalid(const std::string& m) { throw Status(QTNH_E_INVALID_ARGUMENT, m); }
[[noreturn]] inline void throw_resource(const std::string& m, int64_t required) {
  throw Status(QTNH_E_RESOURCE, m + " (requires " + std::to_string(required) + " ranks)", required);
}
[[noreturn]] inline void throw_runtime(const std::string& m) { throw Status(QTNH_E_RUNTIME, m); }

#define QTNH_CUDA(x)                                                                     \
  do {                                                                                   \
    cudaError_t e_ = (x);                                                                \
    if (e_ != cudaSuccess)                                                               \
      ::qtnhb::throw_runtime(std::string("CUDA error ") + cudaGetErrorString(e_) + " at " + \
                             __FILE__ + ":" + std::to_string(__LINE__));                  \
  } while (0)

// Count of kernels this library launched (evidence for bench.py's gpu_launches).
extern std::atomic<int64_t> g_kernel_launches;
inline void note_launch(int64_t n = 1) { g_kernel_launches.fetch_add(n, std::memory_order_relaxed); }
#define QTNH_LAUNCH_CHECK()                        \
  do {                                             \
    ::qtnhb::note_launch();                        \
    QTNH_CUDA(cudaGetLastError());                 \
  } while (0)

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device, size):
// a driver call per launch cost ~1-2 us of host time on every small contraction.
void ensure_max_dynamic_smem(const void* kernel, int bytes);

// ---- sharded layout metadata (indexing.hpp:32-191 semantics) -----------------
// dims with the first `split` indices distributed (they select the rank block,
// row-major) and the rest local (row-major inside the rank's block).
struct Shape {
  std::vector<Dim> dims;
  int split = 0;

  Shape() = default;
  Shape(std::vector<Dim> d, int s) : dims(std::move(d)), split(s) { validate(); }
  void validate() const {
    if (split < 0 || split > n_idx())
      throw_invalid("index split " + std::to_string(split) + " outside [0, " +
                    std::to_string(n_idx()) + "]");
    for (Dim d : dims)
      if (d < 1) throw_invalid("index dimensions must be positive");
  }
  int n_idx() const { return static_cast<int>(dims.size()); }
  int n_local() const { return n_idx() - split; }
  Dim dist_size() const {
    Dim n = 1;
    for (int i = 0; i < split; ++i) n *= dims[i];
    return n;
  }
  Dim local_size() const {
    Dim n = 1;
    for (int i = split; i < n_idx(); ++i) n *= dims[i];
    return n;
  }
  Dim total_size() const { return dist_size() * local_size(); }
  std::vector<Dim> dist_dims() const { return {dims.begin(), dims.begin() + split}; }
  std::vector<Dim> local_dims() const { return {dims.begin() + split, dims.end()}; }
};

// Broadcast pattern: a span of stretch*cycles*N_d consecutive ranks from
// `offset`, cycles outermost, blocks next, stretch innermost (indexing.hpp:84-101).
struct Dist {
  Dim stretch = 1, cycles = 1, offset = 0;
  void validate() const {
    if (stretch < 1 || cycles < 1 || offset < 0)
      throw_invalid("invalid broadcast parameters (str=" + std::to_string(stretch) +
                    ", cyc=" + std::to_string(cycles) + ", off=" + std::to_string(offset) + ")");
  }
  Dim span(Dim nd) const { return stretch * cycles * nd; }
  bool operator==(const Dist& o) const {
    return stretch == o.stretch && cycles == o.cycles && offset == o.offset;
  }
  // Rank of copy (cycle c, slot t) of block b (indexing.hpp:153-154).
  int home(Dim b, Dim nd, Dim c, Dim t) const {
    return static_cast<int>(offset + c * stretch * nd + b * stretch + t);
  }
  int canonical(Dim b) const { return static_cast<int>(offset + b * stretch); }
  std::vector<int> homes(Dim b, Dim nd) const {
    std::vector<int> r;
    for (Dim c = 0; c < cycles; ++c)
      for (Dim t = 0; t < stretch; ++t) r.push_back(home(b, nd, c, t));
    return r;
  }
  // Block/cycle/slot held by `rank`, false outside the span (indexing.hpp:181-191).
  bool locate(int rank, Dim nd, Dim* block, Dim* cycle, Dim* slot) const {
    Dim r = rank - offset;
    if (r < 0 || r >= span(nd)) return false;
    Dim per = stretch * nd;
    *cycle = r / per;
    *block = (r % per) / stretch;
    *slot = r % stretch;
    return true;
  }
};

inline Dist dist_from(const int64_t* d) {
  Dist p;
  if (d) {
    p.stretch = d[0];
    p.cycles = d[1];
    p.offset = d[2];
  }
  return p;
}

inline std::vector<Dim> row_major_strides(const std::vector<Dim>& dims) {
  std::vector<Dim> s(dims.size(), 1);
  for (int i = static_cast<int>(dims.size()) - 2; i >= 0; --i) s[i] = s[i + 1] * dims[i + 1];
  return s;
}

inline std::vector<Dim> unflat(Dim off, const std::vector<Dim>& dims) {
  std::vector<Dim> c(dims.size(), 0);
  for (int i = static_cast<int>(dims.size()) - 1; i >= 0; --i) {
    c[i] = off % dims[i];
    off /= dims[i];
  }
  return c;
}

inline Dim flat(const std::vector<Dim>& c, const std::vector<Dim>& dims) {
  Dim off = 0;
  for (size_t i = 0; i < dims.size(); ++i) off = off * dims[i] + c[i];
  return off;
}

}  // namespace qtnhb
