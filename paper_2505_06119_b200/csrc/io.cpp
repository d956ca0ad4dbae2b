// QTNHTEN1 serialization straight from / into HBM (tensor.hpp:373-446).
//
// The reference gathers the whole tensor onto its first span rank and streams it
// out element by element (save), and every rank parses the whole file into a host
// vector before from_global (load). The payload is the global row-major vector,
// i.e. the blocks concatenated in block order (tensor.hpp:341-371), so here every
// canonical holder writes ITS block at its byte offset (pwrite) and every span rank
// reads only its own block (pread): no gather, no global host copy, the files are
// byte-identical. Blocks move through two pinned staging chunks so the D2H/H2D
// copy of one chunk overlaps the file I/O of the other. Values are raw (signed
// zeros kept), as the reference's dense visit (tensor.hpp:300-311) writes them.
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cstring>

#include "ops.h"

namespace qtnhb {

namespace {

constexpr Dim kChunk = Dim(1) << 20;  // 16 MiB of complex128 per staging chunk

struct Fd {
  int fd = -1;
  ~Fd() {
    if (fd >= 0) ::close(fd);
  }
};

struct Pinned {
  void* p = nullptr;
  explicit Pinned(size_t b) { QTNH_CUDA(cudaHostAlloc(&p, b, cudaHostAllocDefault)); }
  ~Pinned() {
    if (p) cudaFreeHost(p);
  }
};

std::string header_bytes(const Shape& s, const Dist& d) {
  std::string h("QTNHTEN1", 8);
  auto put = [&](const void* v, size_t n) { h.append(static_cast<const char*>(v), n); };
  uint32_t var = 0, rank = static_cast<uint32_t>(s.n_idx()), split = static_cast<uint32_t>(s.split);
  put(&var, 4);
  put(&rank, 4);
  put(&split, 4);
  int64_t st = d.stretch, cy = d.cycles, off = d.offset;
  put(&st, 8);
  put(&cy, 8);
  put(&off, 8);
  for (Dim x : s.dims) {
    int64_t v = x;
    put(&v, 8);
  }
  uint64_t count = static_cast<uint64_t>(s.total_size());
  put(&count, 8);
  return h;
}

void full_pwrite(int fd, const char* p, size_t n, off_t off) {
  while (n) {
    ssize_t w = ::pwrite(fd, p, n, off);
    if (w <= 0) throw Status(QTNH_E_RUNTIME, std::string("write failed: ") + std::strerror(errno));
    p += w;
    n -= static_cast<size_t>(w);
    off += w;
  }
}

void full_pread(int fd, char* p, size_t n, off_t off) {
  while (n) {
    ssize_t g = ::pread(fd, p, n, off);
    if (g < 0) throw Status(QTNH_E_RUNTIME, std::string("read failed: ") + std::strerror(errno));
    if (g == 0) throw Status(QTNH_E_RUNTIME, "truncated tensor stream");
    p += g;
    n -= static_cast<size_t>(g);
    off += g;
  }
}

}  // namespace

void op_save(const TensorImpl& t, const std::string& path) {
  RankCtx& r = *t.rank;
  if (!t.in_span) return;
  auto members = span_ranks(t);
  const std::string hdr = header_bytes(t.shape, t.dist);
  const Dim nl = t.shape.local_size(), total = t.shape.total_size();
  if (r.rank == t.dist.offset) {
    Fd f;
    f.fd = ::open(path.c_str(), O_WRONLY | O_CREAT | O_TRUNC, 0644);
    if (f.fd < 0) throw Status(QTNH_E_RUNTIME, "cannot open " + path + " for writing");
    full_pwrite(f.fd, hdr.data(), hdr.size(), 0);
    if (::ftruncate(f.fd, static_cast<off_t>(hdr.size() + total * 16)) != 0)
      throw Status(QTNH_E_RUNTIME, "cannot size " + path);
  }
  barrier(r, members);  // the file exists at its final size
  if (t.canonical() && nl > 0) {
    Fd f;
    f.fd = ::open(path.c_str(), O_WRONLY);
    if (f.fd < 0) throw Status(QTNH_E_RUNTIME, "cannot open " + path + " for writing");
    const Dim ch = std::min(nl, kChunk);
    Pinned host(static_cast<size_t>(2 * ch) * 16);
    cudaEvent_t ev[2];
    for (auto& e : ev) QTNH_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    const off_t base = static_cast<off_t>(hdr.size() + t.block * nl * 16);
    const Dim nch = (nl + ch - 1) / ch;
    auto issue = [&](Dim c) {
      const int s = static_cast<int>(c & 1);
      const Dim n = std::min(ch, nl - c * ch);
      QTNH_CUDA(cudaMemcpyAsync(static_cast<char*>(host.p) + s * ch * 16,
                                static_cast<const char*>(t.data()) + c * ch * 16, n * 16, cudaMemcpyDeviceToHost,
                                r.stream));
      QTNH_CUDA(cudaEventRecord(ev[s], r.stream));
    };
    auto drain = [&](Dim c) {
      const int s = static_cast<int>(c & 1);
      const Dim n = std::min(ch, nl - c * ch);
      QTNH_CUDA(cudaEventSynchronize(ev[s]));
      full_pwrite(f.fd, static_cast<const char*>(host.p) + s * ch * 16, n * 16, base + c * ch * 16);
    };
    try {
      for (Dim c = 0; c < nch; ++c) {
        issue(c);
        if (c > 0) drain(c - 1);
      }
      drain(nch - 1);
    } catch (...) {
      cudaStreamSynchronize(r.stream);
      for (auto& e : ev) cudaEventDestroy(e);
      throw;
    }
    for (auto& e : ev) cudaEventDestroy(e);
  }
  barrier(r, members);
}

TP op_load(RankCtx& r, const std::string& path) {
  Fd f;
  f.fd = ::open(path.c_str(), O_RDONLY);
  if (f.fd < 0) throw Status(QTNH_E_RUNTIME, "cannot open " + path);
  struct stat sb {};
  if (::fstat(f.fd, &sb) != 0) throw Status(QTNH_E_RUNTIME, "cannot stat " + path);
  const size_t fsize = static_cast<size_t>(sb.st_size);
  char fixed[8 + 12 + 24];
  if (fsize < 8) throw Status(QTNH_E_RUNTIME, "not a qtnh tensor stream");
  full_pread(f.fd, fixed, std::min(sizeof(fixed), fsize), 0);
  if (std::memcmp(fixed, "QTNHTEN1", 8) != 0) throw Status(QTNH_E_RUNTIME, "not a qtnh tensor stream");
  if (fsize < sizeof(fixed)) throw Status(QTNH_E_RUNTIME, "truncated tensor stream");
  uint32_t var, rank, split;
  int64_t st, cy, off;
  std::memcpy(&var, fixed + 8, 4);
  std::memcpy(&rank, fixed + 12, 4);
  std::memcpy(&split, fixed + 16, 4);
  std::memcpy(&st, fixed + 20, 8);
  std::memcpy(&cy, fixed + 28, 8);
  std::memcpy(&off, fixed + 36, 8);
  if (var > 1) throw_invalid("variant " + std::to_string(var) + " is materialised by the host loader");
  if (rank > 64) throw Status(QTNH_E_RUNTIME, "corrupt tensor stream");
  const size_t dims_at = sizeof(fixed), count_at = dims_at + 8 * rank, data_at = count_at + 8;
  if (fsize < data_at) throw Status(QTNH_E_RUNTIME, "truncated tensor stream");
  std::vector<int64_t> dims(rank);
  if (rank) full_pread(f.fd, reinterpret_cast<char*>(dims.data()), 8 * rank, static_cast<off_t>(dims_at));
  uint64_t count = 0;
  full_pread(f.fd, reinterpret_cast<char*>(&count), 8, static_cast<off_t>(count_at));
  Shape s(std::vector<Dim>(dims.begin(), dims.end()), static_cast<int>(split));
  Dist d;
  d.stretch = st;
  d.cycles = cy;
  d.offset = off;
  TP t = make_tensor(r, s, d, true);
  if (count != static_cast<uint64_t>(t->shape.total_size())) throw Status(QTNH_E_RUNTIME, "corrupt tensor stream");
  if (fsize < data_at + count * 16) throw Status(QTNH_E_RUNTIME, "truncated tensor stream");
  if (!t->in_span) return t;
  const Dim nl = t->shape.local_size();
  if (nl == 0) return t;
  const Dim ch = std::min(nl, kChunk);
  Pinned host(static_cast<size_t>(2 * ch) * 16);
  cudaEvent_t ev[2];
  for (auto& e : ev) QTNH_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  const off_t base = static_cast<off_t>(data_at + t->block * nl * 16);
  const Dim nch = (nl + ch - 1) / ch;
  try {
    for (Dim c = 0; c < nch; ++c) {
      const int sl = static_cast<int>(c & 1);
      const Dim n = std::min(ch, nl - c * ch);
      if (c >= 2) QTNH_CUDA(cudaEventSynchronize(ev[sl]));  // the H2D that used this slot is done
      char* hp = static_cast<char*>(host.p) + sl * ch * 16;
      full_pread(f.fd, hp, n * 16, base + c * ch * 16);
      QTNH_CUDA(cudaMemcpyAsync(static_cast<char*>(t->data()) + c * ch * 16, hp, n * 16, cudaMemcpyHostToDevice,
                                r.stream));
      QTNH_CUDA(cudaEventRecord(ev[sl], r.stream));
    }
    QTNH_CUDA(cudaStreamSynchronize(r.stream));  // pinned staging dies here
  } catch (...) {
    cudaStreamSynchronize(r.stream);
    for (auto& e : ev) cudaEventDestroy(e);
    throw;
  }
  for (auto& e : ev) cudaEventDestroy(e);
  return t;
}

}  // namespace qtnhb
