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

// Header up to and including the dims; the payload count (or the pair list of the
// computed variants) follows.
std::string header_bytes(const TensorImpl& t) {
  const Shape& s = t.shape;
  const Dist& d = t.dist;
  std::string h("QTNHTEN1", 8);
  auto put = [&](const void* v, size_t n) { h.append(static_cast<const char*>(v), n); };
  uint32_t var = static_cast<uint32_t>(t.variant), rank = static_cast<uint32_t>(s.n_idx()),
           split = static_cast<uint32_t>(s.split);
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
  if (t.variant == kIdentity || t.variant == kSwap) {  // tensor.hpp:596-601
    uint64_t pairs = t.pair_in.size();
    put(&pairs, 8);
    for (size_t i = 0; i < t.pair_in.size(); ++i) {
      int64_t a = t.pair_in[i], b = t.pair_out[i];
      put(&a, 8);
      put(&b, 8);
    }
    return h;
  }
  uint64_t count = static_cast<uint64_t>(s.total_size());
  if (t.variant == kDiagonal) {
    count = static_cast<uint64_t>(diag_local_count(s));
    for (int i = 0; i < s.split / 2; ++i) count *= static_cast<uint64_t>(s.dims[i]);
  }
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

// n complex elements from device memory into the file at byte offset base, through
// two pinned chunks (the D2H of one overlaps the pwrite of the other).
void write_device_block(int fd, const void* dev, Dim n, off_t base, cudaStream_t st) {
  if (n <= 0) return;
  const Dim ch = std::min(n, kChunk);
  Pinned host(static_cast<size_t>(2 * ch) * 16);
  cudaEvent_t ev[2];
  for (auto& e : ev) QTNH_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  const Dim nch = (n + ch - 1) / ch;
  auto issue = [&](Dim c) {
    const int s = static_cast<int>(c & 1);
    const Dim k = std::min(ch, n - c * ch);
    QTNH_CUDA(cudaMemcpyAsync(static_cast<char*>(host.p) + s * ch * 16, static_cast<const char*>(dev) + c * ch * 16,
                              k * 16, cudaMemcpyDeviceToHost, st));
    QTNH_CUDA(cudaEventRecord(ev[s], st));
  };
  auto drain = [&](Dim c) {
    const int s = static_cast<int>(c & 1);
    const Dim k = std::min(ch, n - c * ch);
    QTNH_CUDA(cudaEventSynchronize(ev[s]));
    full_pwrite(fd, static_cast<const char*>(host.p) + s * ch * 16, k * 16, base + c * ch * 16);
  };
  try {
    for (Dim c = 0; c < nch; ++c) {
      issue(c);
      if (c > 0) drain(c - 1);
    }
    drain(nch - 1);
  } catch (...) {
    cudaStreamSynchronize(st);
    for (auto& e : ev) cudaEventDestroy(e);
    throw;
  }
  for (auto& e : ev) cudaEventDestroy(e);
}

// The reverse: n complex elements of the file at base into device memory.
void read_device_block(int fd, void* dev, Dim n, off_t base, cudaStream_t st) {
  if (n <= 0) return;
  const Dim ch = std::min(n, kChunk);
  Pinned host(static_cast<size_t>(2 * ch) * 16);
  cudaEvent_t ev[2];
  for (auto& e : ev) QTNH_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  const Dim nch = (n + ch - 1) / ch;
  try {
    for (Dim c = 0; c < nch; ++c) {
      const int sl = static_cast<int>(c & 1);
      const Dim k = std::min(ch, n - c * ch);
      if (c >= 2) QTNH_CUDA(cudaEventSynchronize(ev[sl]));  // the H2D that used this slot is done
      char* hp = static_cast<char*>(host.p) + sl * ch * 16;
      full_pread(fd, hp, k * 16, base + c * ch * 16);
      QTNH_CUDA(cudaMemcpyAsync(static_cast<char*>(dev) + c * ch * 16, hp, k * 16, cudaMemcpyHostToDevice, st));
      QTNH_CUDA(cudaEventRecord(ev[sl], st));
    }
    QTNH_CUDA(cudaStreamSynchronize(st));  // pinned staging dies here
  } catch (...) {
    cudaStreamSynchronize(st);
    for (auto& e : ev) cudaEventDestroy(e);
    throw;
  }
  for (auto& e : ev) cudaEventDestroy(e);
}

}  // namespace

// Every variant in the reference's byte layout (tensor.hpp:373-380, :586-608): dense
// and symmetric store the global vector, a diagonal tensor its diagonal in row-major
// order of the input coordinates (each canonical on-diagonal holder writes its
// slice), identity and swap the pair list only.
void op_save(const TensorImpl& t, const std::string& path) {
  RankCtx& r = *t.rank;
  if (!t.in_span) return;
  auto members = span_ranks(t);
  const std::string hdr = header_bytes(t);
  const bool computed = t.variant == kIdentity || t.variant == kSwap;
  Dim mine = 0, at = 0, total = 0;  // this holder's element count, its element offset, the payload size
  if (t.variant == kDiagonal) {
    mine = diag_local_count(t.shape);
    total = mine;
    for (int i = 0; i < t.shape.split / 2; ++i) total *= t.shape.dims[i];
    Dim b_in = 0;
    if (diag_block_on_diagonal(t.shape, t.block, &b_in)) at = b_in * mine;
    else mine = 0;
  } else if (!computed) {
    mine = t.shape.local_size();
    total = t.shape.total_size();
    at = t.block * mine;
  }
  if (r.rank == t.dist.offset) {
    Fd f;
    f.fd = ::open(path.c_str(), O_WRONLY | O_CREAT | O_TRUNC, 0644);
    if (f.fd < 0) throw Status(QTNH_E_RUNTIME, "cannot open " + path + " for writing");
    full_pwrite(f.fd, hdr.data(), hdr.size(), 0);
    if (::ftruncate(f.fd, static_cast<off_t>(hdr.size() + total * 16)) != 0)
      throw Status(QTNH_E_RUNTIME, "cannot size " + path);
  }
  barrier(r, members);  // the file exists at its final size
  if (t.canonical() && mine > 0 && t.data()) {
    Fd f;
    f.fd = ::open(path.c_str(), O_WRONLY);
    if (f.fd < 0) throw Status(QTNH_E_RUNTIME, "cannot open " + path + " for writing");
    write_device_block(f.fd, t.data(), mine, static_cast<off_t>(hdr.size() + at * 16), r.stream);
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
  if (var > kSwap || rank > 64) throw Status(QTNH_E_RUNTIME, "corrupt tensor stream");
  const size_t dims_at = sizeof(fixed), count_at = dims_at + 8 * rank, data_at = count_at + 8;
  if (fsize < data_at) throw Status(QTNH_E_RUNTIME, "truncated tensor stream");
  std::vector<int64_t> dims(rank);
  if (rank) full_pread(f.fd, reinterpret_cast<char*>(dims.data()), 8 * rank, static_cast<off_t>(dims_at));
  uint64_t count = 0;  // payload elements, or pairs for the computed variants
  full_pread(f.fd, reinterpret_cast<char*>(&count), 8, static_cast<off_t>(count_at));
  Shape s(std::vector<Dim>(dims.begin(), dims.end()), static_cast<int>(split));
  Dist d;
  d.stretch = st;
  d.cycles = cy;
  d.offset = off;
  if (var == kIdentity || var == kSwap) {  // tensor.hpp:420-430
    if (count > 64 || fsize < data_at + count * 16) throw Status(QTNH_E_RUNTIME, "truncated tensor stream");
    std::vector<int64_t> pairs(2 * count);
    if (count) full_pread(f.fd, reinterpret_cast<char*>(pairs.data()), 16 * count, static_cast<off_t>(data_at));
    std::vector<int> in_pos(count), out_pos(count);
    for (uint64_t i = 0; i < count; ++i) {
      in_pos[i] = static_cast<int>(pairs[2 * i]);
      out_pos[i] = static_cast<int>(pairs[2 * i + 1]);
    }
    return make_paired(r, s, d, in_pos, out_pos, var == kSwap);
  }
  if (fsize < data_at + count * 16) throw Status(QTNH_E_RUNTIME, "truncated tensor stream");
  if (var == kDiagonal) {
    TP t = make_diagonal(r, s, d, nullptr, static_cast<Dim>(count));
    Dim b_in = 0;
    if (t->buf && diag_block_on_diagonal(t->shape, t->block, &b_in)) {
      const Dim n = diag_local_count(t->shape);
      read_device_block(f.fd, t->data(), n, static_cast<off_t>(data_at + b_in * n * 16), r.stream);
    }
    return t;
  }
  if (var == kSymmetric) check_symmetric_shape(s);
  TP t = make_tensor(r, s, d, true);
  t->variant = static_cast<int>(var);
  if (count != static_cast<uint64_t>(t->shape.total_size())) throw_invalid("global element count mismatch");
  if (!t->in_span) return t;
  const Dim nl = t->shape.local_size();
  read_device_block(f.fd, t->data(), nl, static_cast<off_t>(data_at + t->block * nl * 16), r.stream);
  return t;
}

}  // namespace qtnhb
