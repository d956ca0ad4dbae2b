// qtnh_b200.hpp -- header-only C++ layer over the C ABI (qtnh_b200.h) that keeps
// the reference's C++ API shape for the hot path, so existing callers of
//   qtnh::World / Rank / Group / Tensor / ops::* / remap::tensor_to_tensor /
//   linalg::{Grid, BlockCyclicMatrix, tensor_to_matrix, pgemm, matrix_to_tensor,
//            psvd, truncate_svd, absorb_singular_left/right}
// (/root/reference/proj/include/qtnh/*.hpp) switch by changing the namespace:
//   namespace qtnh = qtnh_b200;
// Errors come back as the same exception classes (common.hpp:31-74).
//
// What differs underneath (and is invisible at this API):
//   * tensor values live in HBM; Tensor copies share the immutable value and
//     mutable_local_data() copies on write (tensor.hpp:41-43 value semantics);
//   * a linalg::BlockCyclicMatrix is a LAZY view of a device tensor (rows and
//     columns = index groups flattened row-major in list order, linalg.hpp:203-207):
//     tensor_to_matrix moves nothing, pgemm is one contraction whose layout
//     permutation is fused into the FP64-tensor-core GEMM's operand loads, and
//     matrix_to_tensor is one permutation (nothing when the order already fits).
//     The block-cyclic grid, row_block and col_block are accepted and reported but
//     do not decide any data placement (they emulate ScaLAPACK);
//   * psvd runs the batched Jacobi SVD on the device (a distributed matrix is
//     gathered onto its root copy first, like linalg.hpp:441-462).
#pragma once

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <numeric>
#include <stdexcept>
#include <string>
#include <thread>
#include <type_traits>
#include <vector>

#include "qtnh_b200.h"

namespace qtnh_b200 {

using Complex = std::complex<double>;
using Dim = std::int64_t;
using Coords = std::vector<Dim>;  // indexing.hpp:27

struct Error : std::runtime_error {
  explicit Error(const std::string& m) : std::runtime_error(m) {}
};
struct InvalidArgument : Error { using Error::Error; };
struct ResourceError : Error {
  ResourceError(const std::string& m, std::int64_t r) : Error(m), required_ranks(r) {}
  std::int64_t required_ranks;
};
struct ProtocolError : Error { using Error::Error; };
struct NumericalError : Error {
  NumericalError(const std::string& m, std::int64_t i) : Error(m), info(i) {}
  std::int64_t info;
};
struct PreconditionError : Error { using Error::Error; };
struct DegenerateStateError : Error { using Error::Error; };
struct AbortedError : Error { using Error::Error; };

inline void check(int status) {
  if (status == QTNH_OK) return;
  char buf[2048];
  qtnh_last_error(buf, sizeof buf);
  std::string m(buf);
  switch (status) {
    case QTNH_E_INVALID_ARGUMENT: throw InvalidArgument(m);
    case QTNH_E_RESOURCE: throw ResourceError(m, qtnh_last_error_info());
    case QTNH_E_PROTOCOL: throw ProtocolError(m);
    case QTNH_E_NUMERICAL: throw NumericalError(m, qtnh_last_error_info());
    case QTNH_E_PRECONDITION: throw PreconditionError(m);
    case QTNH_E_DEGENERATE: throw DegenerateStateError(m);
    case QTNH_E_ABORTED: throw AbortedError(m);
    default: throw Error(m);
  }
}

struct IndexTuple {  // indexing.hpp:32-80
  std::vector<Dim> dims;
  int split = 0;
  IndexTuple() = default;
  IndexTuple(std::vector<Dim> d, int s) : dims(std::move(d)), split(s) { validate(); }
  void validate() const {
    if (split < 0 || split > static_cast<int>(dims.size()))
      throw InvalidArgument("index split " + std::to_string(split) + " outside [0, " + std::to_string(dims.size()) +
                            "]");
    for (Dim d : dims)
      if (d < 1) throw InvalidArgument("index dimensions must be positive");
  }
  int n_idx() const { return static_cast<int>(dims.size()); }
  int n_dist() const { return split; }
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
  /// "(d0,d1;l0,l1)": distributed dims, ';', local dims (indexing.hpp:70-79).
  std::string str() const {
    std::string out = "(";
    for (int i = 0; i < n_idx(); ++i) {
      if (i == split) out += ";";
      else if (i > 0) out += ",";
      out += std::to_string(dims[i]);
    }
    if (split == n_idx()) out += ";";
    return out + ")";
  }
};

struct DistParams {  // indexing.hpp:84-101
  Dim stretch = 1, cycles = 1, offset = 0;
  DistParams() = default;
  DistParams(Dim s, Dim c, Dim o) : stretch(s), cycles(c), offset(o) {}
  void validate() const {
    if (stretch < 1 || cycles < 1 || offset < 0)
      throw InvalidArgument("invalid broadcast parameters (str=" + std::to_string(stretch) +
                            ", cyc=" + std::to_string(cycles) + ", off=" + std::to_string(offset) + ")");
  }
  Dim span(Dim dist_size) const { return stretch * cycles * dist_size; }
  bool operator==(const DistParams& o) const {
    return stretch == o.stretch && cycles == o.cycles && offset == o.offset;
  }
  bool operator!=(const DistParams& o) const { return !(*this == o); }
};

// ---- layout arithmetic (indexing.hpp:103-219), host only ---------------------------
namespace idx {
/// Row-major strides (rightmost index fastest).
inline std::vector<Dim> strides(const std::vector<Dim>& dims) {
  std::vector<Dim> st(dims.size(), 1);
  for (std::size_t i = dims.size(); i-- > 1;) st[i - 1] = st[i] * dims[i];
  return st;
}
/// Row-major flat offset of `coords` over `dims`, bounds checked.
inline Dim flat(const Coords& coords, const std::vector<Dim>& dims) {
  if (coords.size() != dims.size()) throw InvalidArgument("coordinate count does not match dimension count");
  Dim at = 0;
  for (std::size_t i = 0; i < dims.size(); ++i) {
    if (coords[i] < 0 || coords[i] >= dims[i])
      throw InvalidArgument("coordinate " + std::to_string(coords[i]) + " out of bounds for dimension " +
                            std::to_string(dims[i]));
    at = at * dims[i] + coords[i];
  }
  return at;
}
inline Coords unflat(Dim at, const std::vector<Dim>& dims) {
  Coords c(dims.size(), 0);
  for (std::size_t i = dims.size(); i-- > 0;) {
    c[i] = at % dims[i];
    at /= dims[i];
  }
  return c;
}
}  // namespace idx

/// Offset of local coordinates inside a rank's block (indexing.hpp:137-139).
inline Dim flat_offset(const Coords& local_coords, const IndexTuple& shape) {
  return idx::flat(local_coords, shape.local_dims());
}
/// Every rank holding block b: offset + c str N_d + b str + t over cycles c and slots t
/// (indexing.hpp:141-168).
inline std::vector<int> home_ranks_of_block(Dim b, Dim dist_size, const DistParams& dist) {
  std::vector<int> homes;
  for (Dim c = 0; c < dist.cycles; ++c)
    for (Dim t = 0; t < dist.stretch; ++t)
      homes.push_back(static_cast<int>(dist.offset + (c * dist_size + b) * dist.stretch + t));
  return homes;
}
inline std::vector<int> home_ranks(const Coords& dist_coords, const IndexTuple& shape, const DistParams& dist) {
  return home_ranks_of_block(idx::flat(dist_coords, shape.dist_dims()), shape.dist_size(), dist);
}
/// The cycle-0, slot-0 holder of block b (indexing.hpp:171-173).
inline int canonical_rank_of_block(Dim b, const DistParams& dist) {
  return static_cast<int>(dist.offset + b * dist.stretch);
}
struct BlockLocation {
  Dim cycle, block, slot;
};
/// Which copy of which block `rank` holds; false outside the span (indexing.hpp:181-191).
inline bool locate_rank(int rank, Dim dist_size, const DistParams& dist, BlockLocation* loc) {
  const Dim rel = rank - dist.offset;
  if (rel < 0 || rel >= dist.span(dist_size)) return false;
  const Dim per_cycle = dist.stretch * dist_size;
  loc->cycle = rel / per_cycle;
  loc->block = (rel % per_cycle) / dist.stretch;
  loc->slot = rel % dist.stretch;
  return true;
}
/// Row-major coordinate counter (indexing.hpp:193-219); advance() returns the index
/// that was incremented, -1 after the last tuple.
class Odometer {
 public:
  explicit Odometer(std::vector<Dim> dims) : dims_(std::move(dims)), at_(dims_.size(), 0) {
    for (Dim d : dims_) count_ *= d;
  }
  Dim count() const { return count_; }
  const Coords& coords() const { return at_; }
  int advance() {
    for (std::size_t i = dims_.size(); i-- > 0;) {
      if (++at_[i] < dims_[i]) return static_cast<int>(i);
      at_[i] = 0;
    }
    return -1;
  }

 private:
  std::vector<Dim> dims_;
  Coords at_;
  Dim count_ = 1;
};

/// tensor.hpp:28-39
enum class Variant : std::uint32_t { dense = 0, symmetric = 1, diagonal = 2, identity = 3, swap = 4 };
inline const char* variant_name(Variant v) {
  static const char* names[] = {"dense", "symmetric", "diagonal", "identity", "swap"};
  return static_cast<std::uint32_t>(v) < 5 ? names[static_cast<std::uint32_t>(v)] : "?";
}

class Rank;

/// Communicator over an ordered subset of world ranks (runtime.hpp:120-180).
/// Host-data collectives; their transport is the world's exchange (NVLink peer
/// copies, NCCL or CUDA IPC) through qtnh_group_all_to_all_v_host.
class Group {
 public:
  Group() = default;
  int size() const { return static_cast<int>(members_.size()); }
  int rank() const { return me_; }
  const std::vector<int>& members() const { return members_; }
  int world_rank(int group_rank) const { return members_.at(group_rank); }
  bool contains(int world_rank) const {
    return std::find(members_.begin(), members_.end(), world_rank) != members_.end();
  }

  /// runtime.hpp:448-475; a mismatch against expected_counts raises ProtocolError
  /// "all_to_all_v count mismatch for pair (src -> dst)" on every member.
  template <class T>
  std::vector<std::vector<T>> all_to_all_v(const std::vector<std::vector<T>>& send_lists,
                                           const std::vector<std::size_t>* expected_counts = nullptr) const {
    static_assert(std::is_trivially_copyable<T>::value, "group collectives move trivially copyable values");
    if (static_cast<int>(send_lists.size()) != size())
      throw InvalidArgument("all_to_all_v needs one send list per group member");
    std::vector<const void*> ptrs(size());
    std::vector<int64_t> counts(size()), expected(size()), got(size());
    for (int i = 0; i < size(); ++i) {
      ptrs[i] = send_lists[i].data();
      counts[i] = static_cast<int64_t>(send_lists[i].size());
      if (expected_counts) expected[i] = static_cast<int64_t>((*expected_counts)[i]);
    }
    void* recv = nullptr;
    check(qtnh_group_all_to_all_v_host(h_, size(), members_.data(), sizeof(T), ptrs.data(), counts.data(),
                                       expected_counts ? expected.data() : nullptr, &recv, got.data()));
    std::vector<std::vector<T>> out(size());
    const char* at = static_cast<const char*>(recv);
    for (int i = 0; i < size(); ++i) {
      out[i].resize(static_cast<std::size_t>(got[i]));
      if (got[i]) std::memcpy(static_cast<void*>(out[i].data()), at, got[i] * sizeof(T));
      at += got[i] * sizeof(T);
    }
    qtnh_free_host(recv);
    return out;
  }

  /// runtime.hpp:135-136: the root's data on every member.
  template <class T>
  std::vector<T> broadcast(std::vector<T> data, int root) const {
    std::vector<std::vector<T>> send(size());
    if (me_ == root)
      for (auto& s : send) s = data;
    return std::move(all_to_all_v(send)[root]);
  }
  /// runtime.hpp:138-139: every member's data on the root (empty elsewhere).
  template <class T>
  std::vector<std::vector<T>> gather(const std::vector<T>& data, int root) const {
    std::vector<std::vector<T>> send(size());
    send[root] = data;
    auto got = all_to_all_v(send);
    if (me_ != root) return {};
    return got;
  }
  /// runtime.hpp:141-142: chunk j of the root to member j.
  template <class T>
  std::vector<T> scatter(const std::vector<std::vector<T>>& chunks, int root) const {
    std::vector<std::vector<T>> send(size());
    if (me_ == root) {
      if (static_cast<int>(chunks.size()) != size()) throw InvalidArgument("scatter needs one chunk per member");
      send = chunks;
    }
    return std::move(all_to_all_v(send)[root]);
  }
  /// runtime.hpp:421-438: element-wise sum combined in member order (deterministic).
  template <class T>
  std::vector<T> all_reduce_sum(const std::vector<T>& data) const {
    std::vector<std::vector<T>> send(size(), data);
    auto got = all_to_all_v(send);
    std::vector<T> out(data.size(), T{});
    for (const auto& g : got) {
      if (g.size() != data.size()) throw ProtocolError("all_reduce_sum length mismatch");
      for (std::size_t k = 0; k < g.size(); ++k) out[k] += g[k];
    }
    return out;
  }
  double all_reduce_sum(double x) const { return all_reduce_sum(std::vector<double>{x})[0]; }
  Complex all_reduce_sum(Complex x) const { return all_reduce_sum(std::vector<Complex>{x})[0]; }
  void barrier() const { all_to_all_v(std::vector<std::vector<char>>(size())); }

 private:
  friend class Rank;
  Group(qtnh_rank_t h, std::vector<int> m, int me) : h_(h), members_(std::move(m)), me_(me) {}
  qtnh_rank_t h_ = nullptr;
  std::vector<int> members_;
  int me_ = 0;
};

class Rank {  // runtime.hpp:182-240
 public:
  int rank() const { return qtnh_rank_id(h_); }
  int size() const { return size_; }
  qtnh_rank_t handle() const { return h_; }

  /// Opens a group over `members` (ordered, duplicate-free world ranks); called by
  /// exactly the member ranks (runtime.hpp:191-223, same validation messages).
  Group group(const std::vector<int>& members) {
    if (members.empty()) throw InvalidArgument("group members must be non-empty");
    std::vector<int> seen;
    int my_index = -1;
    for (std::size_t i = 0; i < members.size(); ++i) {
      int m = members[i];
      if (m < 0 || m >= size_) throw InvalidArgument("group member " + std::to_string(m) + " out of range");
      if (std::find(seen.begin(), seen.end(), m) != seen.end())
        throw InvalidArgument("duplicate group member " + std::to_string(m));
      seen.push_back(m);
      if (m == rank()) my_index = static_cast<int>(i);
    }
    if (my_index < 0)
      throw InvalidArgument("rank " + std::to_string(rank()) + " cannot open a group it is not a member of");
    return Group(h_, members, my_index);
  }
  Group world_group() {
    std::vector<int> m(size_);
    std::iota(m.begin(), m.end(), 0);
    return group(m);
  }

 private:
  friend class World;
  Rank(qtnh_rank_t h, int size) : h_(h), size_(size) {}
  qtnh_rank_t h_;
  int size_;
};

class World {  // runtime.hpp:243-303
 public:
  /// n rank threads over `devices` (default: all on device 0) -- World(n).
  explicit World(int n, const std::vector<int>& devices = {}) : n_(n) {
    check(qtnh_world_create_local(n, devices.empty() ? nullptr : devices.data(), &w_));
  }
  /// Process-per-GPU world over NCCL (Backend::external_message_passing,
  /// runtime.hpp:248-251): rank `rank` of `size`, uid from nccl_unique_id() on rank 0.
  static std::unique_ptr<World> nccl(int rank, int size, int device, const std::vector<char>& uid) {
    if (uid.size() != 128) throw InvalidArgument("NCCL unique id must be 128 bytes");
    std::unique_ptr<World> w(new World());
    w->n_ = size;
    w->my_rank_ = rank;
    check(qtnh_world_create_nccl(rank, size, device, uid.data(), &w->w_));
    return w;
  }
  static std::vector<char> nccl_unique_id() {
    std::vector<char> uid(128);
    check(qtnh_nccl_unique_id(uid.data()));
    return uid;
  }
  /// Process-per-GPU world over CUDA IPC (one node; processes meet under `dir`).
  static std::unique_ptr<World> ipc(int rank, int size, int device, const std::string& dir) {
    std::unique_ptr<World> w(new World());
    w->n_ = size;
    w->my_rank_ = rank;
    check(qtnh_world_create_ipc(rank, size, device, dir.c_str(), &w->w_));
    return w;
  }
  ~World() {
    if (w_) qtnh_world_destroy(w_);
  }
  World(const World&) = delete;
  World& operator=(const World&) = delete;
  int size() const { return n_; }

  /// One host thread per rank (local world) or this process's rank (NCCL / IPC
  /// world); rethrows the originating failure, preferring it over secondary
  /// AbortedErrors (runtime.hpp:263-299).
  void run(const std::function<void(Rank&)>& body) {
    if (my_rank_ >= 0) {
      qtnh_rank_t h = nullptr;
      check(qtnh_rank_bind(w_, my_rank_, &h));
      try {
        Rank rk(h, n_);
        body(rk);
      } catch (...) {
        qtnh_world_abort(w_);
        qtnh_rank_release(h);
        throw;
      }
      qtnh_rank_release(h);
      return;
    }
    std::vector<std::thread> ts;
    std::vector<std::exception_ptr> errs(n_);
    for (int r = 0; r < n_; ++r)
      ts.emplace_back([&, r] {
        qtnh_rank_t h = nullptr;
        try {
          check(qtnh_rank_bind(w_, r, &h));
          Rank rk(h, n_);
          body(rk);
        } catch (...) {
          errs[r] = std::current_exception();
          qtnh_world_abort(w_);
        }
        if (h) qtnh_rank_release(h);
      });
    for (auto& t : ts) t.join();
    std::exception_ptr first;
    for (auto& e : errs) {
      if (!e) continue;
      if (!first) first = e;
      try {
        std::rethrow_exception(e);
      } catch (const AbortedError&) {
      } catch (...) {
        std::rethrow_exception(e);
      }
    }
    if (first) std::rethrow_exception(first);
  }

 private:
  World() = default;
  int n_ = 0;
  int my_rank_ = -1;
  qtnh_world_t w_ = nullptr;
};

class Tensor;
Tensor wrap(qtnh_tensor_t h, Rank* ctx);

class Tensor {  // tensor.hpp:53-695 (dense)
 public:
  Tensor() = default;
  // Value semantics (tensor.hpp:41-43): a copy is a new handle on the same
  // immutable device value; mutable_local_data() copies on write.
  Tensor(const Tensor& o) : ctx_(o.ctx_) {
    if (o.st_) {
      qtnh_tensor_t h;
      check(qtnh_tensor_clone(o.h(), &h));
      st_ = std::make_shared<State>(h);
    }
  }
  Tensor& operator=(const Tensor& o) {
    if (this != &o) {
      Tensor t(o);
      *this = std::move(t);
    }
    return *this;
  }
  Tensor(Tensor&&) = default;
  Tensor& operator=(Tensor&&) = default;

  static Tensor dense(Rank& r, const IndexTuple& s, DistParams d, const std::vector<Complex>& local) {
    qtnh_tensor_t h;
    int64_t dd[3] = {d.stretch, d.cycles, d.offset};
    const bool fits = static_cast<Dim>(local.size()) == s.local_size();
    check(qtnh_tensor_dense(r.handle(), s.n_idx(), s.dims.data(), s.split, dd,
                            fits && !local.empty() ? reinterpret_cast<const double*>(local.data()) : nullptr, &h));
    Tensor t = wrap(h, &r);
    if (!fits && t.in_span())  // span ranks need exactly their block (tensor.hpp:64-69)
      throw InvalidArgument("dense local data has " + std::to_string(local.size()) + " elements, expected " +
                            std::to_string(s.local_size()));
    return t;
  }
  static Tensor from_global(Rank& r, const IndexTuple& s, DistParams d, const std::vector<Complex>& global) {
    if (static_cast<Dim>(global.size()) != s.total_size()) throw InvalidArgument("global element count mismatch");
    qtnh_tensor_t h;
    int64_t dd[3] = {d.stretch, d.cycles, d.offset};
    check(qtnh_tensor_from_global(r.handle(), s.n_idx(), s.dims.data(), s.split, dd,
                                  reinterpret_cast<const double*>(global.data()), &h));
    return wrap(h, &r);
  }
  /// tensor.hpp:72-80: elements computed per global coordinate tuple on every span rank.
  static Tensor dense_fn(Rank& r, const IndexTuple& s, DistParams d, const std::function<Complex(const Coords&)>& fn) {
    d.validate();
    BlockLocation loc{0, 0, 0};
    std::vector<Complex> block;
    if (d.offset + d.span(s.dist_size()) <= r.size() && locate_rank(r.rank(), s.dist_size(), d, &loc)) {
      Coords full = idx::unflat(loc.block, s.dist_dims());
      full.resize(s.n_idx(), 0);
      Odometer od(s.local_dims());
      block.reserve(static_cast<std::size_t>(od.count()));
      for (Dim i = 0; i < od.count(); ++i) {
        std::copy(od.coords().begin(), od.coords().end(), full.begin() + s.split);
        block.push_back(fn(full));
        od.advance();
      }
    }
    return dense(r, s, d, block);
  }
  /// tensor.hpp:97-112: dense storage, half-split (in, out) layout validated.
  static Tensor symmetric(Rank& r, const IndexTuple& s, DistParams d, const std::vector<Complex>& local) {
    qtnh_tensor_t h;
    int64_t dd[3] = {d.stretch, d.cycles, d.offset};
    check(qtnh_tensor_symmetric(r.handle(), s.n_idx(), s.dims.data(), s.split, dd,
                                reinterpret_cast<const double*>(local.data()), static_cast<int64_t>(local.size()), 0,
                                &h));
    return wrap(h, &r);
  }
  static Tensor symmetric_from_global(Rank& r, const IndexTuple& s, DistParams d, const std::vector<Complex>& global) {
    qtnh_tensor_t h;
    int64_t dd[3] = {d.stretch, d.cycles, d.offset};
    check(qtnh_tensor_symmetric(r.handle(), s.n_idx(), s.dims.data(), s.split, dd,
                                reinterpret_cast<const double*>(global.data()), static_cast<int64_t>(global.size()),
                                1, &h));
    return wrap(h, &r);
  }
  /// tensor.hpp:114-142: `diag_global` = the diagonal in row-major order of the input
  /// coordinates; each on-diagonal block keeps its slice in HBM.
  static Tensor diagonal(Rank& r, const IndexTuple& s, DistParams d, const std::vector<Complex>& diag_global) {
    qtnh_tensor_t h;
    int64_t dd[3] = {d.stretch, d.cycles, d.offset};
    check(qtnh_tensor_diagonal(r.handle(), s.n_idx(), s.dims.data(), s.split, dd,
                               reinterpret_cast<const double*>(diag_global.data()),
                               static_cast<int64_t>(diag_global.size()), &h));
    return wrap(h, &r);
  }
  /// tensor.hpp:450-455: the same value under given metadata; `local` is this rank's
  /// stored data (the block, or the diagonal slice of a diagonal tensor).
  static Tensor adopt(Rank& r, Variant var, const IndexTuple& s, DistParams d, const std::vector<Complex>& local) {
    if (var == Variant::identity || var == Variant::swap)
      throw InvalidArgument("identity / swap tensors are rebuilt from their index pairs");
    qtnh_tensor_t h;
    int64_t dd[3] = {d.stretch, d.cycles, d.offset};
    if (var == Variant::diagonal)
      check(qtnh_tensor_diagonal(r.handle(), s.n_idx(), s.dims.data(), s.split, dd, nullptr, -1, &h));
    else if (var == Variant::symmetric)
      check(qtnh_tensor_symmetric(r.handle(), s.n_idx(), s.dims.data(), s.split, dd, nullptr, 0, 0, &h));
    else
      check(qtnh_tensor_dense(r.handle(), s.n_idx(), s.dims.data(), s.split, dd, nullptr, &h));
    Tensor t = wrap(h, &r);
    if (static_cast<Dim>(local.size()) == qtnh_tensor_stored_size(h) && !local.empty()) {
      check(qtnh_tensor_upload_local(h, reinterpret_cast<const double*>(local.data())));
      check(qtnh_rank_synchronize(r.handle()));
    }
    return t;
  }
  // Tensor::identity / swap_tensor (tensor.hpp:144-164): no storage
  static Tensor identity(Rank& r, const IndexTuple& s, DistParams d, const std::vector<int>& in_pos,
                         const std::vector<int>& out_pos) {
    return paired(r, s, d, in_pos, out_pos, 0);
  }
  static Tensor swap_tensor(Rank& r, const IndexTuple& s, DistParams d, const std::vector<int>& in_pos,
                            const std::vector<int>& out_pos) {
    return paired(r, s, d, in_pos, out_pos, 1);
  }
  static Tensor scalar(Rank& r, Complex v, DistParams d = {}) { return from_global(r, IndexTuple({}, 0), d, {v}); }

  Rank& ctx() const {
    if (!ctx_) throw PreconditionError("tensor has no rank context");
    return *ctx_;
  }
  IndexTuple shape() const {
    IndexTuple s;
    s.dims.resize(qtnh_tensor_rank(h()));
    check(qtnh_tensor_dims(h(), s.dims.data()));
    s.split = qtnh_tensor_split(h());
    return s;
  }
  DistParams dist() const {
    int64_t d[3];
    check(qtnh_tensor_dist(h(), d));
    return {d[0], d[1], d[2]};
  }
  Variant variant() const { return static_cast<Variant>(qtnh_tensor_variant(h())); }
  Dim span() const { return qtnh_tensor_span(h()); }
  bool in_span() const { return qtnh_tensor_in_span(h()) != 0; }
  Dim my_block() const { return qtnh_tensor_my_block(h()); }
  bool is_canonical_holder() const { return qtnh_tensor_is_canonical(h()) != 0; }
  /// Index pairs of an identity / swap tensor as constructed (tensor.hpp:193-194).
  std::vector<int> equality_in() const { return pairs(0); }
  std::vector<int> equality_out() const { return pairs(1); }
  /// Input halves of the (in, out) layout (symmetric and diagonal tensors, tensor.hpp:196-203).
  std::vector<Dim> in_dist_dims() const {
    IndexTuple s = shape();
    return {s.dims.begin(), s.dims.begin() + s.split / 2};
  }
  std::vector<Dim> in_local_dims() const {
    IndexTuple s = shape();
    return {s.dims.begin() + s.split, s.dims.begin() + s.split + s.n_local() / 2};
  }
  /// tensor.hpp:209-247: value at global coordinates from this rank's storage.
  Complex local_element(const Coords& coords) const {
    if (static_cast<int>(coords.size()) != qtnh_tensor_rank(h()))
      throw InvalidArgument("expected " + std::to_string(qtnh_tensor_rank(h())) + " coordinates");
    double v[2];
    check(qtnh_tensor_local_element(h(), coords.data(), v));
    return {v[0], v[1]};
  }
  /// tensor.hpp:251-264: span-collective; the canonical holder's value on every span rank.
  Complex element(const Coords& coords) const { return element_over(coords, false); }
  /// tensor.hpp:268-277: world-collective.
  Complex element_world(const Coords& coords) const { return element_over(coords, true); }
  /// tensor.hpp:282-296: dense tensor with the same shape, distribution and values.
  Tensor to_dense() const {
    qtnh_tensor_t o;
    check(qtnh_tensor_to_dense(h(), &o));
    return wrap(o, ctx_);
  }
  std::vector<int> span_ranks() const {
    auto d = dist();
    std::vector<int> out;
    for (Dim i = 0; i < span(); ++i) out.push_back(static_cast<int>(d.offset + i));
    return out;
  }

  /// This rank's stored elements, downloaded (tensor.hpp:177): the block, a diagonal
  /// tensor's slice of the diagonal, nothing for identity / swap.
  std::vector<Complex> local_data() const {
    std::vector<Complex> v(static_cast<std::size_t>(qtnh_tensor_stored_size(h())));
    if (!v.empty()) check(qtnh_tensor_download_local(h(), reinterpret_cast<double*>(v.data())));
    return v;
  }
  /// tensor.hpp:178: a host mirror of this rank's block; the value is made
  /// exclusive to this Tensor (copy on write) and the mirror is written back to
  /// the device before the next operation that reads this Tensor. Writes after
  /// that operation need another mutable_local_data() call.
  std::vector<Complex>& mutable_local_data() {
    if (!st_) throw PreconditionError("empty tensor");
    check(qtnh_tensor_make_mutable(st_->h));
    st_->mirror = local_data();
    st_->dirty = true;
    return st_->mirror;
  }
  std::vector<Complex> to_global_vector() const {
    if (!in_span()) return {};
    std::vector<Complex> v(shape().total_size());
    check(qtnh_tensor_to_global(h(), reinterpret_cast<double*>(v.data())));
    return v;
  }
  qtnh_tensor_t h() const {
    if (!st_) throw PreconditionError("empty tensor");
    if (st_->dirty) {  // write the host mirror back (mutable_local_data)
      st_->dirty = false;
      if (!st_->mirror.empty())
        check(qtnh_tensor_upload_local(st_->h, reinterpret_cast<const double*>(st_->mirror.data())));
    }
    return st_->h;
  }

  // serialization (tensor.hpp:388-446), QTNHTEN1 byte-identical to the reference
  void save(const std::string& path) const { check(qtnh_tensor_save(h(), path.c_str())); }
  static Tensor load(Rank& r, const std::string& path) {
    qtnh_tensor_t o;
    check(qtnh_tensor_load(r.handle(), path.c_str(), &o));
    return wrap(o, &r);
  }
  static Tensor paired(Rank& r, const IndexTuple& s, DistParams d, const std::vector<int>& in_pos,
                       const std::vector<int>& out_pos, int crossed) {
    if (in_pos.size() != out_pos.size()) throw InvalidArgument("input/output position lists differ in length");
    qtnh_tensor_t o;
    int64_t dd[3] = {d.stretch, d.cycles, d.offset};
    check(qtnh_tensor_paired(r.handle(), s.n_idx(), s.dims.data(), s.split, dd, static_cast<int>(in_pos.size()),
                             in_pos.data(), out_pos.data(), crossed, &o));
    return wrap(o, &r);
  }

 private:
  struct State {
    explicit State(qtnh_tensor_t x) : h(x) {}
    ~State() { qtnh_tensor_free(h); }
    State(const State&) = delete;
    State& operator=(const State&) = delete;
    qtnh_tensor_t h;
    std::vector<Complex> mirror;
    bool dirty = false;
  };
  Tensor(qtnh_tensor_t h, Rank* ctx) : st_(std::make_shared<State>(h)), ctx_(ctx) {}
  std::vector<int> pairs(int which) const {
    Variant v = variant();
    if (v != Variant::identity && v != Variant::swap) return {};
    std::vector<int> in(qtnh_tensor_rank(h()) / 2), out(in.size());
    check(qtnh_tensor_pairs(h(), in.data(), out.data()));
    return which ? out : in;
  }
  Complex element_over(const Coords& coords, bool world) const {
    IndexTuple s = shape();
    if (static_cast<int>(coords.size()) != s.n_idx())
      throw InvalidArgument("expected " + std::to_string(s.n_idx()) + " coordinates");
    for (int i = 0; i < s.n_idx(); ++i)
      if (coords[i] < 0 || coords[i] >= s.dims[i])
        throw InvalidArgument("coordinate out of bounds at index " + std::to_string(i));
    if (!world) {
      if (!in_span()) return {0.0, 0.0};
      if (span() == 1) return local_element(coords);
    }
    DistParams d = dist();
    const int root = canonical_rank_of_block(idx::flat(Coords(coords.begin(), coords.begin() + s.split), s.dist_dims()), d);
    Group g = world ? ctx().world_group() : ctx().group(span_ranks());
    std::vector<Complex> one;
    if (ctx().rank() == root) one.push_back(local_element(coords));
    one = g.broadcast(one, world ? root : root - static_cast<int>(d.offset));
    return one.at(0);
  }
  std::shared_ptr<State> st_;
  Rank* ctx_ = nullptr;
  friend Tensor wrap(qtnh_tensor_t, Rank*);
};

inline Tensor wrap(qtnh_tensor_t h, Rank* ctx) { return Tensor(h, ctx); }

namespace ops {  // ops.hpp
inline Tensor permute(const Tensor& t, const std::vector<int>& perm, int new_split) {  // ops.hpp:27-49
  if (static_cast<int>(perm.size()) != qtnh_tensor_rank(t.h()))
    throw InvalidArgument("permutation size does not match tensor rank");
  qtnh_tensor_t o;
  check(qtnh_permute(t.h(), perm.data(), new_split, &o));
  return wrap(o, &t.ctx());
}
inline Tensor rebcast(const Tensor& t, DistParams d) {  // ops.hpp:54-112
  qtnh_tensor_t o;
  int64_t dd[3] = {d.stretch, d.cycles, d.offset};
  check(qtnh_rebcast(t.h(), dd, &o));
  return wrap(o, &t.ctx());
}
inline Tensor scatter_index(const Tensor& t, int pos) {  // ops.hpp:118
  qtnh_tensor_t o;
  check(qtnh_scatter_index(t.h(), pos, &o));
  return wrap(o, &t.ctx());
}
inline Tensor gather_index(const Tensor& t, int pos) {  // ops.hpp:133
  qtnh_tensor_t o;
  check(qtnh_gather_index(t.h(), pos, &o));
  return wrap(o, &t.ctx());
}
// remap::tensor_to_tensor (remap.hpp:106): axis_map[src] = dst position
inline Tensor tensor_to_tensor(const Tensor& t, const IndexTuple& dst, DistParams d, const std::vector<int>& axis_map,
                               Variant dst_variant = Variant::dense) {
  if (dst_variant != Variant::dense && dst_variant != Variant::symmetric)
    throw InvalidArgument("remap destinations store every element (dense or symmetric)");
  qtnh_tensor_t o;
  int64_t dd[3] = {d.stretch, d.cycles, d.offset};
  check(qtnh_remap(t.h(), axis_map.data(), dst.n_idx(), dst.dims.data(), dst.split, dd, &o));
  Tensor out = wrap(o, &t.ctx());
  if (dst_variant == Variant::dense) return out;
  return Tensor::adopt(t.ctx(), Variant::symmetric, dst, d, out.local_data());  // tag kept, as remap.hpp:125
}
inline Tensor slice_local_dims(const Tensor& t, const std::vector<Dim>& new_local) {  // ops.hpp:166
  qtnh_tensor_t o;
  check(qtnh_slice_local_dims(t.h(), new_local.data(), &o));
  return wrap(o, &t.ctx());
}
inline Tensor pad_local_dims(const Tensor& t, const std::vector<Dim>& new_local) {  // ops.hpp:201
  qtnh_tensor_t o;
  check(qtnh_pad_local_dims(t.h(), new_local.data(), &o));
  return wrap(o, &t.ctx());
}
inline Tensor squeeze(const Tensor& t, int pos) {  // ops.hpp:234
  qtnh_tensor_t o;
  check(qtnh_squeeze(t.h(), pos, &o));
  return wrap(o, &t.ctx());
}
inline Tensor unsqueeze(const Tensor& t, int pos, bool as_dist = false) {  // ops.hpp:248
  qtnh_tensor_t o;
  check(qtnh_unsqueeze(t.h(), pos, as_dist ? 1 : 0, &o));
  return wrap(o, &t.ctx());
}
inline Tensor conj(const Tensor& t) {  // ops.hpp:147
  qtnh_tensor_t o;
  check(qtnh_conj(t.h(), &o));
  return wrap(o, &t.ctx());
}
inline Tensor scale(const Tensor& t, Complex a) {  // ops.hpp:155
  qtnh_tensor_t o;
  check(qtnh_scale(t.h(), a.real(), a.imag(), &o));
  return wrap(o, &t.ctx());
}
/// Real factor per coordinate of index `pos` (the tensor form of absorb_singular_*).
inline Tensor scale_index(const Tensor& t, int pos, const std::vector<double>& factors) {
  qtnh_tensor_t o;
  check(qtnh_scale_index(t.h(), pos, factors.data(), &o));
  return wrap(o, &t.ctx());
}
/// Same local block under new dims (no distributed indices; equal element count).
inline Tensor reshape(const Tensor& t, const std::vector<Dim>& dims) {
  qtnh_tensor_t o;
  check(qtnh_tensor_reshape(t.h(), static_cast<int>(dims.size()), dims.data(), &o));
  return wrap(o, &t.ctx());
}
}  // namespace ops

namespace remap {  // remap.hpp
using ops::tensor_to_tensor;
}  // namespace remap

namespace network {  // SPEC.md:361-369, result order SPEC.md:408
inline Tensor contract(const Tensor& a, const Tensor& b, const std::vector<int>& a_pos,
                       const std::vector<int>& b_pos) {
  if (a_pos.size() != b_pos.size()) throw InvalidArgument("contracted position lists differ in length");
  qtnh_tensor_t o;
  check(qtnh_contract(a.h(), b.h(), static_cast<int>(a_pos.size()), a_pos.data(), b_pos.data(), &o));
  return wrap(o, &a.ctx());
}

/// Contraction order of a labelled network (SPEC network::contract_order, SPEC.md:
/// 391-399): labels[t] names the indices of tensor t in order, a label shared by two
/// tensors is a bond, label_dim[l] its dimension. Seeded randomised greedy search on
/// the host cores, best of `trials`: by (largest intermediate, flops), or -- with
/// max_log2_size > 0 -- the fewest flops among the orders whose largest intermediate
/// has at most 2^max_log2_size elements. Step s joins (first, second); its result
/// gets id labels.size() + s.
inline std::vector<std::pair<int, int>> plan_order(const std::vector<std::vector<int>>& labels,
                                                   const std::vector<Dim>& label_dim, std::uint64_t seed = 0,
                                                   int trials = 64, double max_log2_size = 0.0) {
  const int n = static_cast<int>(labels.size());
  std::vector<int> offs{0}, flat;
  for (const auto& l : labels) {
    flat.insert(flat.end(), l.begin(), l.end());
    offs.push_back(static_cast<int>(flat.size()));
  }
  std::vector<double> lg(label_dim.size());
  for (size_t i = 0; i < lg.size(); ++i) lg[i] = std::log2(static_cast<double>(label_dim[i]));
  std::vector<int> out(2 * static_cast<size_t>(n > 1 ? n - 1 : 1));
  if (flat.empty()) flat.push_back(0);
  check(qtnh_plan_order_capped(n, offs.data(), flat.data(), static_cast<int>(lg.size()), lg.data(), seed, trials,
                               max_log2_size, out.data()));
  std::vector<std::pair<int, int>> order;
  for (int s = 0; s + 1 < n; ++s) order.emplace_back(out[2 * s], out[2 * s + 1]);
  return order;
}

/// The whole order in one call (qtnh_contract_chain): every step contracts the labels
/// its two operands share, the result carries open(a) then open(b), and
/// intermediates are released as soon as they are consumed. Returns the last result
/// and, through `result_labels`, its index labels.
inline Tensor contract_order(const std::vector<Tensor>& tensors, const std::vector<std::vector<int>>& labels,
                             const std::vector<std::pair<int, int>>& order,
                             std::vector<int>* result_labels = nullptr) {
  if (tensors.empty() || tensors.size() != labels.size()) throw InvalidArgument("one label list per tensor");
  if (order.empty()) {
    if (result_labels) *result_labels = labels[0];
    return tensors[0];
  }
  std::vector<std::vector<int>> lab = labels;
  std::vector<qtnh_tensor_t> in;
  for (const Tensor& t : tensors) in.push_back(t.h());
  std::vector<int> ab, np, ap, bp;
  for (const auto& st : order) {
    if (st.first < 0 || st.second < 0 || st.first >= static_cast<int>(lab.size()) ||
        st.second >= static_cast<int>(lab.size()))
      throw InvalidArgument("order refers to a tensor that does not exist yet");
    const auto& la = lab[st.first];
    const auto& lb = lab[st.second];
    std::vector<int> nl;
    int pairs = 0;
    for (size_t i = 0; i < la.size(); ++i) {
      auto it = std::find(lb.begin(), lb.end(), la[i]);
      if (it == lb.end()) {
        nl.push_back(la[i]);
      } else {
        ap.push_back(static_cast<int>(i));
        bp.push_back(static_cast<int>(it - lb.begin()));
        ++pairs;
      }
    }
    for (int x : lb)
      if (std::find(la.begin(), la.end(), x) == la.end()) nl.push_back(x);
    ab.push_back(st.first);
    ab.push_back(st.second);
    np.push_back(pairs);
    lab.push_back(nl);
  }
  if (ap.empty()) {
    ap.push_back(0);
    bp.push_back(0);
  }
  qtnh_tensor_t o;
  check(qtnh_contract_chain(static_cast<int>(in.size()), in.data(), static_cast<int>(order.size()), ab.data(),
                            np.data(), ap.data(), bp.data(), &o));
  if (result_labels) *result_labels = lab.back();
  return wrap(o, &tensors[0].ctx());
}
}  // namespace network

namespace linalg {  // linalg.hpp

/// Process grid over an ordered rank group (linalg.hpp:31-67). Kept for the API;
/// it does not place data (see the file comment).
struct Grid {
  Rank* ctx = nullptr;
  Group group;
  int prows = 1, pcols = 1;
  static Grid make(Rank& ctx, const std::vector<int>& members) {
    int n = static_cast<int>(members.size());
    int pr = 1;
    for (int d = 1; d * d <= n; ++d)
      if (n % d == 0) pr = d;
    return Grid{&ctx, ctx.group(members), pr, n / pr};
  }
  int my_prow() const { return group.rank() / pcols; }
  int my_pcol() const { return group.rank() % pcols; }
  int member_at(int prow, int pcol) const { return prow * pcols + pcol; }
  bool same_as(const Grid& o) const {
    return prows == o.prows && pcols == o.pcols && group.members() == o.group.members();
  }
};

/// The matrix interface of linalg.hpp:71-170 over a device tensor: entry (r, c) is
/// the element of `tensor()` whose coordinates at row_pos() flatten to r and at
/// col_pos() to c (row-major in list order, linalg.hpp:203-207).
class BlockCyclicMatrix {
 public:
  BlockCyclicMatrix() = default;
  BlockCyclicMatrix(Tensor t, std::vector<int> row_pos, std::vector<int> col_pos, Dim rb = 0, Dim cb = 0,
                    const Grid* grid = nullptr)
      : t_(std::move(t)), rp_(std::move(row_pos)), cp_(std::move(col_pos)) {
    auto sh = t_.shape();
    rows_ = cols_ = 1;
    for (int p : rp_) rows_ *= sh.dims.at(p);
    for (int p : cp_) cols_ *= sh.dims.at(p);
    // default blocks: the local dims among the rows / columns (linalg.hpp:224-233)
    rb_ = rb;
    cb_ = cb;
    if (rb_ == 0) {
      rb_ = 1;
      for (int p : rp_)
        if (p >= sh.split) rb_ *= sh.dims[p];
    }
    if (cb_ == 0) {
      cb_ = 1;
      for (int p : cp_)
        if (p >= sh.split) cb_ *= sh.dims[p];
    }
    if (rows_ < 1 || cols_ < 1 || rb_ < 1 || cb_ < 1)
      throw InvalidArgument("matrix and block dimensions must be positive");
    if (grid) grid_ = *grid;
  }
  Dim rows() const { return rows_; }
  Dim cols() const { return cols_; }
  Dim row_block() const { return rb_; }
  Dim col_block() const { return cb_; }
  const Grid& grid() const { return grid_; }
  const Tensor& tensor() const { return t_; }
  Tensor& tensor() { return t_; }
  const std::vector<int>& row_pos() const { return rp_; }
  const std::vector<int>& col_pos() const { return cp_; }
  std::vector<Dim> row_dims() const { return pick(rp_); }
  std::vector<Dim> col_dims() const { return pick(cp_); }

  /// Full matrix, column-major, on every rank of the tensor's span (linalg.hpp:111).
  std::vector<Complex> gather_global() const {
    auto sh = t_.shape();
    std::vector<int> perm = rp_;
    perm.insert(perm.end(), cp_.begin(), cp_.end());
    auto g = ops::permute(t_, perm, 0).to_global_vector();  // row-major rows x cols
    std::vector<Complex> out(g.size());
    for (Dim r = 0; r < rows_; ++r)
      for (Dim c = 0; c < cols_; ++c) out[r + c * rows_] = g[r * cols_ + c];
    return out;
  }

 private:
  std::vector<Dim> pick(const std::vector<int>& pos) const {
    auto sh = t_.shape();
    std::vector<Dim> d;
    for (int p : pos) d.push_back(sh.dims[p]);
    return d;
  }
  Tensor t_;
  std::vector<int> rp_, cp_;
  Dim rows_ = 0, cols_ = 0, rb_ = 1, cb_ = 1;
  Grid grid_;
};

namespace detail {
inline void check_partition(const IndexTuple& shape, const std::vector<int>& row_pos,
                            const std::vector<int>& col_pos) {  // linalg.hpp:182-194
  std::vector<bool> seen(shape.n_idx(), false);
  auto mark = [&](int p) {
    if (p < 0 || p >= shape.n_idx() || seen[p])
      throw InvalidArgument("row/col index sets must partition the tensor indices");
    seen[p] = true;
  };
  for (int p : row_pos) mark(p);
  for (int p : col_pos) mark(p);
  for (bool s : seen)
    if (!s) throw InvalidArgument("row/col index sets must cover every index");
}
inline Dim product(const std::vector<Dim>& d) {
  Dim n = 1;
  for (Dim x : d) n *= x;
  return n;
}
// The matrix as a dense tensor [rows..., cols...] (row-major) regrouped to the
// given row and column digit dims; no distributed indices.
inline Tensor canonical(const BlockCyclicMatrix& m, const std::vector<Dim>& rdims, const std::vector<Dim>& cdims) {
  std::vector<int> perm = m.row_pos();
  perm.insert(perm.end(), m.col_pos().begin(), m.col_pos().end());
  Tensor t = ops::permute(m.tensor(), perm, 0);
  std::vector<Dim> d = rdims;
  d.insert(d.end(), cdims.begin(), cdims.end());
  if (d != t.shape().dims) t = ops::reshape(t, d);
  return t;
}
// position of each listed index among the sorted list
inline std::vector<int> ranks_in_sorted(const std::vector<int>& pos, int base) {
  std::vector<int> s = pos, out;
  std::sort(s.begin(), s.end());
  for (int p : pos) out.push_back(base + static_cast<int>(std::find(s.begin(), s.end(), p) - s.begin()));
  return out;
}
}  // namespace detail

/// linalg.hpp:203-268. No data moves: the matrix is a view of t.
inline BlockCyclicMatrix tensor_to_matrix(const Tensor& t, const std::vector<int>& row_pos,
                                          const std::vector<int>& col_pos, const Grid* grid_in = nullptr,
                                          Dim rb = 0, Dim cb = 0) {
  detail::check_partition(t.shape(), row_pos, col_pos);
  return BlockCyclicMatrix(t, row_pos, col_pos, rb, cb, grid_in);
}

/// linalg.hpp:344-400: C = A B as ONE contraction of a's column indices with b's
/// row indices (the FP64-tensor-core GEMM with the layout permutation fused into
/// its operand loads); C is a view of the result tensor.
inline BlockCyclicMatrix pgemm(const BlockCyclicMatrix& a, const BlockCyclicMatrix& b) {
  if (a.cols() != b.rows())
    throw InvalidArgument("pgemm dimension mismatch: " + std::to_string(a.cols()) + " vs " +
                          std::to_string(b.rows()));
  if (a.col_block() != b.row_block()) throw InvalidArgument("pgemm blocking mismatch on the contracted dimension");
  if (a.grid().ctx && b.grid().ctx && !a.grid().same_as(b.grid()))
    throw InvalidArgument("pgemm operands on different grids");
  if (a.col_dims() == b.row_dims()) {
    Tensor c = network::contract(a.tensor(), b.tensor(), a.col_pos(), b.row_pos());
    const int nr = static_cast<int>(a.row_pos().size());
    return BlockCyclicMatrix(c, detail::ranks_in_sorted(a.row_pos(), 0), detail::ranks_in_sorted(b.col_pos(), nr),
                             a.row_block(), b.col_block(), a.grid().ctx ? &a.grid() : nullptr);
  }
  // different factorisations of the contracted dimension: both as dense matrices
  Tensor ta = detail::canonical(a, {a.rows()}, {a.cols()});
  Tensor tb = detail::canonical(b, {b.rows()}, {b.cols()});
  Tensor c = network::contract(ta, tb, {1}, {0});
  return BlockCyclicMatrix(c, {0}, {1}, a.row_block(), b.col_block(), a.grid().ctx ? &a.grid() : nullptr);
}

/// linalg.hpp:270-342: the tensor of `shape` / `dist` whose coordinates at row_pos
/// (col_pos) flatten to the matrix row (column). One permutation (none when the
/// view already has that order), then a rebcast when the distribution differs.
inline Tensor matrix_to_tensor(const BlockCyclicMatrix& mat, Rank& ctx, IndexTuple shape, DistParams dist,
                               const std::vector<int>& row_pos, const std::vector<int>& col_pos) {
  (void)ctx;
  detail::check_partition(shape, row_pos, col_pos);
  std::vector<Dim> rd, cd;
  for (int p : row_pos) rd.push_back(shape.dims[p]);
  for (int p : col_pos) cd.push_back(shape.dims[p]);
  if (detail::product(rd) != mat.rows() || detail::product(cd) != mat.cols())
    throw InvalidArgument("tensor shape does not match matrix dimensions");
  Tensor src = mat.tensor();
  std::vector<int> srow = mat.row_pos(), scol = mat.col_pos();
  if (rd != mat.row_dims() || cd != mat.col_dims()) {  // regroup the digits
    src = detail::canonical(mat, rd, cd);
    srow.resize(rd.size());
    std::iota(srow.begin(), srow.end(), 0);
    scol.resize(cd.size());
    std::iota(scol.begin(), scol.end(), static_cast<int>(rd.size()));
  }
  std::vector<int> perm(shape.n_idx());  // perm[new] = old (ops.hpp:21-23)
  for (std::size_t i = 0; i < row_pos.size(); ++i) perm[row_pos[i]] = srow[i];
  for (std::size_t i = 0; i < col_pos.size(); ++i) perm[col_pos[i]] = scol[i];
  Tensor out = ops::permute(src, perm, shape.split);
  if (out.dist() != dist) out = ops::rebcast(out, dist);
  return out;
}

struct SvdResult {  // linalg.hpp:402-406
  BlockCyclicMatrix u;
  std::vector<double> s;  // descending
  BlockCyclicMatrix vh;
};

/// linalg.hpp:438-471: thin SVD of the matrix on the device (batched one-sided
/// Jacobi); a distributed matrix is gathered onto its root copy first; S on every
/// rank of the span.
inline SvdResult psvd(const BlockCyclicMatrix& a) {
  const Dim k = std::min(a.rows(), a.cols());
  SvdResult out;
  out.s.assign(k, 0.0);
  qtnh_tensor_t u, vh;
  check(qtnh_svd(a.tensor().h(), static_cast<int>(a.row_pos().size()), a.row_pos().data(),
                 static_cast<int>(a.col_pos().size()), a.col_pos().data(), k, QTNH_ABSORB_NONE, &u, &vh,
                 out.s.data()));
  Tensor tu = wrap(u, &a.tensor().ctx()), tv = wrap(vh, &a.tensor().ctx());
  const int nr = static_cast<int>(a.row_pos().size()), nc = static_cast<int>(a.col_pos().size());
  std::vector<int> ur(nr), vc(nc);
  std::iota(ur.begin(), ur.end(), 0);
  std::iota(vc.begin(), vc.end(), 1);
  const Grid* g = a.grid().ctx ? &a.grid() : nullptr;
  out.u = BlockCyclicMatrix(tu, ur, {nr}, a.row_block(), a.col_block(), g);
  out.vh = BlockCyclicMatrix(tv, {0}, vc, a.row_block(), a.col_block(), g);
  return out;
}

namespace detail {
// The factor with its singular index as ONE index of its tensor (psvd outputs
// already are); position of that index.
inline std::pair<Tensor, int> single_index(const BlockCyclicMatrix& m, bool cols) {
  const auto& pos = cols ? m.col_pos() : m.row_pos();
  if (pos.size() == 1) return {m.tensor(), pos[0]};
  Tensor t = cols ? canonical(m, m.row_dims(), {m.cols()}) : canonical(m, {m.rows()}, m.col_dims());
  return {t, cols ? static_cast<int>(m.row_pos().size()) : 0};
}
}  // namespace detail

/// linalg.hpp:473-505: keep the chi largest triplets, zero-pad to exactly chi.
inline SvdResult truncate_svd(const BlockCyclicMatrix& u, const std::vector<double>& s, const BlockCyclicMatrix& vh,
                              Dim chi) {
  if (chi < 1) throw InvalidArgument("chi must be positive");
  const Dim k = static_cast<Dim>(s.size());
  if (chi == k) return {u, s, vh};
  const Dim keep = std::min(chi, k);
  auto [tu, ui] = detail::single_index(u, true);
  auto [tv, vi] = detail::single_index(vh, false);
  auto resize = [&](Tensor t, int pos, Dim to) {
    auto sh = t.shape();
    if (pos < sh.split) throw PreconditionError("truncate_svd: the singular index is distributed");
    std::vector<Dim> cut = sh.local_dims(), pad;
    cut[pos - sh.split] = keep;
    if (keep < sh.dims[pos]) t = ops::slice_local_dims(t, cut);
    if (to > keep) {
      pad = cut;
      pad[pos - sh.split] = to;
      t = ops::pad_local_dims(t, pad);
    }
    return t;
  };
  SvdResult out;
  out.s.assign(chi, 0.0);
  std::copy(s.begin(), s.begin() + keep, out.s.begin());
  Tensor nu = resize(tu, ui, chi), nv = resize(tv, vi, chi);
  std::vector<int> urow, vcol;
  for (int i = 0; i < nu.shape().n_idx(); ++i)
    if (i != ui) urow.push_back(i);
  for (int i = 0; i < nv.shape().n_idx(); ++i)
    if (i != vi) vcol.push_back(i);
  const Grid* g = u.grid().ctx ? &u.grid() : nullptr;
  out.u = BlockCyclicMatrix(nu, urow, {ui}, u.row_block(), u.col_block(), g);
  out.vh = BlockCyclicMatrix(nv, {vi}, vcol, vh.row_block(), vh.col_block(), g);
  return out;
}

/// linalg.hpp:507-514: column c of U scaled by s[c]^power, in place.
inline void absorb_singular_left(BlockCyclicMatrix& u, const std::vector<double>& s, double power = 1.0) {
  auto [t, pos] = detail::single_index(u, true);
  std::vector<double> f(s.size());
  for (std::size_t c = 0; c < s.size(); ++c) f[c] = std::pow(s[c], power);
  Tensor nt = ops::scale_index(t, pos, f);
  std::vector<int> rows;
  for (int i = 0; i < nt.shape().n_idx(); ++i)
    if (i != pos) rows.push_back(i);
  u = BlockCyclicMatrix(nt, rows, {pos}, u.row_block(), u.col_block(), u.grid().ctx ? &u.grid() : nullptr);
}

/// linalg.hpp:516-523: row r of Vh scaled by s[r]^power, in place.
inline void absorb_singular_right(BlockCyclicMatrix& vh, const std::vector<double>& s, double power = 1.0) {
  auto [t, pos] = detail::single_index(vh, false);
  std::vector<double> f(s.size());
  for (std::size_t c = 0; c < s.size(); ++c) f[c] = std::pow(s[c], power);
  Tensor nt = ops::scale_index(t, pos, f);
  std::vector<int> cols;
  for (int i = 0; i < nt.shape().n_idx(); ++i)
    if (i != pos) cols.push_back(i);
  vh = BlockCyclicMatrix(nt, {pos}, cols, vh.row_block(), vh.col_block(), vh.grid().ctx ? &vh.grid() : nullptr);
}

/// Tensor-level split in one call (SPEC network::decompose): psvd -> truncate_svd
/// -> absorb, on the device.
enum class Absorb { none = QTNH_ABSORB_NONE, left = QTNH_ABSORB_LEFT, right = QTNH_ABSORB_RIGHT,
                    split = QTNH_ABSORB_SPLIT };
struct Svd {
  Tensor u, vh;
  std::vector<double> s;
};
inline Svd svd(const Tensor& t, const std::vector<int>& row_pos, const std::vector<int>& col_pos, Dim chi = 0,
               Absorb absorb = Absorb::none) {
  auto sh = t.shape();
  Dim m = 1, n = 1;
  for (int p : row_pos) m *= sh.dims[p];
  for (int p : col_pos) n *= sh.dims[p];
  Svd r;
  r.s.assign(chi > 0 ? chi : std::min(m, n), 0.0);
  qtnh_tensor_t u, vh;
  check(qtnh_svd(t.h(), static_cast<int>(row_pos.size()), row_pos.data(), static_cast<int>(col_pos.size()),
                 col_pos.data(), chi, static_cast<int>(absorb), &u, &vh, r.s.data()));
  r.u = wrap(u, &t.ctx());
  r.vh = wrap(vh, &t.ctx());
  return r;
}
}  // namespace linalg

namespace gates {  // contract(state, gate) + permute back, in place (copy-on-write)
inline void apply(Tensor& state, const std::vector<int>& targets, const std::vector<Complex>& gate,
                  bool diagonal = false) {
  check(qtnh_gate_apply(state.h(), static_cast<int>(targets.size()), targets.data(),
                        reinterpret_cast<const double*>(gate.data()), diagonal ? 1 : 0));
}
/// The gate as a replicated tensor (outputs; inputs) of any variant: a diagonal gate
/// runs the diagonal kernel from its stored diagonal (no exchange even on distributed
/// targets), an identity does nothing, a swap exchanges the two targets.
inline void apply(Tensor& state, const std::vector<int>& targets, const Tensor& gate) {
  check(qtnh_gate_apply_tensor(state.h(), static_cast<int>(targets.size()), targets.data(), gate.h()));
}
inline void swap_indices(Tensor& state, int a, int b) { check(qtnh_swap_indices(state.h(), a, b)); }
inline void qft(Tensor& state, bool swaps = true) { check(qtnh_qft(state.h(), swaps ? 1 : 0)); }
}  // namespace gates

namespace mps {  // one brickwork layer of two-site updates
struct LayerResult {
  std::vector<std::vector<double>> s;  // kept singular values per pair
  std::vector<double> norm2;           // ||theta||^2 per pair
};
/// sites[q], sites[q+1] for each q in `left_sites` are replaced by U S and Vh.
inline LayerResult apply_layer(std::vector<Tensor>& sites, const std::vector<int>& left_sites,
                               const std::vector<Complex>& gate4x4, Dim chi) {
  const int n = static_cast<int>(left_sites.size());
  std::vector<qtnh_tensor_t> l(n), r(n), nl(n), nr(n);
  for (int i = 0; i < n; ++i) {
    l[i] = sites.at(left_sites[i]).h();
    r[i] = sites.at(left_sites[i] + 1).h();
  }
  std::vector<double> s(static_cast<std::size_t>(n) * chi), nrm(n);
  std::vector<int64_t> keep(n);
  check(qtnh_mps_apply_layer(n, l.data(), r.data(), reinterpret_cast<const double*>(gate4x4.data()), chi, nl.data(),
                             nr.data(), s.data(), keep.data(), nrm.data()));
  LayerResult out;
  for (int i = 0; i < n; ++i) {
    Rank* ctx = &sites[left_sites[i]].ctx();
    sites[left_sites[i]] = wrap(nl[i], ctx);
    sites[left_sites[i] + 1] = wrap(nr[i], ctx);
    out.s.emplace_back(s.begin() + i * chi, s.begin() + i * chi + keep[i]);
    out.norm2.push_back(nrm[i]);
  }
  return out;
}
}  // namespace mps

}  // namespace qtnh_b200
