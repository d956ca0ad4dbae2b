// qtnh_b200.hpp -- header-only C++ layer over the C ABI (qtnh_b200.h) that keeps
// the reference's C++ API shape for the hot path, so existing callers of
//   qtnh::World / Rank / Tensor / ops::permute / ops::rebcast / ops::scatter_index /
//   ops::gather_index / linalg contraction
// (/root/reference/proj/include/qtnh/*.hpp) switch by changing the namespace:
//   namespace qtnh = qtnh_b200;
// Errors come back as the same exception classes (common.hpp:31-74).
#pragma once

#include <complex>
#include <cstdint>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "qtnh_b200.h"

namespace qtnh_b200 {

using Complex = std::complex<double>;
using Dim = std::int64_t;

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
  IndexTuple(std::vector<Dim> d, int s) : dims(std::move(d)), split(s) {}
  int n_idx() const { return static_cast<int>(dims.size()); }
  Dim total_size() const {
    Dim n = 1;
    for (Dim d : dims) n *= d;
    return n;
  }
};

struct DistParams {  // indexing.hpp:84-101
  Dim stretch = 1, cycles = 1, offset = 0;
};

class Rank {
 public:
  int rank() const { return qtnh_rank_id(h_); }
  qtnh_rank_t handle() const { return h_; }

 private:
  friend class World;
  explicit Rank(qtnh_rank_t h) : h_(h) {}
  qtnh_rank_t h_;
};

class World {  // runtime.hpp:243-303
 public:
  explicit World(int n, const std::vector<int>& devices = {}) : n_(n) {
    check(qtnh_world_create_local(n, devices.empty() ? nullptr : devices.data(), &w_));
  }
  ~World() { qtnh_world_destroy(w_); }
  World(const World&) = delete;
  World& operator=(const World&) = delete;
  int size() const { return n_; }

  /// One host thread per rank; rethrows the originating failure (runtime.hpp:263-299).
  void run(const std::function<void(Rank&)>& body) {
    std::vector<std::thread> ts;
    std::vector<std::exception_ptr> errs(n_);
    for (int r = 0; r < n_; ++r)
      ts.emplace_back([&, r] {
        qtnh_rank_t h = nullptr;
        try {
          check(qtnh_rank_bind(w_, r, &h));
          Rank rk(h);
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
  int n_;
  qtnh_world_t w_ = nullptr;
};

class Tensor {  // tensor.hpp:53-695 (dense)
 public:
  Tensor() = default;

  static Tensor dense(Rank& r, const IndexTuple& s, DistParams d, const std::vector<Complex>& local) {
    qtnh_tensor_t h;
    int64_t dd[3] = {d.stretch, d.cycles, d.offset};
    check(qtnh_tensor_dense(r.handle(), s.n_idx(), s.dims.data(), s.split, dd,
                            local.empty() ? nullptr : reinterpret_cast<const double*>(local.data()), &h));
    return Tensor(h);
  }
  static Tensor from_global(Rank& r, const IndexTuple& s, DistParams d, const std::vector<Complex>& global) {
    if (static_cast<Dim>(global.size()) != s.total_size()) throw InvalidArgument("global element count mismatch");
    qtnh_tensor_t h;
    int64_t dd[3] = {d.stretch, d.cycles, d.offset};
    check(qtnh_tensor_from_global(r.handle(), s.n_idx(), s.dims.data(), s.split, dd,
                                  reinterpret_cast<const double*>(global.data()), &h));
    return Tensor(h);
  }

  // Tensor::identity / swap_tensor (tensor.hpp:144-164), dense on the device
  static Tensor identity(Rank& r, const IndexTuple& s, DistParams d, const std::vector<int>& in_pos,
                         const std::vector<int>& out_pos) {
    return paired(r, s, d, in_pos, out_pos, 0);
  }
  static Tensor swap_tensor(Rank& r, const IndexTuple& s, DistParams d, const std::vector<int>& in_pos,
                            const std::vector<int>& out_pos) {
    return paired(r, s, d, in_pos, out_pos, 1);
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
  Dim span() const { return qtnh_tensor_span(h()); }
  bool in_span() const { return qtnh_tensor_in_span(h()) != 0; }
  Dim my_block() const { return qtnh_tensor_my_block(h()); }

  std::vector<Complex> local_data() const {
    std::vector<Complex> v(in_span() ? qtnh_tensor_local_size(h()) : 0);
    if (!v.empty()) check(qtnh_tensor_download_local(h(), reinterpret_cast<double*>(v.data())));
    return v;
  }
  std::vector<Complex> to_global_vector() const {
    if (!in_span()) return {};
    std::vector<Complex> v(shape().total_size());
    check(qtnh_tensor_to_global(h(), reinterpret_cast<double*>(v.data())));
    return v;
  }
  qtnh_tensor_t h() const { return p_.get(); }

  // serialization (tensor.hpp:388-446), QTNHTEN1 byte-identical to the reference
  void save(const std::string& path) const { check(qtnh_tensor_save(h(), path.c_str())); }
  static Tensor paired(Rank& r, const IndexTuple& s, DistParams d, const std::vector<int>& in_pos,
                       const std::vector<int>& out_pos, int crossed) {
    if (in_pos.size() != out_pos.size()) throw InvalidArgument("input/output position lists differ in length");
    qtnh_tensor_t o;
    int64_t dd[3] = {d.stretch, d.cycles, d.offset};
    check(qtnh_tensor_paired(r.handle(), s.n_idx(), s.dims.data(), s.split, dd, static_cast<int>(in_pos.size()),
                             in_pos.data(), out_pos.data(), crossed, &o));
    return Tensor(o);
  }
  static Tensor load(Rank& r, const std::string& path) {
    qtnh_tensor_t o;
    check(qtnh_tensor_load(r.handle(), path.c_str(), &o));
    return Tensor(o);
  }

 private:
  explicit Tensor(qtnh_tensor_t h) : p_(h, [](qtnh_tensor_t x) { qtnh_tensor_free(x); }) {}
  std::shared_ptr<qtnh_tensor_s> p_;
  friend Tensor wrap(qtnh_tensor_t);
};

inline Tensor wrap(qtnh_tensor_t h) { return Tensor(h); }

namespace ops {  // ops.hpp
inline Tensor permute(const Tensor& t, const std::vector<int>& perm, int new_split) {
  qtnh_tensor_t o;
  check(qtnh_permute(t.h(), perm.data(), new_split, &o));
  return wrap(o);
}
inline Tensor rebcast(const Tensor& t, DistParams d) {
  qtnh_tensor_t o;
  int64_t dd[3] = {d.stretch, d.cycles, d.offset};
  check(qtnh_rebcast(t.h(), dd, &o));
  return wrap(o);
}
inline Tensor scatter_index(const Tensor& t, int pos) {
  qtnh_tensor_t o;
  check(qtnh_scatter_index(t.h(), pos, &o));
  return wrap(o);
}
inline Tensor gather_index(const Tensor& t, int pos) {
  qtnh_tensor_t o;
  check(qtnh_gather_index(t.h(), pos, &o));
  return wrap(o);
}
// remap::tensor_to_tensor (remap.hpp:106): axis_map[src] = dst position
inline Tensor tensor_to_tensor(const Tensor& t, const IndexTuple& dst, DistParams d, const std::vector<int>& axis_map) {
  qtnh_tensor_t o;
  int64_t dd[3] = {d.stretch, d.cycles, d.offset};
  check(qtnh_remap(t.h(), axis_map.data(), dst.n_idx(), dst.dims.data(), dst.split, dd, &o));
  return wrap(o);
}
inline Tensor slice_local_dims(const Tensor& t, const std::vector<Dim>& new_local) {  // ops.hpp:166
  qtnh_tensor_t o;
  check(qtnh_slice_local_dims(t.h(), new_local.data(), &o));
  return wrap(o);
}
inline Tensor pad_local_dims(const Tensor& t, const std::vector<Dim>& new_local) {  // ops.hpp:201
  qtnh_tensor_t o;
  check(qtnh_pad_local_dims(t.h(), new_local.data(), &o));
  return wrap(o);
}
inline Tensor conj(const Tensor& t) {  // ops.hpp:147
  qtnh_tensor_t o;
  check(qtnh_conj(t.h(), &o));
  return wrap(o);
}
inline Tensor scale(const Tensor& t, Complex a) {  // ops.hpp:155
  qtnh_tensor_t o;
  check(qtnh_scale(t.h(), a.real(), a.imag(), &o));
  return wrap(o);
}
}  // namespace ops

namespace remap {  // remap.hpp
using ops::tensor_to_tensor;
}  // namespace remap

namespace linalg {  // psvd -> truncate_svd -> absorb_singular_* (linalg.hpp:441-523)
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
  r.u = wrap(u);
  r.vh = wrap(vh);
  return r;
}
}  // namespace linalg

namespace gates {  // contract(state, gate) + permute back, in place (copy-on-write)
inline void apply(Tensor& state, const std::vector<int>& targets, const std::vector<Complex>& gate,
                  bool diagonal = false) {
  check(qtnh_gate_apply(state.h(), static_cast<int>(targets.size()), targets.data(),
                        reinterpret_cast<const double*>(gate.data()), diagonal ? 1 : 0));
}
inline void swap_indices(Tensor& state, int a, int b) { check(qtnh_swap_indices(state.h(), a, b)); }
inline void qft(Tensor& state, bool swaps = true) { check(qtnh_qft(state.h(), swaps ? 1 : 0)); }
}  // namespace gates

namespace network {  // SPEC.md:361-369, result order SPEC.md:408
inline Tensor contract(const Tensor& a, const Tensor& b, const std::vector<int>& a_pos,
                       const std::vector<int>& b_pos) {
  if (a_pos.size() != b_pos.size()) throw InvalidArgument("contracted position lists differ in length");
  qtnh_tensor_t o;
  check(qtnh_contract(a.h(), b.h(), static_cast<int>(a_pos.size()), a_pos.data(), b_pos.data(), &o));
  return wrap(o);
}
}  // namespace network

}  // namespace qtnh_b200
