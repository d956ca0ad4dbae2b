// Reference oracle driver -- TEST INFRASTRUCTURE ONLY.
//
// Compiles the UNMODIFIED reference headers (/root/reference/proj/include/qtnh,
// header-only C++20) together with the prototype shims in oracle/shim into
// oracle/_ref/libqtnh_ref.so, and exposes a flat C ABI so that tests/, bench.py's
// cpu_baseline leg and __graft_entry__.smoke() can call the real reference as the
// parity checker. Nothing in the product path (paper_2505_06119_b200/) links or
// loads this library.
//
// Every entry point runs the reference's own SPMD runtime (qtnh::World, one thread
// per simulated rank, runtime.hpp:263-299) and its public operations:
//   ops::permute / rebcast / scatter_index / gather_index  (ops.hpp:27-144)
//   ops::slice_local_dims / pad_local_dims                  (ops.hpp:166-230)
//   linalg::tensor_to_matrix / pgemm / matrix_to_tensor     (linalg.hpp:208,347,273)
//   linalg::psvd / truncate_svd / absorb_singular_*         (linalg.hpp:441-523)
// Tensors cross this ABI as global row-major vectors of interleaved (re, im)
// doubles, the layout of Tensor::to_global_vector (tensor.hpp:341-371).

#include <chrono>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "qtnh/linalg.hpp"

using namespace qtnh;

extern "C" void scipy_openblas_set_num_threads(int);

namespace {

thread_local std::string g_err;
thread_local long long g_info = 0;

int fail(const std::exception& e) {
  g_err = e.what();
  g_info = 0;
  if (auto* r = dynamic_cast<const ResourceError*>(&e)) { g_info = r->required_ranks; return 2; }
  if (dynamic_cast<const InvalidArgument*>(&e)) return 1;
  if (dynamic_cast<const ProtocolError*>(&e)) return 3;
  if (auto* n = dynamic_cast<const NumericalError*>(&e)) { g_info = n->info; return 4; }
  if (dynamic_cast<const PreconditionError*>(&e)) return 5;
  if (dynamic_cast<const DegenerateStateError*>(&e)) return 6;
  if (dynamic_cast<const AbortedError*>(&e)) return 7;
  return 8;
}

std::vector<Complex> to_cvec(const double* p, Dim n) {
  std::vector<Complex> v(n);
  for (Dim i = 0; i < n; ++i) v[i] = {p[2 * i], p[2 * i + 1]};
  return v;
}

void from_cvec(const std::vector<Complex>& v, double* p) {
  for (std::size_t i = 0; i < v.size(); ++i) {
    p[2 * i] = v[i].real();
    p[2 * i + 1] = v[i].imag();
  }
}

IndexTuple make_shape(int nd, const int64_t* dims, int split) {
  return IndexTuple(std::vector<Dim>(dims, dims + nd), split);
}

DistParams make_dist(const int64_t* d) {
  DistParams p;
  if (d) { p.stretch = d[0]; p.cycles = d[1]; p.offset = d[2]; }
  return p;
}

struct OutMeta {
  double* out;
  int64_t* dims;
  int* split;
  int64_t* dist;
  std::mutex mu;
  void capture(const Tensor& t) {
    // The first span rank (rank == offset) reports; to_global_vector is
    // span-collective, so every span rank must call it (tensor.hpp:341-371).
    auto g = t.to_global_vector();
    if (t.in_span() && t.ctx().rank() == t.dist().offset) {
      std::lock_guard<std::mutex> lk(mu);
      if (out) from_cvec(g, out);
      if (dims) for (int i = 0; i < t.shape().n_idx(); ++i) dims[i] = t.shape().dims[i];
      if (split) *split = t.shape().split;
      if (dist) { dist[0] = t.dist().stretch; dist[1] = t.dist().cycles; dist[2] = t.dist().offset; }
    }
  }
};

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

}  // namespace

extern "C" {

int qref_last_error(char* buf, int len) {
  if (buf && len > 0) {
    std::strncpy(buf, g_err.c_str(), len - 1);
    buf[len - 1] = 0;
  }
  return static_cast<int>(g_err.size());
}
long long qref_last_info() { return g_info; }
void qref_set_threads(int n) { scipy_openblas_set_num_threads(n); }

// ---- RNG (common.hpp:83-146) -------------------------------------------------
uint64_t qref_hash_counter(uint64_t seed, uint64_t k0, uint64_t k1, uint64_t k2) {
  return hash_counter(seed, k0, k1, k2);
}
/// `count` complex numbers from one sequential Rng(seed) via next_complex_normal.
void qref_rng_complex_normals(uint64_t seed, int64_t count, double* out) {
  Rng rng(seed);
  for (int64_t i = 0; i < count; ++i) {
    Complex c = rng.next_complex_normal();
    out[2 * i] = c.real();
    out[2 * i + 1] = c.imag();
  }
}

// ---- structural ops -----------------------------------------------------------
int qref_permute(int world, int nd, const int64_t* dims, int split, const int64_t* dist,
                 const double* in, const int* perm, int new_split, double* out,
                 int64_t* out_dims, int* out_split, int64_t* out_dist) {
  return guarded([&] {
    IndexTuple shape = make_shape(nd, dims, split);
    auto global = to_cvec(in, shape.total_size());
    std::vector<int> p(perm, perm + nd);
    OutMeta om{out, out_dims, out_split, out_dist, {}};
    World w(world);
    w.run([&](Rank& rk) {
      Tensor t = Tensor::from_global(rk, shape, make_dist(dist), global);
      om.capture(ops::permute(t, p, new_split));
    });
  });
}

int qref_rebcast(int world, int nd, const int64_t* dims, int split, const int64_t* dist,
                 const double* in, const int64_t* new_dist, double* out, int64_t* out_dist) {
  return guarded([&] {
    IndexTuple shape = make_shape(nd, dims, split);
    auto global = to_cvec(in, shape.total_size());
    OutMeta om{out, nullptr, nullptr, out_dist, {}};
    World w(world);
    w.run([&](Rank& rk) {
      Tensor t = Tensor::from_global(rk, shape, make_dist(dist), global);
      om.capture(ops::rebcast(t, make_dist(new_dist)));
    });
  });
}

/// op: 0 = scatter_index(pos), 1 = gather_index(pos).
int qref_scatter_gather(int world, int op, int nd, const int64_t* dims, int split,
                        const int64_t* dist, const double* in, int pos, double* out,
                        int64_t* out_dims, int* out_split) {
  return guarded([&] {
    IndexTuple shape = make_shape(nd, dims, split);
    auto global = to_cvec(in, shape.total_size());
    OutMeta om{out, out_dims, out_split, nullptr, {}};
    World w(world);
    w.run([&](Rank& rk) {
      Tensor t = Tensor::from_global(rk, shape, make_dist(dist), global);
      om.capture(op == 0 ? ops::scatter_index(t, pos) : ops::gather_index(t, pos));
    });
  });
}

/// op: 0 = slice_local_dims, 1 = pad_local_dims; new_local has n_local entries.
int qref_slice_pad(int world, int op, int nd, const int64_t* dims, int split,
                   const int64_t* dist, const double* in, const int64_t* new_local,
                   double* out) {
  return guarded([&] {
    IndexTuple shape = make_shape(nd, dims, split);
    auto global = to_cvec(in, shape.total_size());
    std::vector<Dim> nl(new_local, new_local + shape.n_local());
    OutMeta om{out, nullptr, nullptr, nullptr, {}};
    World w(world);
    w.run([&](Rank& rk) {
      Tensor t = Tensor::from_global(rk, shape, make_dist(dist), global);
      om.capture(op == 0 ? ops::slice_local_dims(t, nl) : ops::pad_local_dims(t, nl));
    });
  });
}

// ---- contraction -----------------------------------------------------------------
// The reference ships no contract(); SPEC.md:361-369 composes it from
// tensor_to_matrix (linalg.hpp:208) -> pgemm (:347) -> matrix_to_tensor (:273)
// with result order "open(a) then open(b)" and DistParams of the
// first operand. Result split = number of distributed indices of
// `a` left open (they stay leftmost); b's open indices are local.
namespace {
Tensor contract_ref(const Tensor& a, const Tensor& b, const std::vector<int>& apos,
                    const std::vector<int>& bpos, double* t_ms) {
  Rank& ctx = a.ctx();
  const auto& sa = a.shape();
  const auto& sb = b.shape();
  std::vector<int> a_open, b_open;
  std::vector<bool> ca(sa.n_idx(), false), cb(sb.n_idx(), false);
  for (int p : apos) ca.at(p) = true;
  for (int p : bpos) cb.at(p) = true;
  for (int i = 0; i < sa.n_idx(); ++i) if (!ca[i]) a_open.push_back(i);
  for (int i = 0; i < sb.n_idx(); ++i) if (!cb[i]) b_open.push_back(i);
  Dim K = 1;
  for (std::size_t i = 0; i < apos.size(); ++i) {
    if (sa.dims[apos[i]] != sb.dims[bpos[i]]) throw InvalidArgument("contracted dims differ");
    K *= sa.dims[apos[i]];
  }
  std::vector<int> all(ctx.size());
  for (int i = 0; i < ctx.size(); ++i) all[i] = i;
  auto grid = linalg::Grid::make(ctx, all);
  auto t0 = std::chrono::steady_clock::now();
  auto ma = linalg::tensor_to_matrix(a, a_open, apos, &grid, 0, K);
  auto mb = linalg::tensor_to_matrix(b, bpos, b_open, &grid, K, 0);
  auto t1 = std::chrono::steady_clock::now();
  auto mc = linalg::pgemm(ma, mb);
  auto t2 = std::chrono::steady_clock::now();
  std::vector<Dim> cdims;
  int csplit = 0;
  for (int p : a_open) { cdims.push_back(sa.dims[p]); if (p < sa.split) ++csplit; }
  for (int p : b_open) cdims.push_back(sb.dims[p]);
  std::vector<int> rows, cols;
  for (std::size_t i = 0; i < a_open.size(); ++i) rows.push_back(static_cast<int>(i));
  for (std::size_t i = 0; i < b_open.size(); ++i) cols.push_back(static_cast<int>(a_open.size() + i));
  Tensor c = linalg::matrix_to_tensor(mc, ctx, IndexTuple(cdims, csplit), a.dist(), rows, cols);
  auto t3 = std::chrono::steady_clock::now();
  if (t_ms && ctx.rank() == 0) {
    auto ms = [](auto x, auto y) { return std::chrono::duration<double, std::milli>(y - x).count(); };
    t_ms[0] = ms(t0, t1);
    t_ms[1] = ms(t1, t2);
    t_ms[2] = ms(t2, t3);
    t_ms[3] = ms(t0, t3);
  }
  return c;
}
}  // namespace

int qref_contract(int world, int nda, const int64_t* dims_a, int split_a, const int64_t* dist_a,
                  const double* in_a, int ndb, const int64_t* dims_b, int split_b,
                  const int64_t* dist_b, const double* in_b, int npairs, const int* a_pos,
                  const int* b_pos, double* out, int64_t* out_dims, int* out_split,
                  double* t_ms) {
  return guarded([&] {
    IndexTuple sa = make_shape(nda, dims_a, split_a), sb = make_shape(ndb, dims_b, split_b);
    auto ga = to_cvec(in_a, sa.total_size());
    auto gb = to_cvec(in_b, sb.total_size());
    std::vector<int> ap(a_pos, a_pos + npairs), bp(b_pos, b_pos + npairs);
    OutMeta om{out, out_dims, out_split, nullptr, {}};
    World w(world);
    w.run([&](Rank& rk) {
      Tensor a = Tensor::from_global(rk, sa, make_dist(dist_a), ga);
      Tensor b = Tensor::from_global(rk, sb, make_dist(dist_b), gb);
      om.capture(contract_ref(a, b, ap, bp, t_ms));
    });
  });
}

// ---- gate application as contraction + permute back ------------------------------
namespace {
Tensor apply_gate_ref(const Tensor& state, int k, const int* qubits, const Tensor& gate) {
  int n = state.shape().n_idx();
  std::vector<int> apos(qubits, qubits + k), bpos(k);
  for (int j = 0; j < k; ++j) bpos[j] = k + j;  // gate indices (out_1..out_k, in_1..in_k)
  Tensor c = contract_ref(state, gate, apos, bpos, nullptr);
  // c = (state open indices in order, gate out_1..out_k): move out_j back to qubits[j].
  std::vector<int> perm(n), opens;
  std::vector<int> slot(n, -1);
  for (int j = 0; j < k; ++j) slot[qubits[j]] = j;
  int next_open = 0;
  for (int p = 0; p < n; ++p) perm[p] = slot[p] >= 0 ? (n - k) + slot[p] : next_open++;
  return ops::permute(c, perm, state.shape().split);
}

std::vector<Complex> qft_gate_h() {
  double r = 1.0 / std::sqrt(2.0);
  return {{r, 0}, {r, 0}, {r, 0}, {-r, 0}};
}
std::vector<Complex> qft_gate_cp(double theta) {
  std::vector<Complex> g(16, Complex{0, 0});
  g[0] = g[5] = g[10] = 1.0;
  g[15] = std::polar(1.0, theta);
  return g;
}
}  // namespace

int qref_gate(int world, int n, int split, const int64_t* dist, const double* in, int k,
              const int* qubits, const double* gate, double* out) {
  return guarded([&] {
    IndexTuple shape(std::vector<Dim>(n, 2), split);
    auto global = to_cvec(in, shape.total_size());
    auto g = to_cvec(gate, Dim(1) << (2 * k));
    OutMeta om{out, nullptr, nullptr, nullptr, {}};
    World w(world);
    w.run([&](Rank& rk) {
      Tensor s = Tensor::from_global(rk, shape, make_dist(dist), global);
      Tensor gt = Tensor::from_global(rk, IndexTuple(std::vector<Dim>(2 * k, 2), 0), {}, g);
      om.capture(apply_gate_ref(s, k, qubits, gt));
    });
  });
}

/// Statevector QFT: for j = 0..n-1, H on
/// qubit j, then CP(2*pi/2^m) between qubit j and qubit j+m-1 for m = 2..n-j;
/// then (optionally) SWAP(j, n-1-j) realised as a permutation (contraction with a
/// swap tensor is a pure index exchange, tensor.hpp:157-164). Input state is
/// `in` (global, split `split`). gate_limit < 0 applies all gates.
int qref_qft(int world, int n, int split, const double* in, int swaps, int gate_limit,
             double* out, double* t_ms) {
  return guarded([&] {
    IndexTuple shape(std::vector<Dim>(n, 2), split);
    auto global = to_cvec(in, shape.total_size());
    OutMeta om{out, nullptr, nullptr, nullptr, {}};
    World w(world);
    w.run([&](Rank& rk) {
      Tensor s = Tensor::from_global(rk, shape, {}, global);
      Tensor h = Tensor::from_global(rk, IndexTuple({2, 2}, 0), {}, qft_gate_h());
      auto t0 = std::chrono::steady_clock::now();
      int applied = 0;
      auto budget = [&] { return gate_limit < 0 || applied < gate_limit; };
      for (int j = 0; j < n && budget(); ++j) {
        int q1[1] = {j};
        s = apply_gate_ref(s, 1, q1, h);
        ++applied;
        for (int m = 2; m <= n - j && budget(); ++m) {
          double theta = 2.0 * M_PI / std::ldexp(1.0, m);
          Tensor cp = Tensor::from_global(rk, IndexTuple({2, 2, 2, 2}, 0), {}, qft_gate_cp(theta));
          int q2[2] = {j + m - 1, j};
          s = apply_gate_ref(s, 2, q2, cp);
          ++applied;
        }
      }
      if (swaps) {
        for (int j = 0; j < n / 2 && budget(); ++j) {
          std::vector<int> perm(n);
          for (int p = 0; p < n; ++p) perm[p] = p;
          std::swap(perm[j], perm[n - 1 - j]);
          s = ops::permute(s, perm, split);
          ++applied;
        }
      }
      auto t1 = std::chrono::steady_clock::now();
      if (t_ms && rk.rank() == 0) t_ms[0] = std::chrono::duration<double, std::milli>(t1 - t0).count();
      om.capture(s);
    });
  });
}

// ---- serialization (tensor.hpp:373-446): QTNHTEN1 files ----------------------------
int qref_save(int world, int nd, const int64_t* dims, int split, const int64_t* dist, const double* in,
              const char* path) {
  return guarded([&] {
    IndexTuple shape = make_shape(nd, dims, split);
    auto global = to_cvec(in, shape.total_size());
    std::string p(path);
    World w(world);
    w.run([&](Rank& rk) {
      Tensor t = Tensor::from_global(rk, shape, make_dist(dist), global);
      t.save(p);
    });
  });
}

/// Loads on World(world); writes dims (up to 64), split, dist and the global vector.
int qref_load(int world, const char* path, int64_t* dims, int* nd, int* split, int64_t* dist, double* out,
              int64_t cap) {
  return guarded([&] {
    std::string p(path);
    std::mutex mu;
    World w(world);
    w.run([&](Rank& rk) {
      Tensor t = Tensor::load(rk, p);
      auto g = t.to_global_vector();
      if (t.in_span() && rk.rank() == t.dist().offset) {
        std::lock_guard<std::mutex> lk(mu);
        *nd = t.shape().n_idx();
        *split = t.shape().split;
        for (int i = 0; i < t.shape().n_idx(); ++i) dims[i] = t.shape().dims[i];
        dist[0] = t.dist().stretch;
        dist[1] = t.dist().cycles;
        dist[2] = t.dist().offset;
        if (static_cast<int64_t>(g.size()) > cap) throw Error("output capacity too small");
        from_cvec(g, out);
      }
    });
  });
}

// ---- SVD / truncation / absorption (linalg.hpp:402-523) -------------------------
/// a: m x n ROW-major. Outputs ROW-major u (m x chi), s (chi), vh (chi x n).
/// chi <= 0 means no truncation (chi = min(m, n)). absorb: 0 none, 1 left
/// (U *= s), 2 right (Vh *= s), 3 split (both by sqrt(s)).
int qref_svd(int world, int64_t m, int64_t n, const double* a, int64_t chi, int absorb,
             double* u, double* s, double* vh, double* t_ms) {
  return guarded([&] {
    std::vector<Complex> colmaj(m * n);
    for (int64_t r = 0; r < m; ++r)
      for (int64_t c = 0; c < n; ++c) colmaj[r + c * m] = {a[2 * (r * n + c)], a[2 * (r * n + c) + 1]};
    int64_t k = std::min(m, n);
    int64_t keep = chi > 0 ? chi : k;
    std::mutex mu;
    World w(world);
    w.run([&](Rank& rk) {
      std::vector<int> all(rk.size());
      for (int i = 0; i < rk.size(); ++i) all[i] = i;
      auto grid = linalg::Grid::make(rk, all);
      auto mat = linalg::BlockCyclicMatrix::from_global(grid, m, n, std::max<int64_t>(1, m / 2),
                                                        std::max<int64_t>(1, n / 2), colmaj);
      auto t0 = std::chrono::steady_clock::now();
      auto res = linalg::psvd(mat);
      auto t1 = std::chrono::steady_clock::now();
      auto tr = linalg::truncate_svd(res.u, res.s, res.vh, keep);
      if (absorb == 1) linalg::absorb_singular_left(tr.u, tr.s, 1.0);
      if (absorb == 2) linalg::absorb_singular_right(tr.vh, tr.s, 1.0);
      if (absorb == 3) {
        linalg::absorb_singular_left(tr.u, tr.s, 0.5);
        linalg::absorb_singular_right(tr.vh, tr.s, 0.5);
      }
      auto t2 = std::chrono::steady_clock::now();
      auto gu = tr.u.gather_global();
      auto gvh = tr.vh.gather_global();
      if (rk.rank() == 0) {
        std::lock_guard<std::mutex> lk(mu);
        for (int64_t r = 0; r < m; ++r)
          for (int64_t c = 0; c < keep; ++c) {
            u[2 * (r * keep + c)] = gu[r + c * m].real();
            u[2 * (r * keep + c) + 1] = gu[r + c * m].imag();
          }
        for (int64_t r = 0; r < keep; ++r)
          for (int64_t c = 0; c < n; ++c) {
            vh[2 * (r * n + c)] = gvh[r + c * keep].real();
            vh[2 * (r * n + c) + 1] = gvh[r + c * keep].imag();
          }
        for (int64_t i = 0; i < keep; ++i) s[i] = tr.s[i];
        if (t_ms) {
          t_ms[0] = std::chrono::duration<double, std::milli>(t1 - t0).count();
          t_ms[1] = std::chrono::duration<double, std::milli>(t2 - t1).count();
        }
      }
    });
  });
}

}  // extern "C"
