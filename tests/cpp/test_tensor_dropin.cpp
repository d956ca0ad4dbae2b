// Tensor / ops / indexing call sequences, compiled UNCHANGED against either
// implementation (like test_linalg_dropin.cpp):
//   * the reference headers (/root/reference/proj/include/qtnh):
//     `make -C oracle dropin` -> tests/golden/tensor_dropin_ref.txt
//   * the B200 drop-in (include/qtnh_b200.hpp, -DQTNH_B200): namespace swap only.
// It walks the API the reference's own structural tests walk (test_tensor.cpp,
// test_ops.cpp): layout arithmetic, dense distribution and element lookup, the
// storage variants (symmetric, diagonal, identity, swap), to_dense, variant-keeping
// rebcast / conj / scale, every structural op on every variant, the QTNHTEN1 files
// of every variant (their BYTES are recorded), error classes and messages.
// Every rank records what it sees under "<case>.<rank>.<what>"; the sorted
// records go to argv[1] and the pytest compares the two files EXACTLY.
#include <unistd.h>

#include <cmath>
#include <complex>
#include <cstdint>
#include <cstdio>
#include <fstream>
#include <functional>
#include <map>
#include <mutex>
#include <sstream>
#include <string>
#include <vector>

#ifdef QTNH_B200
#include "qtnh_b200.hpp"
namespace qtnh = qtnh_b200;
#else
#include <qtnh/ops.hpp>
#include <qtnh/runtime.hpp>
#include <qtnh/tensor.hpp>
#endif

using qtnh::Complex;
using qtnh::Coords;
using qtnh::Dim;
using qtnh::DistParams;
using qtnh::IndexTuple;
using qtnh::Rank;
using qtnh::Tensor;
using qtnh::Variant;
using qtnh::World;
namespace ops = qtnh::ops;

namespace {

std::mutex g_mu;
std::map<std::string, std::string> g_rec;

void rec(const std::string& key, const std::string& value) {
  std::lock_guard<std::mutex> lk(g_mu);
  g_rec[key] = value;
}
std::string key(const char* c, Rank& rk, const char* what) {
  return std::string(c) + "." + std::to_string(rk.rank()) + "." + what;
}
std::string str(const std::vector<Complex>& v) {
  std::ostringstream os;
  os << v.size() << ":";
  char buf[64];
  for (const auto& c : v) {
    std::snprintf(buf, sizeof buf, " %.17g,%.17g", c.real(), c.imag());
    os << buf;
  }
  return os.str();
}
std::string str(Complex c) { return str(std::vector<Complex>{c}); }
template <class T>
std::string ints(const std::vector<T>& v) {
  std::ostringstream os;
  for (auto x : v) os << " " << x;
  return os.str();
}
std::string describe(const Tensor& t) {
  std::ostringstream os;
  os << qtnh::variant_name(t.variant()) << " " << t.shape().str() << " str=" << t.dist().stretch
     << " cyc=" << t.dist().cycles << " off=" << t.dist().offset << " span=" << t.span() << " in=" << t.in_span();
  if (t.in_span()) os << " block=" << t.my_block() << " canon=" << t.is_canonical_holder();
  os << " stored=" << t.local_data().size();
  return os.str();
}
std::string file_hex(const std::string& path) {
  std::ifstream is(path, std::ios::binary);
  std::ostringstream os;
  char c;
  static const char* hex = "0123456789abcdef";
  while (is.get(c)) os << hex[(static_cast<unsigned char>(c) >> 4) & 15] << hex[static_cast<unsigned char>(c) & 15];
  return os.str();
}
// values with signed zeros, denormal-free and distinct
std::vector<Complex> ramp(std::size_t n, double a, double b) {
  std::vector<Complex> v(n);
  for (std::size_t i = 0; i < n; ++i) v[i] = Complex(a * (double(i) + 1.0), b / (double(i) + 2.0));
  return v;
}
template <class F>
void expect_error(const std::string& k, F&& f) {
  try {
    f();
    rec(k, "no error");
  } catch (const qtnh::ResourceError& e) {
    rec(k, std::string("ResourceError[") + std::to_string(e.required_ranks) + "] " + e.what());
  } catch (const qtnh::InvalidArgument& e) {
    rec(k, std::string("InvalidArgument ") + e.what());
  } catch (const qtnh::ProtocolError& e) {
    rec(k, std::string("ProtocolError ") + e.what());
  } catch (const qtnh::Error& e) {
    rec(k, std::string("Error ") + e.what());
  }
}

void case_indexing() {
  IndexTuple s({2, 3, 4, 5}, 2);
  std::ostringstream os;
  os << s.str() << " nd=" << s.dist_size() << " nl=" << s.local_size() << " tot=" << s.total_size()
     << " n_dist=" << s.n_dist() << " n_local=" << s.n_local() << " all_dist=" << IndexTuple({2, 2}, 2).str()
     << " scalar=" << IndexTuple({}, 0).str();
  rec("indexing.shape", os.str());
  rec("indexing.flat_offset", std::to_string(qtnh::flat_offset({3, 4}, s)) + " " +
                                  std::to_string(qtnh::idx::flat({1, 2, 3, 4}, s.dims)));
  rec("indexing.unflat", ints(qtnh::idx::unflat(97, s.dims)));
  rec("indexing.strides", ints(qtnh::idx::strides(s.dims)));
  DistParams d{2, 3, 1};
  rec("indexing.home_ranks", ints(qtnh::home_ranks({1, 2}, s, d)));
  rec("indexing.home_ranks_of_block", ints(qtnh::home_ranks_of_block(4, s.dist_size(), d)));
  rec("indexing.canonical", std::to_string(qtnh::canonical_rank_of_block(4, d)));
  std::ostringstream loc;
  for (int r = 0; r < 40; ++r) {
    qtnh::BlockLocation b{0, 0, 0};
    if (qtnh::locate_rank(r, s.dist_size(), d, &b)) loc << " " << r << ":" << b.cycle << "/" << b.block << "/" << b.slot;
    else loc << " " << r << ":-";
  }
  rec("indexing.locate", loc.str());
  qtnh::Odometer od({2, 1, 3});
  std::ostringstream o2;
  o2 << od.count() << ":";
  for (Dim i = 0; i < od.count(); ++i) {
    o2 << " (" << ints(od.coords()) << " )";
    o2 << od.advance();
  }
  rec("indexing.odometer", o2.str());
  expect_error("indexing.err.split", [] { IndexTuple({2, 2}, 3); });
  expect_error("indexing.err.dim", [] { IndexTuple({2, 0}, 1); });
  expect_error("indexing.err.flat", [&] { qtnh::idx::flat({1, 3, 0, 0}, s.dims); });
  expect_error("indexing.err.flat_count", [&] { qtnh::idx::flat({1, 2}, s.dims); });
  expect_error("indexing.err.dist", [] { DistParams{0, 1, 0}.validate(); });
}

void case_dense() {
  const auto global = ramp(48, 0.5, -1.0);
  World w(6);
  w.run([&](Rank& rk) {
    Tensor t = Tensor::from_global(rk, IndexTuple({2, 3, 4, 2}, 2), DistParams{1, 1, 0}, global);
    rec(key("dense", rk, "describe"), describe(t));
    rec(key("dense", rk, "local"), str(t.local_data()));
    rec(key("dense", rk, "global"), str(t.to_global_vector()));
    rec(key("dense", rk, "element"), str(t.element({1, 2, 3, 1})) + " |" + str(t.element({0, 1, 2, 0})));
    rec(key("dense", rk, "element_world"), str(t.element_world({1, 0, 1, 1})));
    expect_error(key("dense", rk, "local_element"), [&] { rec(key("dense", rk, "le"), str(t.local_element({0, 2, 1, 1}))); });
    expect_error(key("dense", rk, "coords"), [&] { t.element({0, 3, 0, 0}); });
    expect_error(key("dense", rk, "coord_count"), [&] { t.element({0, 0}); });
    Tensor f = Tensor::dense_fn(rk, IndexTuple({3, 2, 2}, 1), DistParams{2, 1, 0}, [](const Coords& c) {
      return Complex(double(100 * c[0] + 10 * c[1] + c[2]), -double(c[0]));
    });
    rec(key("dense_fn", rk, "describe"), describe(f));
    rec(key("dense_fn", rk, "global"), str(f.to_global_vector()));
    Tensor sc = Tensor::scalar(rk, Complex(2.5, -1.0));
    rec(key("scalar", rk, "describe"), describe(sc));
    rec(key("scalar", rk, "global"), str(sc.to_global_vector()));
  });
  World w8(8);
  w8.run([&](Rank& rk) {  // replicated copies hold identical blocks
    Tensor t = Tensor::from_global(rk, IndexTuple({2, 3}, 1), DistParams{2, 2, 0}, ramp(6, 1.0, 1.0));
    rec(key("bcast", rk, "describe"), describe(t));
    rec(key("bcast", rk, "local"), str(t.local_data()));
  });
  World w2(2);
  expect_error("resource.span", [&] {
    w2.run([](Rank& rk) { Tensor::from_global(rk, IndexTuple({4}, 1), DistParams{1, 1, 0}, std::vector<Complex>(4)); });
  });
  expect_error("dense.count", [&] {
    w2.run([](Rank& rk) { Tensor::from_global(rk, IndexTuple({2, 2}, 0), {}, std::vector<Complex>(3)); });
  });
  expect_error("dense.local_count", [&] {
    w2.run([](Rank& rk) { Tensor::dense(rk, IndexTuple({2, 2}, 0), {}, std::vector<Complex>(3)); });
  });
}

void case_special_elements() {
  World w(2);
  w.run([&](Rank& rk) {
    Tensor id = Tensor::identity(rk, IndexTuple({2, 2}, 1), {}, {0}, {1});
    rec(key("special", rk, "id"), describe(id) + " |" + str(id.element({1, 1})) + " |" + str(id.element({0, 1})));
    rec(key("special", rk, "id_pairs"), ints(id.equality_in()) + " |" + ints(id.equality_out()));
    Tensor sw = Tensor::swap_tensor(rk, IndexTuple({2, 3, 3, 2}, 0), {}, {0, 1}, {2, 3});
    if (sw.in_span())
      rec(key("special", rk, "swap"), describe(sw) + " |" + str(sw.element({0, 1, 1, 0})) + " |" +
                                          str(sw.element({0, 1, 0, 1})) + " |" + str(sw.element({1, 2, 2, 1})));
    Tensor dg = Tensor::diagonal(rk, IndexTuple({2, 2}, 0), {}, {{0, 2}, {3, 0}});
    if (dg.in_span())
      rec(key("special", rk, "diag"), describe(dg) + " |" + str(dg.element({1, 0})) + " |" + str(dg.element({0, 0})) +
                                          " |" + str(dg.element({1, 1})) + " |" + str(dg.local_data()));
    rec(key("special", rk, "diag_dims"), ints(dg.in_dist_dims()) + " |" + ints(dg.in_local_dims()));
  });
  World w1(1);
  expect_error("special.err.swap_pairs", [&] {
    w1.run([](Rank& rk) { Tensor::swap_tensor(rk, IndexTuple({2, 2}, 0), {}, {0}, {1}); });
  });
  expect_error("special.err.pair_len", [&] {
    w1.run([](Rank& rk) { Tensor::identity(rk, IndexTuple({2, 2, 2}, 0), {}, {0, 1}, {2}); });
  });
  expect_error("special.err.pair_dup", [&] {
    w1.run([](Rank& rk) { Tensor::identity(rk, IndexTuple({2, 2}, 0), {}, {0}, {0}); });
  });
  expect_error("special.err.pair_cover", [&] {
    w1.run([](Rank& rk) { Tensor::identity(rk, IndexTuple({2, 2, 2, 2}, 0), {}, {0}, {1}); });
  });
  expect_error("special.err.pair_dims", [&] {
    w1.run([](Rank& rk) { Tensor::identity(rk, IndexTuple({2, 3}, 0), {}, {0}, {1}); });
  });
  expect_error("special.err.diag_len", [&] {
    w1.run([](Rank& rk) { Tensor::diagonal(rk, IndexTuple({2, 2}, 0), {}, std::vector<Complex>(3)); });
  });
  expect_error("special.err.sym_odd", [&] {
    w1.run([](Rank& rk) { Tensor::symmetric(rk, IndexTuple({2, 2, 2}, 0), {}, std::vector<Complex>(8)); });
  });
  expect_error("special.err.sym_dims", [&] {
    w1.run([](Rank& rk) { Tensor::symmetric(rk, IndexTuple({2, 3}, 0), {}, std::vector<Complex>(6)); });
  });
  expect_error("special.err.sym_dist_dims", [&] {
    w1.run([](Rank& rk) { Tensor::diagonal(rk, IndexTuple({1, 2, 2, 2}, 2), {}, std::vector<Complex>(2)); });
  });
}

std::vector<Tensor> variant_zoo(Rank& rk) {
  std::vector<Tensor> v;
  v.push_back(Tensor::identity(rk, IndexTuple({2, 2}, 0), {}, {0}, {1}));
  v.push_back(Tensor::diagonal(rk, IndexTuple({2, 2}, 0), {}, {{1, 1}, {0, -2}}));
  v.push_back(Tensor::identity(rk, IndexTuple({2, 2, 2, 2}, 2), DistParams{1, 1, 0}, {0, 2}, {1, 3}));
  v.push_back(Tensor::swap_tensor(rk, IndexTuple({2, 2, 2, 2}, 2), DistParams{1, 2, 0}, {0, 2}, {1, 3}));
  v.push_back(Tensor::diagonal(rk, IndexTuple({2, 2, 3, 3}, 2), DistParams{2, 1, 1}, ramp(6, 1.0, -0.0)));
  v.push_back(Tensor::symmetric_from_global(rk, IndexTuple({2, 2, 2, 2}, 2), DistParams{1, 1, 3}, ramp(16, -1.0, 2.0)));
  v.push_back(Tensor::identity(rk, IndexTuple({3, 2, 3, 2}, 1), DistParams{1, 1, 2}, {0, 1}, {2, 3}));
  v.push_back(Tensor::swap_tensor(rk, IndexTuple({3, 3, 3, 3}, 1), DistParams{2, 1, 0}, {0, 1}, {2, 3}));
  return v;
}

void case_to_dense() {
  World w(12);
  w.run([&](Rank& rk) {
    auto zoo = variant_zoo(rk);
    for (std::size_t i = 0; i < zoo.size(); ++i) {
      const Tensor& t = zoo[i];
      std::string c = "zoo" + std::to_string(i);
      rec(key(c.c_str(), rk, "describe"), describe(t));
      Tensor d = t.to_dense();
      rec(key(c.c_str(), rk, "dense"), describe(d));
      if (t.in_span()) {
        rec(key(c.c_str(), rk, "global"), str(t.to_global_vector()));
        rec(key(c.c_str(), rk, "dense_global"), str(d.to_global_vector()));
        rec(key(c.c_str(), rk, "dense_local"), str(d.local_data()));
      }
    }
    Tensor plain = Tensor::from_global(rk, IndexTuple({2}, 0), {}, {{5, 0}, {0, 1}});
    rec(key("zoo", rk, "idempotent"), describe(plain.to_dense()) + " |" + str(plain.to_dense().to_global_vector()));
  });
}

void case_variant_ops() {
  World w(12);
  w.run([&](Rank& rk) {
    auto zoo = variant_zoo(rk);
    for (std::size_t i = 0; i < zoo.size(); ++i) {
      const Tensor& t = zoo[i];
      std::string c = "vop" + std::to_string(i);
      auto put = [&](const char* what, const std::function<Tensor()>& op) {
        expect_error(key(c.c_str(), rk, (std::string(what) + ".status").c_str()), [&] {
          Tensor r = op();
          rec(key(c.c_str(), rk, what), describe(r) + (r.in_span() ? " |" + str(r.to_global_vector()) : std::string()));
        });
      };
      const int n = t.shape().n_idx(), split = t.shape().split;
      std::vector<int> rev(n);
      for (int p = 0; p < n; ++p) rev[p] = n - 1 - p;
      const bool rev_fits = i != 4;  // the reversed (2,2;3,3) needs 19 ranks: a collective ResourceError on every rank
      put("conj", [&] { return ops::conj(t); });
      put("scale", [&] { return ops::scale(t, Complex(0.0, 2.0)); });
      if (rev_fits) put("permute_rev", [&] { return ops::permute(t, rev, split); });
      if (split == 0) put("permute_split1", [&] { return ops::permute(t, rev, 1); });
      if (split > 0) put("gather0", [&] { return ops::gather_index(t, 0); });
      if (i == 2 || i == 6) put("scatter", [&] { return ops::scatter_index(t, split); });
      if (t.shape().n_local() > 0) {
        auto ld = t.shape().local_dims();
        auto small = ld;
        small[0] = 1;
        put("slice", [&] { return ops::slice_local_dims(t, small); });
        auto big = ld;
        big.back() += 1;
        put("pad", [&] { return ops::pad_local_dims(t, big); });
      }
      put("unsqueeze", [&] { return ops::unsqueeze(t, n, false); });
      put("unsqueeze_dist", [&] { return ops::unsqueeze(t, 0, true); });
      put("squeeze", [&] { return ops::squeeze(ops::unsqueeze(t, split, false), split); });
    }
    // rebcast keeps the variant
    Tensor dg = zoo[4];
    Tensor moved = ops::rebcast(dg, DistParams{1, 2, 4});
    rec(key("rebcast", rk, "diag"), describe(moved) + " |" + str(moved.local_data()) +
                                        (moved.in_span() ? " |" + str(moved.to_dense().to_global_vector()) : ""));
    Tensor back = ops::rebcast(moved, DistParams{3, 1, 0});
    rec(key("rebcast", rk, "diag_back"), describe(back) + " |" + str(back.local_data()));
    Tensor id2 = ops::rebcast(zoo[2], DistParams{2, 1, 1});
    rec(key("rebcast", rk, "identity"), describe(id2) + " |" + ints(id2.equality_in()) + " |" + ints(id2.equality_out()) +
                                            (id2.in_span() ? " |" + str(id2.to_global_vector()) : ""));
    Tensor sw2 = ops::rebcast(zoo[3], DistParams{1, 1, 8});
    rec(key("rebcast", rk, "swap"), describe(sw2) + (sw2.in_span() ? " |" + str(sw2.to_global_vector()) : ""));
    Tensor sy2 = ops::rebcast(zoo[5], DistParams{2, 1, 0});
    rec(key("rebcast", rk, "symmetric"), describe(sy2) + " |" + str(sy2.local_data()));
    // a diagonal tensor is mutable through its stored slice
    Tensor dm = zoo[1];
    if (dm.in_span()) {
      auto& st = dm.mutable_local_data();
      if (!st.empty()) st[0] = Complex(7.0, -7.0);
    }
    rec(key("mutable", rk, "diag"), describe(dm) + (dm.in_span() ? " |" + str(dm.to_dense().to_global_vector()) : "") +
                                        (zoo[1].in_span() ? " |" + str(zoo[1].to_global_vector()) : ""));
    expect_error(key("vop", rk, "squeeze_err"), [&] { ops::squeeze(zoo[0], 0); });
    expect_error(key("vop", rk, "unsqueeze_err"), [&] { ops::unsqueeze(zoo[2], 3, true); });
  });
}

void case_structural() {
  World w(8);
  const auto g = ramp(48, 1.0, 3.0);
  w.run([&](Rank& rk) {
    Tensor t = Tensor::from_global(rk, IndexTuple({2, 2, 3, 4}, 1), DistParams{1, 1, 0}, g);
    Tensor same = ops::permute(t, {0, 1, 2, 3}, 1);
    rec(key("perm", rk, "identity"), describe(same));
    Tensor p1 = ops::permute(t, {3, 0, 2, 1}, 1);  // asymmetric: distributed size 2 -> 4
    rec(key("perm", rk, "asym"), describe(p1) + (p1.in_span() ? " |" + str(p1.to_global_vector()) : ""));
    Tensor p2 = ops::permute(p1, {1, 3, 2, 0}, 1);  // back
    rec(key("perm", rk, "round_trip"), describe(p2) + (p2.in_span() ? " |" + str(p2.to_global_vector()) : ""));
    Tensor p3 = ops::permute(t, {2, 1, 0, 3}, 2);  // split grows: 6 blocks
    rec(key("perm", rk, "split2"), describe(p3) + " |" + str(p3.local_data()));
    Tensor sc = ops::scatter_index(t, 1);
    rec(key("perm", rk, "scatter"), describe(sc) + " |" + str(sc.local_data()));
    Tensor ga = ops::gather_index(sc, 0);
    rec(key("perm", rk, "gather"), describe(ga) + (ga.in_span() ? " |" + str(ga.to_global_vector()) : ""));
    Tensor rb = ops::rebcast(t, DistParams{2, 2, 0});
    rec(key("perm", rk, "rebcast"), describe(rb) + " |" + str(rb.local_data()));
    Tensor rb2 = ops::rebcast(rb, DistParams{1, 1, 5});
    rec(key("perm", rk, "rebcast_shift"), describe(rb2) + " |" + str(rb2.local_data()));
    Tensor sl = ops::slice_local_dims(t, {2, 2, 3});
    Tensor pd = ops::pad_local_dims(sl, {2, 3, 4});
    rec(key("perm", rk, "slice_pad"), describe(sl) + " |" + describe(pd) + (pd.in_span() ? " |" + str(pd.to_global_vector()) : ""));
    expect_error(key("perm", rk, "err_size"), [&] { ops::permute(t, {0, 1}, 1); });
    expect_error(key("perm", rk, "err_dup"), [&] { ops::permute(t, {0, 1, 1, 3}, 1); });
    expect_error(key("perm", rk, "err_split"), [&] { ops::permute(t, {0, 1, 2, 3}, 5); });
    expect_error(key("perm", rk, "err_scatter"), [&] { ops::scatter_index(t, 0); });
    expect_error(key("perm", rk, "err_gather"), [&] { ops::gather_index(t, 2); });
    expect_error(key("perm", rk, "err_slice"), [&] { ops::slice_local_dims(t, {2, 3, 5}); });
    expect_error(key("perm", rk, "err_pad"), [&] { ops::pad_local_dims(t, {2, 3, 3}); });
    expect_error(key("perm", rk, "err_dist"), [&] { ops::rebcast(t, DistParams{0, 1, 0}); });
  });
  World w4(4);
  expect_error("perm.err_resource", [&] {
    w4.run([&](Rank& rk) {
      Tensor t = Tensor::from_global(rk, IndexTuple({2, 2, 3, 4}, 1), DistParams{1, 1, 0}, g);
      ops::permute(t, {2, 1, 0, 3}, 2);  // needs 6 ranks
    });
  });
}

void case_files(const std::string& dir) {
  World w(6);
  const auto g = ramp(48, 0.5, 1.0);
  w.run([&](Rank& rk) {
    Tensor t = Tensor::from_global(rk, IndexTuple({2, 3, 4, 2}, 2), DistParams{1, 1, 0}, g);
    t.save(dir + "/dense.qtt");
    rk.world_group().barrier();
    Tensor r = Tensor::load(rk, dir + "/dense.qtt");
    rec(key("file", rk, "dense"), describe(r) + " |" + str(r.local_data()));
    Tensor dd = Tensor::diagonal(rk, IndexTuple({2, 2, 3, 3}, 2), DistParams{1, 1, 1}, ramp(6, 2.0, -1.0));
    dd.save(dir + "/diag_dist.qtt");
    rk.world_group().barrier();
    Tensor rd = Tensor::load(rk, dir + "/diag_dist.qtt");
    rec(key("file", rk, "diag_dist"), describe(rd) + " |" + str(rd.local_data()));
    Tensor sy = Tensor::symmetric_from_global(rk, IndexTuple({2, 2, 2, 2}, 2), DistParams{1, 1, 2}, ramp(16, 1.0, 1.0));
    sy.save(dir + "/sym.qtt");
    rk.world_group().barrier();
    Tensor rs = Tensor::load(rk, dir + "/sym.qtt");
    rec(key("file", rk, "sym"), describe(rs) + " |" + str(rs.local_data()));
  });
  World w1(1);
  w1.run([&](Rank& rk) {
    Tensor dg = Tensor::diagonal(rk, IndexTuple({2, 2}, 0), {}, {{1, 2}, {3, 4}});
    dg.save(dir + "/diag.qtt");
    Tensor r = Tensor::load(rk, dir + "/diag.qtt");
    rec("file.diag", describe(r) + " |" + str(r.to_dense().to_global_vector()));
    Tensor sw = Tensor::swap_tensor(rk, IndexTuple({2, 2, 2, 2}, 0), {}, {0, 1}, {2, 3});
    sw.save(dir + "/swap.qtt");
    Tensor rs = Tensor::load(rk, dir + "/swap.qtt");
    rec("file.swap", describe(rs) + " |" + ints(rs.equality_in()) + " |" + ints(rs.equality_out()) + " |" +
                         str(rs.to_dense().to_global_vector()));
    Tensor id = Tensor::identity(rk, IndexTuple({3, 2, 2, 3}, 0), {}, {0, 2}, {3, 1});
    id.save(dir + "/id.qtt");
    Tensor ri = Tensor::load(rk, dir + "/id.qtt");
    rec("file.id", describe(ri) + " |" + ints(ri.equality_in()) + " |" + ints(ri.equality_out()) + " |" +
                       str(ri.to_dense().to_global_vector()));
  });
  for (const char* f : {"dense", "diag_dist", "sym", "diag", "swap", "id"})
    rec(std::string("file.bytes.") + f, file_hex(dir + "/" + f + ".qtt"));
  {
    std::ofstream bad(dir + "/bad.qtt", std::ios::binary);
    bad << "NOTATENSOR";
  }
  expect_error("file.err.magic", [&] { w1.run([&](Rank& rk) { Tensor::load(rk, dir + "/bad.qtt"); }); });
  expect_error("file.err.missing", [&] { w1.run([&](Rank& rk) { Tensor::load(rk, dir + "/absent.qtt"); }); });
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 3) return 2;  // argv[1] = output file, argv[2] = scratch directory
  case_indexing();
  case_dense();
  case_special_elements();
  case_to_dense();
  case_variant_ops();
  case_structural();
  if (chdir(argv[2]) != 0) return 4;  // relative paths: error messages must not depend on the scratch location
  case_files(".");
  std::FILE* f = std::fopen(argv[1], "w");  // absolute path (opened after the chdir)
  if (!f) return 3;
  for (const auto& kv : g_rec) std::fprintf(f, "%s = %s\n", kv.first.c_str(), kv.second.c_str());
  std::fclose(f);
  std::printf("tensor dropin ok (%zu records)\n", g_rec.size());
  return 0;
}
