// One reference call sequence, compiled UNCHANGED against either implementation:
//   * the reference headers (/root/reference/proj/include/qtnh, with the oracle's
//     BLAS/LAPACK shims): `make -C oracle dropin` -> tests/golden/linalg_dropin_ref.txt
//   * the B200 drop-in (include/qtnh_b200.hpp, -DQTNH_B200): namespace swap only.
// The sequence is linalg.hpp's contraction and MPS split as a caller writes it:
// tensor_to_matrix -> pgemm -> matrix_to_tensor -> tensor_to_matrix -> psvd ->
// truncate_svd (cut and zero pad) -> absorb_singular_left/right(power) ->
// pgemm -> matrix_to_tensor, plus Tensor value semantics (mutable_local_data) and
// Group collectives (runtime.hpp). Rank 0 writes every result to argv[1]; the
// pytest compares the two files (contractions / reconstructions within 1e-10,
// S within 1e-10, structural values and error messages exactly).
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

#ifdef QTNH_B200
#include "qtnh_b200.hpp"
namespace qtnh = qtnh_b200;
#else
#include <qtnh/linalg.hpp>
#include <qtnh/ops.hpp>
#include <qtnh/runtime.hpp>
#include <qtnh/tensor.hpp>
#endif

using qtnh::Complex;
using qtnh::DistParams;
using qtnh::IndexTuple;
using qtnh::Rank;
using qtnh::Tensor;
using qtnh::World;
namespace linalg = qtnh::linalg;

static std::vector<Complex> lcg_values(std::size_t n, std::uint64_t seed) {
  std::vector<Complex> v(n);
  std::uint64_t x = seed;
  auto next = [&] {
    x = x * 6364136223846793005ULL + 1442695040888963407ULL;
    return static_cast<double>(x >> 11) * 0x1.0p-53 - 0.5;
  };
  for (auto& c : v) {
    double re = next();
    c = Complex(re, next());
  }
  return v;
}

static void put(std::FILE* f, const char* name, const std::vector<Complex>& v) {
  std::fprintf(f, "%s %zu\n", name, v.size());
  for (const auto& c : v) std::fprintf(f, "%.17g %.17g\n", c.real(), c.imag());
}
static void put_real(std::FILE* f, const char* name, const std::vector<double>& v) {
  std::vector<Complex> c(v.begin(), v.end());
  put(f, name, c);
}

int main(int argc, char** argv) {
  if (argc < 2) return 2;
  const std::vector<Complex> ga = lcg_values(2 * 4 * 6 * 8, 11), gb = lcg_values(4 * 10 * 8, 12);
  std::vector<Complex> c_out, rec3, rec12, cpy_out, orig_out, u_out;
  std::vector<double> s_out, s12, sums;
  std::string a2a_msg;
  double sub_out = 0.0;
  World w(4);
  w.run([&](Rank& ctx) {
    auto grid = linalg::Grid::make(ctx, {0, 1, 2, 3});
    // a (2; 4, 6, 8) over 2 ranks, b (4, 10, 8) replicated on all 4
    Tensor a = Tensor::from_global(ctx, IndexTuple({2, 4, 6, 8}, 1), DistParams{1, 1, 0}, ga);
    Tensor b = Tensor::from_global(ctx, IndexTuple({4, 10, 8}, 0), DistParams{4, 1, 0}, gb);
    // contract a[1], a[3] with b[0], b[2] (K = 8 * 4 = 32)
    auto ma = linalg::tensor_to_matrix(a, {0, 2}, {3, 1}, &grid, 0, 32);
    auto mb = linalg::tensor_to_matrix(b, {2, 0}, {1}, &grid, 32, 0);
    auto mc = linalg::pgemm(ma, mb);  // 12 x 10
    Tensor c = linalg::matrix_to_tensor(mc, ctx, IndexTuple({2, 6, 10}, 1), a.dist(), {0, 1}, {2});
    auto cg = c.to_global_vector();
    // MPS-style split of c: rows (2, 6), cols (10), chi = 3 (cut) and 12 (pad)
    auto m = linalg::tensor_to_matrix(c, {0, 1}, {2}, &grid, 4, 4);  // square blocks: U and Vh chain in pgemm
    auto sv = linalg::psvd(m);
    auto tr = linalg::truncate_svd(sv.u, sv.s, sv.vh, 3);
    linalg::absorb_singular_left(tr.u, tr.s, 0.5);
    linalg::absorb_singular_right(tr.vh, tr.s, 0.5);
    Tensor r3 = linalg::matrix_to_tensor(linalg::pgemm(tr.u, tr.vh), ctx, IndexTuple({2, 6, 10}, 1), a.dist(),
                                         {0, 1}, {2});
    auto tp = linalg::truncate_svd(sv.u, sv.s, sv.vh, 12);
    linalg::absorb_singular_left(tp.u, tp.s, 1.0);
    Tensor r12 = linalg::matrix_to_tensor(linalg::pgemm(tp.u, tp.vh), ctx, IndexTuple({2, 6, 10}, 0),
                                          DistParams{1, 1, 0}, {0, 1}, {2});
    Tensor ut = linalg::matrix_to_tensor(tr.u, ctx, IndexTuple({12, 3}, 0), DistParams{1, 1, 0}, {0}, {1});
    auto r3g = r3.to_global_vector();
    auto r12g = r12.to_global_vector();
    auto ug = ut.to_global_vector();
    // value semantics: a copy mutated through mutable_local_data leaves the original
    Tensor d = c;
    if (d.in_span()) {
      auto& loc = d.mutable_local_data();
      for (auto& x : loc) x *= Complex(0.0, 2.0);
    }
    auto dg = d.to_global_vector();
    auto c2 = c.to_global_vector();
    // Group collectives
    auto g = ctx.group({0, 1, 2, 3});
    double tot = g.all_reduce_sum(static_cast<double>(ctx.rank() + 1));
    auto bc = g.broadcast(std::vector<double>{ctx.rank() == 2 ? 7.5 : -1.0, 2.5}, 2);
    auto gat = g.gather(std::vector<double>(ctx.rank() + 1, 1.0 * ctx.rank()), 0);
    std::vector<std::vector<double>> chunks;
    if (ctx.rank() == 1)
      for (int j = 0; j < 4; ++j) chunks.push_back(std::vector<double>(j + 1, 10.0 * j));
    auto sc = g.scatter(chunks, 1);
    std::vector<std::vector<int>> sends(4);
    for (int j = 0; j < 4; ++j) sends[j].assign(ctx.rank() == 0 && j == 1 ? 2 : 3, ctx.rank());
    std::vector<std::size_t> expect(4, 3);
    try {
      g.all_to_all_v(sends, &expect);
    } catch (const qtnh::ProtocolError& e) {
      if (ctx.rank() == 1) a2a_msg = e.what();
    }
    double sub_tot = 0.0;
    if (ctx.rank() == 1 || ctx.rank() == 3) {  // member-only group in the given order
      auto sub = ctx.group({3, 1});
      sub_tot = sub.all_reduce_sum(static_cast<double>(ctx.rank()));
    }
    if (ctx.rank() == 0) {
      c_out = cg;
      s_out = sv.s;
      s12 = tp.s;
      rec3 = r3g;
      rec12 = r12g;
      u_out = ug;
      cpy_out = dg;
      orig_out = c2;
      double gsum = 0;
      for (auto& v : gat) gsum += v.size();
      sums = {tot, bc[0], bc[1], gsum, static_cast<double>(sc.size()), sc.empty() ? -1.0 : sc[0]};
    }
    if (ctx.rank() == 1) sub_out = sub_tot;
  });
  sums.push_back(sub_out);
  std::FILE* f = std::fopen(argv[1], "w");
  if (!f) return 3;
  put(f, "contract", c_out);
  put_real(f, "s", s_out);
  put_real(f, "s_pad12", s12);
  put(f, "recon_chi3", rec3);
  put(f, "recon_chi12", rec12);
  put(f, "copy_scaled", cpy_out);
  put(f, "original_after_copy", orig_out);
  put_real(f, "collectives", sums);
  std::fprintf(f, "a2a_error %s\n", a2a_msg.c_str());
  std::fprintf(f, "u_chi3_absorbed %zu\n", u_out.size());
  std::fclose(f);
  std::printf("linalg dropin ok\n");
  return 0;
}
