// C++ caller of the B200 path through include/qtnh_b200.hpp, written like the
// reference's own tests (proj/tests/test_ops.cpp:77-110) to show the drop-in.
#include <cmath>
#include <cstdio>
#include <string>
#include <cstdlib>

#include "qtnh_b200.hpp"

namespace qtnh = qtnh_b200;
using qtnh::Complex;

#define EXPECT(c)                                                   \
  do {                                                              \
    if (!(c)) {                                                     \
      std::fprintf(stderr, "FAILED %s at line %d\n", #c, __LINE__); \
      std::exit(1);                                                 \
    }                                                               \
  } while (0)

int main() {
  // matrix transpose (test_ops.cpp:77-85)
  {
    qtnh::World w(1);
    std::vector<Complex> got;
    w.run([&](qtnh::Rank& rk) {
      auto t = qtnh::Tensor::from_global(rk, {{2, 2}, 0}, {}, {{1, 0}, {2, 0}, {3, 0}, {4, 0}});
      got = qtnh::ops::permute(t, {1, 0}, 0).to_global_vector();
    });
    EXPECT((got == std::vector<Complex>{{1, 0}, {3, 0}, {2, 0}, {4, 0}}));
  }
  // asymmetric permutation recruits more ranks (test_ops.cpp:87-110)
  {
    std::vector<Complex> g(32);
    for (int i = 0; i < 32; ++i) g[i] = {double(i + 1), 0.1 * i};
    qtnh::World w(4);
    std::vector<Complex> got;
    w.run([&](qtnh::Rank& rk) {
      auto t = qtnh::Tensor::from_global(rk, {{2, 2, 4, 2}, 1}, {1, 1, 0}, g);
      EXPECT(t.span() == 2);
      auto p = qtnh::ops::permute(t, {2, 0, 1, 3}, 1);
      EXPECT(p.span() == 4);
      auto v = p.to_global_vector();
      if (rk.rank() == 0) got = v;
    });
    // element (c0,c1,c2,c3) of the source lands at (c2,c0,c1,c3)
    for (int c0 = 0; c0 < 2; ++c0)
      for (int c1 = 0; c1 < 2; ++c1)
        for (int c2 = 0; c2 < 4; ++c2)
          for (int c3 = 0; c3 < 2; ++c3)
            EXPECT(got[((c2 * 2 + c0) * 2 + c1) * 2 + c3] == g[((c0 * 2 + c1) * 4 + c2) * 2 + c3]);
    qtnh::World w2(2);
    bool threw = false;
    try {
      w2.run([&](qtnh::Rank& rk) {
        auto t = qtnh::Tensor::from_global(rk, {{2, 2, 4, 2}, 1}, {1, 1, 0}, g);
        qtnh::ops::permute(t, {2, 0, 1, 3}, 1);
      });
    } catch (const qtnh::ResourceError& e) {
      threw = e.required_ranks == 4;
    }
    EXPECT(threw);
  }
  // matrix-vector contraction known answer
  {
    qtnh::World w(1);
    std::vector<Complex> got;
    w.run([&](qtnh::Rank& rk) {
      auto a = qtnh::Tensor::from_global(rk, {{2, 2}, 0}, {}, {{0, 0}, {1, 0}, {1, 0}, {0, 0}});
      auto v = qtnh::Tensor::from_global(rk, {{2}, 0}, {}, {{1, 0}, {0, 0}});
      got = qtnh::network::contract(a, v, {1}, {0}).to_global_vector();
    });
    EXPECT((got == std::vector<Complex>{{0, 0}, {1, 0}}));
  }
  // truncated SVD reconstruction + QTNHTEN1 round trip through the C++ layer
  {
    qtnh::World w(1);
    double err = 1.0;
    bool same = false;
    w.run([&](qtnh::Rank& rk) {
      std::vector<Complex> g(6 * 4);
      for (int i = 0; i < 24; ++i) g[i] = {std::cos(1.3 * i), std::sin(0.7 * i * i)};
      auto t = qtnh::Tensor::from_global(rk, {{6, 4}, 0}, {}, g);
      auto f = qtnh::linalg::svd(t, {0}, {1}, 0, qtnh::linalg::Absorb::left);
      auto back = qtnh::network::contract(f.u, f.vh, {1}, {0}).to_global_vector();
      double num = 0, den = 0;
      for (int i = 0; i < 24; ++i) {
        num += std::norm(back[i] - g[i]);
        den += std::norm(g[i]);
      }
      err = std::sqrt(num / den);
      const std::string path = "/tmp/qtnh_cpp_api_test.qtt";
      t.save(path);
      same = qtnh::Tensor::load(rk, path).to_global_vector() == g;
    });
    EXPECT(err < 1e-12);
    EXPECT(same);
  }
  // network::plan_order + contract_order: D[d] = sum A[a,b] B[b,c] C[c,d,a]
  {
    qtnh::World w(1);
    std::vector<Complex> got;
    std::vector<int> res_labels;
    std::vector<Complex> A(2 * 3), B(3 * 4), Cc(4 * 2 * 2);
    for (int i = 0; i < 6; ++i) A[i] = {0.3 * i - 1.0, 0.2 * i};
    for (int i = 0; i < 12; ++i) B[i] = {std::cos(0.9 * i), 0.1 * i - 0.4};
    for (int i = 0; i < 16; ++i) Cc[i] = {0.05 * i * i - 0.7, std::sin(1.1 * i)};
    const std::vector<std::vector<int>> labels{{0, 1}, {1, 2}, {2, 3, 0}};  // a b c d = 0 1 2 3
    const std::vector<qtnh::Dim> dims{2, 3, 4, 2};
    auto order = qtnh::network::plan_order(labels, dims, 7, 8);
    auto capped = qtnh::network::plan_order(labels, dims, 7, 8, 4.0);
    EXPECT(order.size() == 2 && capped.size() == 2);
    w.run([&](qtnh::Rank& rk) {
      std::vector<qtnh::Tensor> ts{qtnh::Tensor::from_global(rk, {{2, 3}, 0}, {}, A),
                                   qtnh::Tensor::from_global(rk, {{3, 4}, 0}, {}, B),
                                   qtnh::Tensor::from_global(rk, {{4, 2, 2}, 0}, {}, Cc)};
      got = qtnh::network::contract_order(ts, labels, capped, &res_labels).to_global_vector();
    });
    EXPECT((res_labels == std::vector<int>{3}) && got.size() == 2);
    for (int d = 0; d < 2; ++d) {
      Complex want = 0;
      for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 3; ++b)
          for (int c = 0; c < 4; ++c) want += A[a * 3 + b] * B[b * 4 + c] * Cc[(c * 2 + d) * 2 + a];
      EXPECT(std::abs(got[d] - want) < 1e-12 * (1.0 + std::abs(want)));
    }
  }
  std::printf("cpp api ok\n");
  return 0;
}
