// The reference's own unit-test cases (/root/reference/proj/tests/, cited per case),
// restated against the drop-in header: the same ndconv:: calls, now executed by
// libndconv_b200.so on the GPU.  Exact-equality KATs stay exact (small integers are
// exact in float32); floating-point identities use float32 tolerances.
// Exit status = number of failed checks.
#include <cmath>
#include <cstdio>
#include <random>

#include "ndconv_b200/ndconv.hpp"

using namespace ndconv;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                         \
  do {                                                                      \
    if (cond) {                                                             \
      ++g_pass;                                                             \
    } else {                                                                \
      ++g_fail;                                                             \
      std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #cond);           \
    }                                                                       \
  } while (0)
#define CHECK_THROWS_AS(expr, T)            \
  do {                                      \
    bool ok = false;                        \
    try {                                   \
      (void)(expr);                         \
    } catch (const T&) {                    \
      ok = true;                            \
    } catch (...) {                         \
    }                                       \
    CHECK(ok && "throws " #T);              \
  } while (0)

static Tensor rnd(std::mt19937_64& g, const Shape& s) {
  std::uniform_real_distribution<double> d(-1.0, 1.0);
  Tensor t = Tensor::zeros(s);
  for (std::size_t i = 0; i < t.size(); ++i) t[i] = static_cast<float>(d(g));  // fp32-exact
  return t;
}

int main() {
  // test_convolution.cpp:11-19
  CHECK(conv_full(Tensor(Shape({2}), {1.0, 2.0}), Kernel(Tensor(Shape({3}), {1.0, 1.0, 1.0}))) ==
        Tensor(Shape({4}), {1.0, 3.0, 3.0, 2.0}));
  CHECK(conv_full(Tensor(Shape({3}), {1.0, 2.0, 3.0}), Kernel(Tensor(Shape({3}), {0.0, 1.0, 0.0}))) ==
        Tensor(Shape({5}), {0.0, 1.0, 2.0, 3.0, 0.0}));
  // test_convolution.cpp:33-38
  {
    const Tensor x(Shape({2, 2}), {1.0, 2.0, 3.0, 4.0});
    const Kernel h1(Tensor(Shape({3}), {1.0, 1.0, 1.0}));
    CHECK_THROWS_AS(conv_full(x, h1), ShapeError);
    CHECK_THROWS_AS(adjoint_apply(x, h1, Shape({2, 2})), ShapeError);
  }
  // test_convolution.cpp:40-45
  CHECK(conv_full(Tensor(Shape({1}), {3.0}), Kernel(Tensor(Shape({5}), {1.0, 2.0, 4.0, 2.0, 1.0}))) ==
        Tensor(Shape({5}), {3.0, 6.0, 12.0, 6.0, 3.0}));
  // test_convolution.cpp:47-59 (linearity) and 110-122 (adjoint identity), fp32 tolerance
  {
    std::mt19937_64 g(22);
    for (int c = 0; c < 10; ++c) {
      const Shape s({std::size_t(3 + c % 4), std::size_t(2 + c % 3)});
      const Kernel h(rnd(g, Shape({std::size_t(1 + 2 * (c % 3)), 3})));
      const Tensor a = rnd(g, s), b = rnd(g, s);
      const Tensor lhs = conv_full(add(scale(a, 2.5), scale(b, -1.25)), h);
      const Tensor rhs = add(scale(conv_full(a, h), 2.5), scale(conv_full(b, h), -1.25));
      double worst = 0.0;
      for (std::size_t i = 0; i < lhs.size(); ++i) worst = std::max(worst, std::abs(lhs[i] - rhs[i]));
      CHECK(worst <= 1e-5);
      const Tensor y = rnd(g, conv_output_shape(s, h));
      const double l = dot(conv_full(a, h), y), r = dot(a, adjoint_apply(y, h, s));
      CHECK(std::abs(l - r) / std::max({1.0, std::abs(l), std::abs(r)}) <= 1e-5);
    }
  }
  // test_convolution.cpp:61-82 flip
  {
    const Kernel h(Tensor(Shape({1, 3}), {1.0, 2.0, 3.0}));
    CHECK(flip(h).tensor() == Tensor(Shape({1, 3}), {3.0, 2.0, 1.0}));
    CHECK(flip(flip(h)).tensor() == h.tensor());
  }
  // test_convolution.cpp:84-102 crop
  {
    std::vector<double> v(25);
    for (std::size_t i = 0; i < 25; ++i) v[i] = double(i + 1);
    const Tensor t(Shape({5, 5}), v);
    CHECK(crop_center(t, Shape({3, 3})) ==
          Tensor(Shape({3, 3}), {7.0, 8.0, 9.0, 12.0, 13.0, 14.0, 17.0, 18.0, 19.0}));
    CHECK_THROWS_AS(crop_center(t, Shape({4, 4})), ShapeError);
    const std::vector<std::size_t> radii{2};
    CHECK_THROWS_AS(crop_m(Tensor::zeros(Shape({9})), radii, Shape({3})), ShapeError);
  }
  // test_convolution.cpp:104-108
  CHECK(adjoint_apply(Tensor(Shape({4}), {1.0, 0.0, 0.0, 0.0}), Kernel(Tensor(Shape({3}), {1.0, 2.0, 3.0})),
                      Shape({2})) == Tensor(Shape({2}), {1.0, 0.0}));
  // test_convolution.cpp:124-136 missing-flip guard
  {
    const Shape s({4});
    const Kernel h(Tensor(Shape({3}), {1.0, 0.0, -2.0}));
    const Tensor x(Shape({4}), {1.0, -1.0, 2.0, 0.5});
    const Tensor y(Shape({6}), {0.5, 1.0, -2.0, 0.0, 1.5, -1.0});
    const double good = dot(x, adjoint_apply(y, h, s));
    const double bad = dot(x, crop_m(conv_full(y, h), h.radii(), s));
    CHECK(std::abs(dot(conv_full(x, h), y) - good) <= 1e-6);
    CHECK(std::abs(dot(conv_full(x, h), y) - bad) > 1e-6);
  }
  // test_solvers.cpp:12-22
  CHECK(objective(Tensor(Shape({1}), {1.0}), Tensor(Shape({1}), {3.0}), Kernel(Tensor(Shape({1}), {1.0}))) == 2.0);
  // test_solvers.cpp:24-40
  CHECK(std::abs(estimate_step(Kernel(Tensor(Shape({1}), {1.0})), Shape({5}), 10) - 1.0) <= 1e-6);
  CHECK(std::abs(estimate_step(Kernel(Tensor(Shape({1}), {2.0})), Shape({5}), 10) - 0.25) <= 1e-6);
  {
    const double s = estimate_step(Kernel(Tensor(Shape({3}), {1.0, 1.0, 1.0})), Shape({8}), 30);
    CHECK(s >= 1.0 / 9.0 - 1e-7 && s <= 1.0);
    CHECK_THROWS_AS(estimate_step(Kernel(Tensor(Shape({3}), {0.0, 0.0, 0.0})), Shape({4}), 5), NumericError);
  }
  // test_solvers.cpp:42-60
  {
    const Kernel h(Tensor(Shape({3}), {0.5, 1.0, 0.25}));
    const Tensor truth(Shape({4}), {0.0, 2.0, 0.0, 1.0});
    CHECK(kkt_residual(truth, conv_full(truth, h), h) <= 1e-6);
    const Tensor zero = Tensor::zeros(Shape({4}));
    CHECK(kkt_residual(zero, Tensor::filled(conv_output_shape(zero.shape(), h), -1.0), h) == 0.0);
  }
  // test_solvers.cpp:62-71 identity kernel
  {
    DeconvConfig cfg;
    cfg.max_iters = 50;
    const Tensor y(Shape({4}), {3.0, -2.0, 0.0, 5.0});
    auto rep = deconv_pg(y, Kernel(Tensor(Shape({1}), {1.0})), y.shape(), cfg);
    CHECK(rep.estimate == clamp_nonneg(y));
    CHECK(rep.stop_reason == StopReason::converged);
    CHECK(rep.iterations_run <= 2);
  }
  // test_solvers.cpp:73-83 sparse 1-d recovery
  {
    const Tensor truth(Shape({3}), {0.0, 4.0, 0.0});
    const Kernel h(Tensor(Shape({3}), {0.0, 1.0, 0.0}));
    DeconvConfig cfg;
    cfg.max_iters = 200;
    cfg.tol_rel_objective = 0.0;
    auto rep = deconv_pg(conv_full(truth, h), h, truth.shape(), cfg);
    for (std::size_t i = 0; i < 3; ++i) CHECK(std::abs(rep.estimate[i] - truth[i]) <= 1e-6);
  }
  // test_solvers.cpp:85-93 negative data -> zero
  {
    DeconvConfig cfg;
    cfg.max_iters = 100;
    auto rep = deconv_pg(Tensor::filled(Shape({6}), -2.0), Kernel(Tensor(Shape({3}), {0.2, 0.5, 0.3})),
                         Shape({4}), cfg);
    CHECK(rep.estimate == Tensor::zeros(Shape({4})));
    CHECK(rep.kkt_trace.back() == 0.0);
  }
  // test_solvers.cpp:95-112 monotone, nonnegative, trace lengths
  {
    std::mt19937_64 g(41);
    for (int c = 0; c < 6; ++c) {
      const Shape s({std::size_t(2 + c % 4), std::size_t(3 + c % 3)});
      const Kernel h(rnd(g, Shape({3, std::size_t(1 + 2 * (c % 2))})));
      const Tensor y = rnd(g, conv_output_shape(s, h));
      DeconvConfig cfg;
      cfg.max_iters = 40;
      cfg.tol_rel_objective = 0.0;
      auto rep = deconv_pg(y, h, s, cfg);
      CHECK(rep.objective_trace.size() == rep.iterations_run + 1);
      for (std::size_t k = 1; k < rep.objective_trace.size(); ++k)
        CHECK(rep.objective_trace[k] < rep.objective_trace[k - 1]);
      for (std::size_t i = 0; i < rep.estimate.size(); ++i) CHECK(rep.estimate[i] >= 0.0);
      CHECK(rep.kkt_trace.size() == rep.objective_trace.size());
    }
  }
  // test_solvers.cpp:168-189 typed errors
  {
    const Kernel h(Tensor(Shape({3}), {0.1, 0.8, 0.1}));
    const Tensor y = Tensor::zeros(Shape({6}));
    CHECK_THROWS_AS(deconv_pg(y, h, Shape({5})), ShapeError);
    CHECK_THROWS_AS(deconv_pg(y, Kernel(Tensor(Shape({3}), {0.0, 0.0, 0.0})), Shape({4})), NumericError);
    DeconvConfig bad;
    bad.backtrack_factor = 1.0;
    CHECK_THROWS_AS(deconv_pg(y, h, Shape({4}), bad), Error);
    DeconvConfig bad2;
    bad2.max_iters = 0;
    CHECK_THROWS_AS(deconv_pg(y, h, Shape({4}), bad2), Error);
  }
  std::printf("dropin: %d passed, %d failed\n", g_pass, g_fail);
  return g_fail;
}
