// Drop-in check: reference-style user code (README.md:106-116 of the
// reference) compiled against include/rectri/ and linked to librectri_cu.so.
// Host MatrixBuffers exercise the staged path; exits non-zero on failure.
#include <cmath>
#include <cstdio>
#include <random>

#include "rectri/recursion.hpp"

using namespace rectri;

static int failures = 0;
#define EXPECT(c)                                                     \
  do {                                                                \
    if (!(c)) {                                                       \
      std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c);        \
      ++failures;                                                     \
    }                                                                 \
  } while (0)

int main() {
  // Frozen example (test_recursion.cpp:114-130).
  {
    MatrixBuffer<double> a(2, 2), b(2, 1);
    a(0, 0) = 2; a(1, 0) = 1; a(1, 1) = 4;
    b(0, 0) = 2; b(1, 0) = 6;
    rec_trsm<double>(TriangularSpec{}, a.view(), b.view(), Threshold{1});
    EXPECT(b(0, 0) == 1.0 && b(1, 0) == 1.25);
  }
  // README usage, float, alpha = 2, parallel backend spelling.
  const index_t n = 300, m = 40;
  TriangularSpec spec;
  spec.alpha = 2.0;
  MatrixBuffer<float> a(n, n), b(n, m);
  std::mt19937_64 rng(7);
  std::uniform_real_distribution<double> u(-1, 1);
  for (index_t c = 0; c < n; ++c)
    for (index_t r = 0; r < n; ++r) a(r, c) = static_cast<float>(u(rng));
  for (index_t r = 0; r < n; ++r) {
    double s = 0;
    for (index_t c = 0; c < r; ++c) s += std::fabs(a(r, c));
    a(r, r) = static_cast<float>(s + 1);
  }
  for (index_t c = 0; c < m; ++c)
    for (index_t r = 0; r < n; ++r) b(r, c) = static_cast<float>(u(rng));
  MatrixBuffer<float> x = b;
  index_t gemms = 0, leaves = 0;
  rec_trsm<float>(spec, a.view(), x.view(), Threshold{64}, Backend::par(),
                  [&](RecEvent e, index_t, index_t) { (e == RecEvent::Gemm ? gemms : leaves)++; });
  EXPECT(gemms == 7 && leaves == 8);
  double worst = 0, anorm = 0;
  for (index_t r = 0; r < n; ++r) {
    double s = 0;
    for (index_t c = 0; c <= r; ++c) s += std::fabs(a(r, c));
    anorm = std::max(anorm, s);
  }
  for (index_t c = 0; c < m; ++c)
    for (index_t r = 0; r < n; ++r) {
      double lhs = 0;
      for (index_t k = 0; k <= r; ++k) lhs += double(a(r, k)) * x(k, c);
      worst = std::max(worst, std::fabs(lhs - 2.0 * b(r, c)));
    }
  EXPECT(worst <= 32.0 * n * 1.2e-7 * anorm * 2.0);
  // Singularity: global row, exception type.
  {
    MatrixBuffer<double> s(16, 16), rhs(16, 2, 1.0);
    for (index_t i = 0; i < 16; ++i) s(i, i) = i == 11 ? 0.0 : 3.0;
    bool threw = false;
    try {
      rec_trsm<double>(TriangularSpec{}, s.view(), rhs.view(), Threshold{4});
    } catch (const SingularityError& e) {
      threw = e.index() == 11;
    }
    EXPECT(threw);
  }
  // Validation: ConfigError for threshold 0, AliasError for overlapping views.
  {
    MatrixBuffer<double> s(8, 8, 1.0);
    bool cfg = false, alias = false;
    try {
      rec_trmm<double>(TriangularSpec{}, s.view().subview(0, 0, 4, 4), s.view().subview(4, 4, 4, 4), Threshold{0});
    } catch (const ConfigError&) { cfg = true; }
    try {
      rec_trmm<double>(TriangularSpec{}, s.view().subview(0, 0, 4, 4), s.view().subview(3, 3, 4, 4), Threshold{2});
    } catch (const AliasError&) { alias = true; }
    EXPECT(cfg && alias);
  }
  std::printf("dropin_example: %s (residual %.3e)\n", failures ? "FAILED" : "ok", worst);
  return failures ? 1 : 0;
}
