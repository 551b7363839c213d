// End-to-end timing through the C++ drop-in with reference-caller memory.
// Each timed call is rectri::rec_trsm<double> exactly as reference code
// writes it (src/bench.cpp:184-192).  Two storages:
//   buffer    rectri::MatrixBuffer, as the reference's callers allocate it --
//             the drop-in's MatrixBuffer keeps its bytes page-locked
//             (rectri_cu_host_alloc), so the library streams them directly;
//   pageable  plain std::vector<double> wrapped in MatrixViews (the public
//             MatrixView constructor, matrix.hpp:82-90): PAGEABLE memory the
//             library stages through its pinned bounce buffers.
// Either way the library computes on the GPU and writes X back into host
// memory before returning.
//
//   dropin_bench N M STEPS WARMUP [buffer|pageable]   -> one JSON line on stdout
//
// B is restored from a pristine copy between calls, outside the clock
// (bench.cpp:184-218 methodology: steady_clock around the call).  A sampled
// residual ||tril(A) X - B||_max / (||A||_inf max(|X|,|B|,1) n eps) on 8
// columns checks the last result.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <limits>
#include <string>
#include <thread>
#include <vector>

#include "rectri/recursion.hpp"

using namespace rectri;

namespace {
// counter-based uniform [-1, 1) (splitmix64), so the fill can run on threads
double uniform(uint64_t key) {
  uint64_t z = key + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  return static_cast<double>(z >> 11) * (2.0 / 9007199254740992.0) - 1.0;
}

template <typename F>
void parallel_cols(index_t cols, F&& f) {
  const int nt = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  std::vector<std::thread> ts;
  for (int t = 0; t < nt; ++t)
    ts.emplace_back([&, t] {
      for (index_t c = t; c < cols; c += nt) f(c);
    });
  for (auto& th : ts) th.join();
}
}  // namespace

int main(int argc, char** argv) {
  const index_t n = argc > 1 ? std::atoll(argv[1]) : 16384;
  const index_t m = argc > 2 ? std::atoll(argv[2]) : 16384;
  const int steps = argc > 3 ? std::atoi(argv[3]) : 5;
  const int warmup = argc > 4 ? std::atoi(argv[4]) : 2;

  const bool pageable = argc > 5 && std::string(argv[5]) == "pageable";
  // storage: MatrixBuffers, or plain vectors behind views of the same shape
  MatrixBuffer<double> Ab(pageable ? 0 : n, pageable ? 0 : n), Bb(pageable ? 0 : n, pageable ? 0 : m),
      B0b(pageable ? 0 : n, pageable ? 0 : m);
  std::vector<double> Av(pageable ? static_cast<size_t>(n * n) : 0), Bv(pageable ? static_cast<size_t>(n * m) : 0),
      B0v(pageable ? static_cast<size_t>(n * m) : 0);
  auto mk = [&](MatrixBuffer<double>& b, std::vector<double>& v, index_t r, index_t c) {
    return pageable ? MatrixView<double>(v.data(), r, c, 0, 0, r, c) : b.view();
  };
  const MatrixView<double> A = mk(Ab, Av, n, n), B = mk(Bb, Bv, n, m), B0 = mk(B0b, B0v, n, m);
  parallel_cols(n, [&](index_t c) {
    for (index_t r = 0; r < n; ++r) A(r, c) = uniform(1000003ull * c + r);
  });
  std::vector<double> diag(n, 0.0);
  parallel_cols(n, [&](index_t r) {  // diagonally dominant lower triangle (bench.cpp:40-51)
    double s = 0;
    for (index_t c = 0; c < r; ++c) s += std::fabs(A(r, c));
    diag[r] = s + 1.0;
  });
  for (index_t r = 0; r < n; ++r) A(r, r) = diag[r];
  parallel_cols(m, [&](index_t c) {
    for (index_t r = 0; r < n; ++r) B0(r, c) = uniform(0xABCDEFull + 7777777ull * c + r);
  });

  const TriangularSpec spec{};  // Left / Lower / NoTrans / NonUnit, alpha = 1
  std::vector<double> ms;
  for (int i = 0; i < warmup + steps; ++i) {
    parallel_cols(m, [&](index_t c) { std::copy(&B0(0, c), &B0(0, c) + n, &B(0, c)); });
    const auto t0 = std::chrono::steady_clock::now();
    rec_trsm<double>(spec, MatrixView<const double>(A), B, Threshold{256});
    const auto t1 = std::chrono::steady_clock::now();
    if (i >= warmup) ms.push_back(std::chrono::duration<double, std::milli>(t1 - t0).count());
  }
  // residual on 8 sampled columns
  double anorm = 0;
  for (index_t r = 0; r < n; ++r) anorm = std::max(anorm, diag[r] * 2 - 1);  // row sum of |tril(A)|
  double worst = 0, xmax = 0, bmax = 0;
  bool finite = true;
  for (int k = 0; k < 8; ++k) {
    const index_t c = (m - 1) * k / 7;
    for (index_t r = 0; r < n; ++r) {
      double lhs = 0;
      for (index_t q = 0; q <= r; ++q) lhs += A(r, q) * B(q, c);
      worst = std::max(worst, std::fabs(lhs - B0(r, c)));
      xmax = std::max(xmax, std::fabs(B(r, c)));
      bmax = std::max(bmax, std::fabs(B0(r, c)));
      finite = finite && std::isfinite(B(r, c));
    }
  }
  const double eta =
      worst / (anorm * std::max({xmax, bmax, 1.0}) * n * std::numeric_limits<double>::epsilon());
  double sum = 0;
  for (double v : ms) sum += v;
  std::vector<double> sorted = ms;
  std::sort(sorted.begin(), sorted.end());
  std::printf("{\"storage\": \"%s\", \"n\": %lld, \"m\": %lld, \"steps\": %d, \"ms_per_step\": %.3f, "
              "\"median_step_ms\": %.3f, \"eta\": %.3e, \"finite\": %s, \"step_ms\": [",
              pageable ? "pageable" : "buffer", static_cast<long long>(n), static_cast<long long>(m), steps,
              sum / ms.size(),
              sorted[sorted.size() / 2], eta, finite ? "true" : "false");
  for (size_t i = 0; i < ms.size(); ++i) std::printf("%s%.2f", i ? ", " : "", ms[i]);
  std::printf("]}\n");
  return finite && eta <= 32 ? 0 : 1;
}
