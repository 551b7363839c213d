// bench_host.cpp -- host-side helpers of the benchmark harness (bench CLI
// parity): the reference's input generator and
// residual-gate column sampling, evaluated with libstdc++'s own <random> so
// the streams are bit-identical to the reference's (src/bench.cpp:32-61,
// 100-117).  No compute runs here; the solves run on the GPU.
#include <cmath>
#include <cstdint>
#include <random>

namespace {

// src/bench.cpp:32-61: A (n x n) then B from one mt19937_64 stream,
// uniform [-1, 1); TRSM NonUnit diagonal := off-diagonal |row sum| + 1.
template <typename T>
void bench_inputs(T* a, T* b, int64_t n, int64_t brows, int64_t bcols, int is_trsm, int uplo, int diag,
                  uint64_t seed) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> dist(-1.0, 1.0);
  for (int64_t c = 0; c < n; ++c)
    for (int64_t r = 0; r < n; ++r) a[c * n + r] = static_cast<T>(dist(rng));
  if (is_trsm && diag == 0) {
    for (int64_t r = 0; r < n; ++r) {
      double sum = 0.0;
      const int64_t c0 = uplo == 0 ? 0 : r + 1, c1 = uplo == 0 ? r : n;
      for (int64_t c = c0; c < c1; ++c) sum += std::fabs(static_cast<double>(a[c * n + r]));
      a[r * n + r] = static_cast<T>(sum + 1.0);
    }
  }
  for (int64_t c = 0; c < bcols; ++c)
    for (int64_t r = 0; r < brows; ++r) b[c * brows + r] = static_cast<T>(dist(rng));
}

}  // namespace

extern "C" {

void rectri_cu_bench_inputs_f64(double* a, double* b, int64_t n, int64_t brows, int64_t bcols, int32_t is_trsm,
                                int32_t uplo, int32_t diag, uint64_t seed) {
  bench_inputs<double>(a, b, n, brows, bcols, is_trsm, uplo, diag, seed);
}
void rectri_cu_bench_inputs_f32(float* a, float* b, int64_t n, int64_t brows, int64_t bcols, int32_t is_trsm,
                                int32_t uplo, int32_t diag, uint64_t seed) {
  bench_inputs<float>(a, b, n, brows, bcols, is_trsm, uplo, diag, seed);
}

// src/bench.cpp:109-117: all columns when cols <= 8, else 8 draws of
// uniform_int_distribution<int64>(0, cols - 1) from mt19937_64(seed).
int32_t rectri_cu_gate_columns(uint64_t seed, int64_t cols, int64_t out[8]) {
  if (cols <= 8) {
    for (int64_t c = 0; c < cols; ++c) out[c] = c;
    return static_cast<int32_t>(cols);
  }
  std::mt19937_64 rng(seed);
  std::uniform_int_distribution<int64_t> pick(0, cols - 1);
  for (int s = 0; s < 8; ++s) out[s] = pick(rng);
  return 8;
}

}  // extern "C"
