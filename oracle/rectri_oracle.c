/*
 * rectri_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the parity referee of arxiv/paper_2504_13821 ("rectri").
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library, and only as the checker.  The product path
 * (paper_2504_13821_b200/) never links or calls it.
 *
 * Every function cites the reference file:line it restates (paths relative
 * to /root/reference/proj).  Parity is pinned: tests/test_oracle_golden.py
 * checks this restatement against fixtures produced by the reference's own
 * compiled sources (oracle/_ref, recipe in oracle/Makefile; fixtures written
 * by tests/golden/make_golden.py).
 *
 * Conventions: column-major storage, element (r, c) at p[c * ld + r].
 * Enumerations match include/rectri_cu.h (side 0 = Left, 1 = Right; uplo
 * 0 = Lower, 1 = Upper; trans 0 = N, 1 = T, 2 = C; diag 0 = NonUnit, 1 = Unit).
 * Compile with -ffp-contract=off, as the reference does
 * (src/CMakeLists.txt:19-24), so the generators round like the reference.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define RO_OK 0
#define RO_SHAPE 2
#define RO_SINGULAR 4

/* ------------------------------------------------------------------------ */
/* mt19937_64 (Matsumoto & Nishimura 2004 parameters), the engine behind
 * std::mt19937_64 used by every reference generator
 * (tests/test_support.hpp:38-47, src/bench.cpp:32-61). */

typedef struct {
  uint64_t mt[312];
  int mti;
} ro_mt64;

static void mt64_seed(ro_mt64* s, uint64_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) +
               (uint64_t)i;
  s->mti = 312;
}

static uint64_t mt64_next(ro_mt64* s) {
  static const uint64_t mag01[2] = {0ULL, 0xB5026F5AA96619E9ULL};
  const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
  if (s->mti >= 312) {
    int i;
    uint64_t x;
    for (i = 0; i < 312 - 156; ++i) {
      x = (s->mt[i] & UM) | (s->mt[i + 1] & LM);
      s->mt[i] = s->mt[i + 156] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
    }
    for (; i < 311; ++i) {
      x = (s->mt[i] & UM) | (s->mt[i + 1] & LM);
      s->mt[i] = s->mt[i + (156 - 312)] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
    }
    x = (s->mt[311] & UM) | (s->mt[0] & LM);
    s->mt[311] = s->mt[155] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
    s->mti = 0;
  }
  uint64_t y = s->mt[s->mti++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= (y >> 43);
  return y;
}

/* std::uniform_real_distribution<double>(lo, hi) as libstdc++ evaluates it:
 * generate_canonical<double, 53> draws one 64-bit word, converts it to double
 * (round to nearest), divides by 2^64, clamps 1.0 to nextafter(1, 0), then
 * returns u * (hi - lo) + lo with no contraction. */
static double mt64_uniform(ro_mt64* s, double lo, double hi) {
  double u = (double)mt64_next(s) / 18446744073709551616.0;
  if (u >= 1.0) u = nextafter(1.0, 0.0);
  double span = hi - lo;
  double prod = u * span;
  return prod + lo;
}

/* ------------------------------------------------------------------------ */
/* Generators (tests/test_support.hpp:38-85, src/bench.cpp:32-61).
 * The *_f32 variants narrow each draw with static_cast<float>, exactly like
 * MatrixBuffer<float> filling in the reference. */

/* make_random: tests/test_support.hpp:38-47 */
void ro_make_random_f64(double* out, int64_t rows, int64_t cols, uint64_t seed,
                        double lo, double hi) {
  ro_mt64 s;
  mt64_seed(&s, seed);
  for (int64_t c = 0; c < cols; ++c)
    for (int64_t r = 0; r < rows; ++r)
      out[c * rows + r] = mt64_uniform(&s, lo, hi);
}
void ro_make_random_f32(float* out, int64_t rows, int64_t cols, uint64_t seed,
                        double lo, double hi) {
  ro_mt64 s;
  mt64_seed(&s, seed);
  for (int64_t c = 0; c < cols; ++c)
    for (int64_t r = 0; r < rows; ++r)
      out[c * rows + r] = (float)mt64_uniform(&s, lo, hi);
}

/* make_dominant: tests/test_support.hpp:52-62 (diagonal := sum of the stored
 * off-diagonal row magnitudes + 1). */
void ro_make_dominant_f64(double* a, int64_t n, int uplo, uint64_t seed) {
  ro_make_random_f64(a, n, n, seed, -1.0, 1.0);
  for (int64_t r = 0; r < n; ++r) {
    double sum = 0.0;
    int64_t c0 = uplo == 0 ? 0 : r + 1, c1 = uplo == 0 ? r : n;
    for (int64_t c = c0; c < c1; ++c) sum += fabs(a[c * n + r]);
    a[r * n + r] = sum + 1.0;
  }
}
void ro_make_dominant_f32(float* a, int64_t n, int uplo, uint64_t seed) {
  ro_make_random_f32(a, n, n, seed, -1.0, 1.0);
  for (int64_t r = 0; r < n; ++r) {
    double sum = 0.0;
    int64_t c0 = uplo == 0 ? 0 : r + 1, c1 = uplo == 0 ? r : n;
    for (int64_t c = c0; c < c1; ++c) sum += fabs((double)a[c * n + r]);
    a[r * n + r] = (float)(sum + 1.0);
  }
}

/* damp_off_diagonal: tests/test_support.hpp:66-70 */
void ro_damp_off_diagonal_f64(double* a, int64_t n, double factor) {
  for (int64_t c = 0; c < n; ++c)
    for (int64_t r = 0; r < n; ++r)
      if (r != c) a[c * n + r] = a[c * n + r] * factor;
}
void ro_damp_off_diagonal_f32(float* a, int64_t n, double factor) {
  for (int64_t c = 0; c < n; ++c)
    for (int64_t r = 0; r < n; ++r)
      if (r != c) a[c * n + r] = (float)((double)a[c * n + r] * factor);
}

/* bench make_inputs: src/bench.cpp:32-61.  A (n x n) then B (brows x bcols)
 * from one stream; the TRSM NonUnit diagonal becomes row |sum| + 1. */
void ro_bench_inputs_f64(double* a, double* b, int64_t n, int64_t brows,
                         int64_t bcols, int is_trsm, int uplo, int diag,
                         uint64_t seed) {
  ro_mt64 s;
  mt64_seed(&s, seed);
  for (int64_t c = 0; c < n; ++c)
    for (int64_t r = 0; r < n; ++r) a[c * n + r] = mt64_uniform(&s, -1.0, 1.0);
  if (is_trsm && diag == 0) {
    for (int64_t r = 0; r < n; ++r) {
      double sum = 0.0;
      int64_t c0 = uplo == 0 ? 0 : r + 1, c1 = uplo == 0 ? r : n;
      for (int64_t c = c0; c < c1; ++c) sum += fabs(a[c * n + r]);
      a[r * n + r] = sum + 1.0;
    }
  }
  for (int64_t c = 0; c < bcols; ++c)
    for (int64_t r = 0; r < brows; ++r)
      b[c * brows + r] = mt64_uniform(&s, -1.0, 1.0);
}

/* ------------------------------------------------------------------------ */
/* The oracles (src/oracle.cpp). All arithmetic in double. */

/* materialize_triangle: src/oracle.cpp:39-54.  Stored triangle copied, the
 * opposite strict triangle zero and never read, diagonal 1 under Unit. */
static void materialize(const double* a, int64_t lda, int64_t n, int uplo,
                        int diag, double* out) {
  memset(out, 0, sizeof(double) * (size_t)(n * n));
  for (int64_t c = 0; c < n; ++c) {
    int64_t r0 = uplo == 0 ? c : 0, r1 = uplo == 0 ? n : c + 1;
    for (int64_t r = r0; r < r1; ++r) out[c * n + r] = a[c * lda + r];
  }
  if (diag == 1)
    for (int64_t r = 0; r < n; ++r) out[r * n + r] = 1.0;
}

/* materialize_op: src/oracle.cpp:25-34 (ConjTrans == Trans on reals). */
static double* materialize_op(const double* a, int64_t lda, int64_t n,
                              int uplo, int trans, int diag) {
  double* dense = (double*)malloc(sizeof(double) * (size_t)(n * n + 1));
  materialize(a, lda, n, uplo, diag, dense);
  if (trans == 0) return dense;
  double* t = (double*)malloc(sizeof(double) * (size_t)(n * n + 1));
  for (int64_t c = 0; c < n; ++c)
    for (int64_t r = 0; r < n; ++r) t[c * n + r] = dense[r * n + c];
  free(dense);
  return t;
}

/* oracle_trmm: src/oracle.cpp:57-82.  alpha * op(A) * B (Left) or
 * alpha * B * op(A) (Right) by naive triple loop in double.  Inputs are
 * widened to double by the caller-facing wrappers below. */
static int oracle_trmm_d(int side, int uplo, int trans, int diag, double alpha,
                         const double* a, int64_t lda, int64_t n,
                         const double* b, int64_t ldb, int64_t brows,
                         int64_t bcols, double* out /* brows x bcols, ld brows */) {
  if ((side == 0 ? brows : bcols) != n) return RO_SHAPE;
  double* M = materialize_op(a, lda, n, uplo, trans, diag);
  if (side == 0) {
    for (int64_t j = 0; j < bcols; ++j)
      for (int64_t i = 0; i < brows; ++i) {
        double acc = 0.0;
        for (int64_t k = 0; k < n; ++k) acc += M[k * n + i] * b[j * ldb + k];
        out[j * brows + i] = alpha * acc;
      }
  } else {
    for (int64_t j = 0; j < bcols; ++j)
      for (int64_t i = 0; i < brows; ++i) {
        double acc = 0.0;
        for (int64_t k = 0; k < n; ++k) acc += b[k * ldb + i] * M[j * n + k];
        out[j * brows + i] = alpha * acc;
      }
  }
  free(M);
  return RO_OK;
}

/* oracle_trsm: src/oracle.cpp:85-137.  Right is reduced to a Left solve on
 * the transposed system (:90-100); exact-zero diagonal -> singular (:101-102);
 * column-wise forward or back substitution in double (:115-130). */
static int oracle_trsm_d(int side, int uplo, int trans, int diag, double alpha,
                         const double* a, int64_t lda, int64_t n,
                         const double* b, int64_t ldb, int64_t brows,
                         int64_t bcols, double* out, int64_t* singular_row) {
  const int left = side == 0;
  if ((left ? brows : bcols) != n) return RO_SHAPE;
  double* M = materialize_op(a, lda, n, uplo, trans, diag);
  if (!left) {
    double* t = (double*)malloc(sizeof(double) * (size_t)(n * n + 1));
    for (int64_t c = 0; c < n; ++c)
      for (int64_t r = 0; r < n; ++r) t[c * n + r] = M[r * n + c];
    free(M);
    M = t;
  }
  for (int64_t r = 0; r < n; ++r)
    if (M[r * n + r] == 0.0) {
      if (singular_row) *singular_row = r;
      free(M);
      return RO_SINGULAR;
    }
  const int64_t k = left ? bcols : brows;
  const int eff_t = trans != 0;
  int lower = (uplo == 0) == (eff_t == 0);
  if (!left) lower = !lower;
  double* x = (double*)malloc(sizeof(double) * (size_t)(n * k + 1));
  for (int64_t c = 0; c < k; ++c) {
    if (lower) {
      for (int64_t r = 0; r < n; ++r) {
        double acc = alpha * (left ? b[c * ldb + r] : b[r * ldb + c]);
        for (int64_t j = 0; j < r; ++j) acc -= M[j * n + r] * x[c * n + j];
        x[c * n + r] = acc / M[r * n + r];
      }
    } else {
      for (int64_t r = n - 1; r >= 0; --r) {
        double acc = alpha * (left ? b[c * ldb + r] : b[r * ldb + c]);
        for (int64_t j = r + 1; j < n; ++j) acc -= M[j * n + r] * x[c * n + j];
        x[c * n + r] = acc / M[r * n + r];
      }
    }
  }
  for (int64_t c = 0; c < bcols; ++c)
    for (int64_t r = 0; r < brows; ++r)
      out[c * brows + r] = left ? x[c * n + r] : x[r * n + c];
  free(x);
  free(M);
  return RO_OK;
}

static double* widen_f32(const float* p, int64_t ld, int64_t rows, int64_t cols) {
  double* d = (double*)malloc(sizeof(double) * (size_t)(rows * cols + 1));
  for (int64_t c = 0; c < cols; ++c)
    for (int64_t r = 0; r < rows; ++r) d[c * rows + r] = (double)p[c * ld + r];
  return d;
}

int ro_oracle_trmm_f64(int side, int uplo, int trans, int diag, double alpha,
                       const double* a, int64_t lda, int64_t n, const double* b,
                       int64_t ldb, int64_t brows, int64_t bcols, double* out) {
  return oracle_trmm_d(side, uplo, trans, diag, alpha, a, lda, n, b, ldb, brows,
                       bcols, out);
}
int ro_oracle_trmm_f32(int side, int uplo, int trans, int diag, double alpha,
                       const float* a, int64_t lda, int64_t n, const float* b,
                       int64_t ldb, int64_t brows, int64_t bcols, double* out) {
  double* ad = widen_f32(a, lda, n, n);
  double* bd = widen_f32(b, ldb, brows, bcols);
  int rc = oracle_trmm_d(side, uplo, trans, diag, alpha, ad, n, n, bd, brows,
                         brows, bcols, out);
  free(ad);
  free(bd);
  return rc;
}
int ro_oracle_trsm_f64(int side, int uplo, int trans, int diag, double alpha,
                       const double* a, int64_t lda, int64_t n, const double* b,
                       int64_t ldb, int64_t brows, int64_t bcols, double* out,
                       int64_t* singular_row) {
  return oracle_trsm_d(side, uplo, trans, diag, alpha, a, lda, n, b, ldb, brows,
                       bcols, out, singular_row);
}
int ro_oracle_trsm_f32(int side, int uplo, int trans, int diag, double alpha,
                       const float* a, int64_t lda, int64_t n, const float* b,
                       int64_t ldb, int64_t brows, int64_t bcols, double* out,
                       int64_t* singular_row) {
  double* ad = widen_f32(a, lda, n, n);
  double* bd = widen_f32(b, ldb, brows, bcols);
  int rc = oracle_trsm_d(side, uplo, trans, diag, alpha, ad, n, n, bd, brows,
                         brows, bcols, out, singular_row);
  free(ad);
  free(bd);
  return rc;
}

/* Column-sampled oracle (the exact per-column form of the above, used where
 * the full O(n^2 m) oracle is too slow; cf. the sampled residual gate of
 * src/bench.cpp:100-165).  Left side only: columns of B are independent
 * (src/base_kernels.cpp:73-88), so oracle(B)[:, cols] == oracle(B[:, cols]).
 * Output is n x ncols (ld n). */
int ro_oracle_cols_f64(int is_trsm, int uplo, int trans, int diag,
                       double alpha, const double* a, int64_t lda, int64_t n,
                       const double* b, int64_t ldb, const int64_t* cols,
                       int64_t ncols, double* out, int64_t* singular_row) {
  double* bs = (double*)malloc(sizeof(double) * (size_t)(n * ncols + 1));
  for (int64_t j = 0; j < ncols; ++j)
    memcpy(bs + j * n, b + cols[j] * ldb, sizeof(double) * (size_t)n);
  int rc = is_trsm ? oracle_trsm_d(0, uplo, trans, diag, alpha, a, lda, n, bs,
                                   n, n, ncols, out, singular_row)
                   : oracle_trmm_d(0, uplo, trans, diag, alpha, a, lda, n, bs,
                                   n, n, ncols, out);
  free(bs);
  return rc;
}

/* ------------------------------------------------------------------------ */
/* Norms and residuals (tests/test_support.hpp:129-202). */

/* masked_norm_inf: tests/test_support.hpp:129-140 */
double ro_masked_norm_inf_f64(const double* a, int64_t lda, int64_t n, int uplo,
                              int diag) {
  double norm = 0.0;
  for (int64_t r = 0; r < n; ++r) {
    double sum = diag == 1 ? 1.0 : fabs(a[r * lda + r]);
    int64_t c0 = uplo == 0 ? 0 : r + 1, c1 = uplo == 0 ? r : n;
    for (int64_t c = c0; c < c1; ++c) sum += fabs(a[c * lda + r]);
    if (sum > norm) norm = sum;
  }
  return norm;
}

/* masked_op_entry: tests/test_support.hpp:144-152 */
static double masked_op_entry(const double* a, int64_t lda, int uplo, int diag,
                              int trans, int64_t i, int64_t k) {
  const int tr = trans != 0;
  const int64_t r = tr ? k : i, c = tr ? i : k;
  if (r == c) return diag == 1 ? 1.0 : a[r * lda + r];
  const int stored = uplo == 0 ? r > c : r < c;
  return stored ? a[c * lda + r] : 0.0;
}

/* trsm_residual_inf: tests/test_support.hpp:182-202.
 * max |op(A) X - alpha B| (Left) or |X op(A) - alpha B| (Right). */
double ro_trsm_residual_inf_f64(int side, int uplo, int trans, int diag,
                                double alpha, const double* a, int64_t lda,
                                int64_t n, const double* x, int64_t ldx,
                                const double* b, int64_t ldb, int64_t rows,
                                int64_t cols) {
  double worst = 0.0;
  for (int64_t c = 0; c < cols; ++c)
    for (int64_t i = 0; i < rows; ++i) {
      double lhs = 0.0;
      if (side == 0) {
        for (int64_t k = 0; k < n; ++k)
          lhs += masked_op_entry(a, lda, uplo, diag, trans, i, k) * x[c * ldx + k];
      } else {
        for (int64_t k = 0; k < n; ++k)
          lhs += x[k * ldx + i] * masked_op_entry(a, lda, uplo, diag, trans, k, c);
      }
      double d = fabs(lhs - alpha * b[c * ldb + i]);
      if (d > worst || d != d) worst = d != d ? INFINITY : (d > worst ? d : worst);
    }
  return worst;
}
