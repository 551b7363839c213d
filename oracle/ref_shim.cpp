// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" wrappers over the UNMODIFIED reference library, compiled by
// oracle/Makefile from the reference's own sources where they lie under
// /root/reference/proj (nothing is copied into this repo).  The resulting
// oracle/_ref/librectri_ref.so is used (a) to pin the C restatement in
// oracle/rectri_oracle.c against the reference's outputs and (b) as the CPU
// baseline (bench.py cpu_baseline, kind "reference"; bench.py --impl
// reference).  The product path never loads it.
//
// Wrapped reference entry points (paths relative to /root/reference/proj):
//   rectri::rec_trmm / rec_trsm     include/rectri/recursion.hpp:66-86
//   rectri::trmm_base / trsm_base   include/rectri/base_kernels.hpp:15-30
//   rectri::gemm / scale            include/rectri/gemm.hpp:18-33
//   rectri::schema_for              include/rectri/recursion.hpp:58
//   rectri::oracle::oracle_trmm/... include/rectri/oracle.hpp:17-30
//   rectri::testing generators      tests/test_support.hpp:38-85
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "rectri/base_kernels.hpp"
#include "rectri/gemm.hpp"
#include "rectri/oracle.hpp"
#include "rectri/recursion.hpp"
#include "test_support.hpp"  // reference tests/test_support.hpp

using namespace rectri;

namespace {

thread_local std::string g_msg;

enum Status {
  kOk = 0,
  kConfig = 1,
  kShape = 2,
  kAlias = 3,
  kSingular = 4,
  kTileLimit = 5,
  kBounds = 7,
  kSplit = 8,
  kOther = 9,
};

TriangularSpec make(int side, int uplo, int trans, int diag, double alpha) {
  TriangularSpec s;
  s.side = side == 0 ? Side::Left : Side::Right;
  s.uplo = uplo == 0 ? Uplo::Lower : Uplo::Upper;
  s.trans = trans == 0 ? Trans::NoTrans
                       : (trans == 1 ? Trans::Trans : Trans::ConjTrans);
  s.diag = diag == 0 ? Diag::NonUnit : Diag::Unit;
  s.alpha = alpha;
  return s;
}

Backend backend_of(int width) {
  if (width == 0) return Backend::seq();
  return Backend::par(width < 0 ? 0 : width);
}

template <typename F>
int guarded(F&& f, int64_t* err_index) {
  try {
    f();
    return kOk;
  } catch (const SingularityError& e) {
    g_msg = e.what();
    if (err_index) *err_index = e.index();
    return kSingular;
  } catch (const ConfigError& e) {
    g_msg = e.what();
    return kConfig;
  } catch (const ShapeError& e) {
    g_msg = e.what();
    return kShape;
  } catch (const AliasError& e) {
    g_msg = e.what();
    return kAlias;
  } catch (const TileLimitError& e) {
    g_msg = e.what();
    return kTileLimit;
  } catch (const BoundsError& e) {
    g_msg = e.what();
    return kBounds;
  } catch (const SplitError& e) {
    g_msg = e.what();
    return kSplit;
  } catch (const std::exception& e) {
    g_msg = e.what();
    return kOther;
  }
}

// Event trace sink: triples (event, n, m) appended while capacity lasts.
struct Trace {
  int64_t* buf;
  int64_t cap;
  int64_t* count;
};

EventSink sink_of(Trace t) {
  if (!t.buf || !t.count) return {};
  return [t](RecEvent e, index_t n, index_t m) {
    const int64_t i = *t.count;
    if (i < t.cap) {
      t.buf[3 * i + 0] = static_cast<int64_t>(e);
      t.buf[3 * i + 1] = n;
      t.buf[3 * i + 2] = m;
    }
    *t.count = i + 1;
  };
}

template <typename T>
int rec_call(bool trsm, int side, int uplo, int trans, int diag, double alpha,
             const T* a, int64_t n, T* b, int64_t brows, int64_t bcols,
             int64_t threshold, int width, int64_t* trace, int64_t trace_cap,
             int64_t* trace_count, int64_t* err_index) {
  return guarded(
      [&] {
        const TriangularSpec spec = make(side, uplo, trans, diag, alpha);
        MatrixView<const T> A(a, n, n, 0, 0, n, n);
        MatrixView<T> B(b, brows, bcols, 0, 0, brows, bcols);
        const Backend be = backend_of(width);
        const EventSink sink = sink_of(Trace{trace, trace_cap, trace_count});
        if (trsm)
          rec_trsm<T>(spec, A, B, Threshold{threshold}, be, sink);
        else
          rec_trmm<T>(spec, A, B, Threshold{threshold}, be, sink);
      },
      err_index);
}

template <typename T>
int base_call(bool trsm, int side, int uplo, int trans, int diag, double alpha,
              const T* a, int64_t n, T* b, int64_t brows, int64_t bcols,
              int64_t tile_limit, int width, int64_t* err_index) {
  return guarded(
      [&] {
        const TriangularSpec spec = make(side, uplo, trans, diag, alpha);
        MatrixView<const T> A(a, n, n, 0, 0, n, n);
        MatrixView<T> B(b, brows, bcols, 0, 0, brows, bcols);
        if (trsm)
          trsm_base<T>(spec, A, B, tile_limit, backend_of(width));
        else
          trmm_base<T>(spec, A, B, tile_limit, backend_of(width));
      },
      err_index);
}

template <typename T>
int oracle_call(bool trsm, int side, int uplo, int trans, int diag,
                double alpha, const T* a, int64_t n, const T* b, int64_t brows,
                int64_t bcols, double* out, int64_t* err_index) {
  return guarded(
      [&] {
        const TriangularSpec spec = make(side, uplo, trans, diag, alpha);
        MatrixView<const T> A(a, n, n, 0, 0, n, n);
        MatrixView<const T> B(b, brows, bcols, 0, 0, brows, bcols);
        MatrixBuffer<double> r = trsm ? oracle::oracle_trsm<T>(spec, A, B)
                                      : oracle::oracle_trmm<T>(spec, A, B);
        std::memcpy(out, r.data(), sizeof(double) * brows * bcols);
      },
      err_index);
}

}  // namespace

extern "C" {

const char* rref_last_error() { return g_msg.c_str(); }

#define RREF_REC(NAME, T, TRSM)                                                \
  int NAME(int side, int uplo, int trans, int diag, double alpha, const T* a,  \
           int64_t n, T* b, int64_t brows, int64_t bcols, int64_t threshold,   \
           int width, int64_t* trace, int64_t trace_cap, int64_t* trace_count, \
           int64_t* err_index) {                                               \
    return rec_call<T>(TRSM, side, uplo, trans, diag, alpha, a, n, b, brows,   \
                       bcols, threshold, width, trace, trace_cap, trace_count, \
                       err_index);                                             \
  }
RREF_REC(rref_rec_trsm_f64, double, true)
RREF_REC(rref_rec_trsm_f32, float, true)
RREF_REC(rref_rec_trmm_f64, double, false)
RREF_REC(rref_rec_trmm_f32, float, false)

#define RREF_BASE(NAME, T, TRSM)                                               \
  int NAME(int side, int uplo, int trans, int diag, double alpha, const T* a,  \
           int64_t n, T* b, int64_t brows, int64_t bcols, int64_t tile_limit,  \
           int width, int64_t* err_index) {                                    \
    return base_call<T>(TRSM, side, uplo, trans, diag, alpha, a, n, b, brows,  \
                        bcols, tile_limit, width, err_index);                  \
  }
RREF_BASE(rref_trsm_base_f64, double, true)
RREF_BASE(rref_trsm_base_f32, float, true)
RREF_BASE(rref_trmm_base_f64, double, false)
RREF_BASE(rref_trmm_base_f32, float, false)

#define RREF_ORACLE(NAME, T, TRSM)                                             \
  int NAME(int side, int uplo, int trans, int diag, double alpha, const T* a,  \
           int64_t n, const T* b, int64_t brows, int64_t bcols, double* out,   \
           int64_t* err_index) {                                               \
    return oracle_call<T>(TRSM, side, uplo, trans, diag, alpha, a, n, b,       \
                          brows, bcols, out, err_index);                       \
  }
RREF_ORACLE(rref_oracle_trsm_f64, double, true)
RREF_ORACLE(rref_oracle_trsm_f32, float, true)
RREF_ORACLE(rref_oracle_trmm_f64, double, false)
RREF_ORACLE(rref_oracle_trmm_f32, float, false)

// C <- alpha * op(A) * op(B) + beta * C, all contiguous column-major.
int rref_gemm_f64(double alpha, int ta, const double* a, int64_t ar, int64_t ac,
                  int tb, const double* b, int64_t br, int64_t bc, double beta,
                  double* c, int64_t cr, int64_t cc, int width) {
  return guarded(
      [&] {
        MatrixView<const double> A(a, ar, ac, 0, 0, ar, ac);
        MatrixView<const double> B(b, br, bc, 0, 0, br, bc);
        MatrixView<double> C(c, cr, cc, 0, 0, cr, cc);
        gemm<double>(alpha, ta ? Trans::Trans : Trans::NoTrans, A,
                     tb ? Trans::Trans : Trans::NoTrans, B, beta, C,
                     backend_of(width));
      },
      nullptr);
}

// schema_for(op, spec): out = {first_is_a22, off_trans, off_on_left,
// read_half(0=B1), write_half, sign, carries_alpha, second_is_a22}.
void rref_schema_for(int trsm, int side, int uplo, int trans, double* out) {
  const RecursionSchema s =
      schema_for(trsm ? OpKind::Trsm : OpKind::Trmm, make(side, uplo, trans, 0, 1.0));
  out[0] = s.first_block == DiagBlock::A22;
  out[1] = s.update.off_trans == Trans::NoTrans ? 0 : 1;
  out[2] = s.update.off_on_left;
  out[3] = s.update.read_half == BHalf::B2;
  out[4] = s.update.write_half == BHalf::B2;
  out[5] = s.update.sign;
  out[6] = s.update.carries_alpha;
  out[7] = s.second_block == DiagBlock::A22;
}

void rref_make_random_f64(double* out, int64_t rows, int64_t cols,
                          uint64_t seed, double lo, double hi) {
  auto m = testing::make_random<double>(rows, cols, seed, lo, hi);
  std::memcpy(out, m.data(), sizeof(double) * rows * cols);
}
void rref_make_random_f32(float* out, int64_t rows, int64_t cols, uint64_t seed,
                          double lo, double hi) {
  auto m = testing::make_random<float>(rows, cols, seed, lo, hi);
  std::memcpy(out, m.data(), sizeof(float) * rows * cols);
}
void rref_make_dominant_f64(double* out, int64_t n, int uplo, uint64_t seed) {
  auto m = testing::make_dominant<double>(n, uplo == 0 ? Uplo::Lower : Uplo::Upper,
                                          seed);
  std::memcpy(out, m.data(), sizeof(double) * n * n);
}
void rref_make_dominant_f32(float* out, int64_t n, int uplo, uint64_t seed) {
  auto m = testing::make_dominant<float>(n, uplo == 0 ? Uplo::Lower : Uplo::Upper,
                                         seed);
  std::memcpy(out, m.data(), sizeof(float) * n * n);
}
void rref_damp_off_diagonal_f64(double* a, int64_t n, double factor) {
  MatrixBuffer<double> m(n, n);
  std::memcpy(m.data(), a, sizeof(double) * n * n);
  testing::damp_off_diagonal(m, factor);
  std::memcpy(a, m.data(), sizeof(double) * n * n);
}
void rref_damp_off_diagonal_f32(float* a, int64_t n, double factor) {
  MatrixBuffer<float> m(n, n);
  std::memcpy(m.data(), a, sizeof(float) * n * n);
  testing::damp_off_diagonal(m, factor);
  std::memcpy(a, m.data(), sizeof(float) * n * n);
}
double rref_masked_norm_inf_f64(const double* a, int64_t n, int uplo, int diag) {
  MatrixBuffer<double> m(n, n);
  std::memcpy(m.data(), a, sizeof(double) * n * n);
  return testing::masked_norm_inf(m, uplo == 0 ? Uplo::Lower : Uplo::Upper,
                                  diag == 0 ? Diag::NonUnit : Diag::Unit);
}

}  // extern "C"
