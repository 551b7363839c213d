// cublas_cmp.cu -- reported-comparison shim (NOT the product path): cuBLAS
// ?trsm / ?trmm / ?gemm on caller-provided device buffers, timed with CUDA
// events on the legacy stream.  Built into tools/libcublas_cmp.so by
// paper_2504_13821_b200/build.py; loaded only by bench.py.
#include <cublas_v2.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace {
cublasHandle_t handle() {
  static cublasHandle_t h = nullptr;
  if (!h) cublasCreate(&h);
  return h;
}
// reps <= 0: exactly one (timed) call, no warm-up -- for in-place solves whose
// result is checked afterwards.
template <typename F>
double timed(F f, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  if (reps > 0) f();
  else reps = 1;
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int i = 0; i < reps; ++i) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return best;
}
}  // namespace

extern "C" {
// Left/Lower/NoTrans/NonUnit in-place solve of A X = B (n x m), ms.
double cmp_dtrsm_lln(const double* A, int64_t n, double* B, int64_t m, int reps) {
  const double one = 1.0;
  return timed([&] {
    cublasDtrsm(handle(), CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, n, m, &one,
                A, n, B, n);
  }, reps);
}
// Left/Upper/NoTrans/NonUnit C = A B (out of place, as cuBLAS trmm), ms.
double cmp_dtrmm_lun(const double* A, int64_t n, const double* B, double* C, int64_t m, int reps) {
  const double one = 1.0;
  return timed([&] {
    cublasDtrmm(handle(), CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, n, m, &one, A,
                n, B, n, C, n);
  }, reps);
}
double cmp_dgemm(const double* A, const double* B, double* C, int64_t n, int reps) {
  const double one = 1.0, zero = 0.0;
  return timed([&] { cublasDgemm(handle(), CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &one, A, n, B, n, &zero, C, n); },
               reps);
}
double cmp_strsm_lln(const float* A, int64_t n, float* B, int64_t m, int reps) {
  const float one = 1.f;
  return timed([&] {
    cublasStrsm(handle(), CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, n, m, &one,
                A, n, B, n);
  }, reps);
}
double cmp_strmm_lun(const float* A, int64_t n, const float* B, float* C, int64_t m, int reps) {
  const float one = 1.f;
  return timed([&] {
    cublasStrmm(handle(), CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, n, m, &one, A,
                n, B, n, C, n);
  }, reps);
}
double cmp_sgemm(const float* A, const float* B, float* C, int64_t n, int reps) {
  const float one = 1.f, zero = 0.f;
  return timed([&] { cublasSgemm(handle(), CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &one, A, n, B, n, &zero, C, n); },
               reps);
}

// Any variant (0/1 flags as rectri_cu_spec: side 0 Left, uplo 0 Lower, trans
// 0 N / 1 T, diag 0 NonUnit; dtype 1 = f64, 0 = f32).  B is rows x cols
// (ld = rows); A is rows x rows (Left) or cols x cols (Right), ld lda.
// trsm solves in place; trmm is out of place (C = alpha op(A) B), ms.
double cmp_trsm(int dtype, int side, int uplo, int trans, int diag, const void* A, int64_t lda, void* B,
                int64_t rows, int64_t cols, int reps) {
  const cublasSideMode_t sd = side ? CUBLAS_SIDE_RIGHT : CUBLAS_SIDE_LEFT;
  const cublasFillMode_t ul = uplo ? CUBLAS_FILL_MODE_UPPER : CUBLAS_FILL_MODE_LOWER;
  const cublasOperation_t tr = trans ? CUBLAS_OP_T : CUBLAS_OP_N;
  const cublasDiagType_t dg = diag ? CUBLAS_DIAG_UNIT : CUBLAS_DIAG_NON_UNIT;
  if (dtype == 1) {
    const double one = 1.0;
    return timed([&] {
      cublasDtrsm(handle(), sd, ul, tr, dg, rows, cols, &one, static_cast<const double*>(A), lda,
                  static_cast<double*>(B), rows);
    }, reps);
  }
  const float one = 1.f;
  return timed([&] {
    cublasStrsm(handle(), sd, ul, tr, dg, rows, cols, &one, static_cast<const float*>(A), lda, static_cast<float*>(B),
                rows);
  }, reps);
}
double cmp_trmm(int dtype, int side, int uplo, int trans, int diag, const void* A, int64_t lda, const void* B,
                void* C, int64_t rows, int64_t cols, int reps) {
  const cublasSideMode_t sd = side ? CUBLAS_SIDE_RIGHT : CUBLAS_SIDE_LEFT;
  const cublasFillMode_t ul = uplo ? CUBLAS_FILL_MODE_UPPER : CUBLAS_FILL_MODE_LOWER;
  const cublasOperation_t tr = trans ? CUBLAS_OP_T : CUBLAS_OP_N;
  const cublasDiagType_t dg = diag ? CUBLAS_DIAG_UNIT : CUBLAS_DIAG_NON_UNIT;
  if (dtype == 1) {
    const double one = 1.0;
    return timed([&] {
      cublasDtrmm(handle(), sd, ul, tr, dg, rows, cols, &one, static_cast<const double*>(A), lda,
                  static_cast<const double*>(B), rows, static_cast<double*>(C), rows);
    }, reps);
  }
  const float one = 1.f;
  return timed([&] {
    cublasStrmm(handle(), sd, ul, tr, dg, rows, cols, &one, static_cast<const float*>(A), lda,
                static_cast<const float*>(B), rows, static_cast<float*>(C), rows);
  }, reps);
}
}
