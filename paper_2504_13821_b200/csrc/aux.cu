// aux.cu -- HBM-bound helpers: scale (src/gemm.cpp:218-227) and the
// exact-zero pivot pre-scan (src/base_kernels.cpp:166-169).
#include "common.cuh"
#include "launch.h"

namespace rectri_cu {
namespace {

// B <- alpha * B over a strided rows x cols window: one plain IEEE multiply
// per element (no NaN clearing, as the reference).  Grid sized in multiples
// of the SM count; each CTA walks whole columns so accesses coalesce.
template <typename T>
__global__ void scale_kernel(T* B, i64 ld, i64 rows, i64 cols, T alpha) {
  pdl_wait();  // PDL: no-op unless launched programmatically (launch_kernel)
  const i64 total = rows * cols;
  for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 c = i / rows, r = i - c * rows;
    T* x = B + r + c * ld;
    *x = *x * alpha;
  }
}

// D <- fma(c, S, D) over a rows x cols window (S packed, ld = rows): the
// epilogue of a GEMM update with beta = 1, applied to a product that was
// computed into S with alpha = 1, beta = 0 -- the same single rounding.
template <typename T>
__global__ void accumulate_kernel(T* D, i64 ldd, const T* S, i64 rows, i64 cols, T c) {
  pdl_wait();  // PDL: no-op unless launched programmatically (launch_kernel)
  const i64 total = rows * cols;
  for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 col = i / rows, r = i - col * rows;
    T* d = D + r + col * ldd;
    *d = fma(c, S[i], *d);
  }
}

template <typename T>
__global__ void diag_zero_scan_kernel(const T* A, i64 lda, i64 n, uint8_t* flags) {
  pdl_wait();  // PDL: no-op unless launched programmatically (launch_kernel)
  for (i64 r = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; r < n;
       r += static_cast<i64>(gridDim.x) * blockDim.x)
    flags[r] = A[r + r * lda] == T(0) ? 1 : 0;
}

int sm_count() {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

template <typename T>
void scale(T* B, i64 ld, i64 rows, i64 cols, T alpha, cudaStream_t s) {
  if (rows <= 0 || cols <= 0) return;
  const i64 total = rows * cols;
  const i64 want = ceil_div(total, 256);
  const unsigned grid = static_cast<unsigned>(want < 8 * sm_count() ? want : 8 * sm_count());
  launch_kernel(scale_kernel<T>, grid, 256, 0, s, B, ld, rows, cols, alpha);
  ++launch_counter();
}

template <typename T>
void accumulate(T* D, i64 ldd, const T* S, i64 rows, i64 cols, T c, cudaStream_t s) {
  if (rows <= 0 || cols <= 0) return;
  const i64 want = ceil_div(rows * cols, 256);
  const unsigned grid = static_cast<unsigned>(want < 8 * sm_count() ? want : 8 * sm_count());
  launch_kernel(accumulate_kernel<T>, grid, 256, 0, s, D, ldd, S, rows, cols, c);
  ++launch_counter();
}

template <typename T>
void scan(const T* A, i64 lda, i64 n, uint8_t* flags, cudaStream_t s) {
  if (n <= 0) return;
  const unsigned grid = static_cast<unsigned>(ceil_div(n, 256) < sm_count() ? ceil_div(n, 256) : sm_count());
  launch_kernel(diag_zero_scan_kernel<T>, grid, 256, 0, s, A, lda, n, flags);
  ++launch_counter();
}

}  // namespace

i64& launch_counter() {
  static i64 count = 0;
  return count;
}

void launch_scale_f64(double* B, i64 ld, i64 rows, i64 cols, double alpha, cudaStream_t s) {
  scale<double>(B, ld, rows, cols, alpha, s);
}
void launch_scale_f32(float* B, i64 ld, i64 rows, i64 cols, float alpha, cudaStream_t s) {
  scale<float>(B, ld, rows, cols, alpha, s);
}
void launch_accumulate_f64(double* D, i64 ldd, const double* S, i64 rows, i64 cols, double c, cudaStream_t s) {
  accumulate<double>(D, ldd, S, rows, cols, c, s);
}
void launch_accumulate_f32(float* D, i64 ldd, const float* S, i64 rows, i64 cols, float c, cudaStream_t s) {
  accumulate<float>(D, ldd, S, rows, cols, c, s);
}
void launch_diag_zero_scan_f64(const double* A, i64 lda, i64 n, uint8_t* flags, cudaStream_t s) {
  scan<double>(A, lda, n, flags, s);
}
void launch_diag_zero_scan_f32(const float* A, i64 lda, i64 n, uint8_t* flags, cudaStream_t s) {
  scan<float>(A, lda, n, flags, s);
}

}  // namespace rectri_cu

// ---------------------------------------------------------------------------
// Synthetic-input utilities (the device-side counterpart of the reference's
// bench generators, src/bench.cpp:32-61): a counter-based uniform[-1, 1)
// fill keyed by the GLOBAL element index, so a column shard generated on any
// GPU holds exactly the values of the same columns of the unsharded matrix;
// and the diagonal-dominance fixup (diag := stored off-diagonal |row sum| + 1).
namespace rectri_cu {
namespace {

__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

template <typename T>
__global__ void fill_uniform_kernel(T* B, i64 ld, i64 rows, i64 cols, i64 col0, i64 global_rows,
                                    uint64_t seed) {
  const i64 total = rows * cols;
  for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 c = i / rows, r = i - c * rows;
    const uint64_t id = static_cast<uint64_t>((col0 + c) * global_rows + r);
    const uint64_t z = splitmix64(seed * 0xd1b54a32d192ed03ull ^ id);
    const double u = static_cast<double>(z >> 11) * 0x1.0p-53;  // [0, 1)
    B[r + c * ld] = static_cast<T>(2.0 * u - 1.0);
  }
}

template <typename T>
__global__ void dominant_kernel(T* A, i64 lda, i64 n, int upper) {
  const i64 r = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (r >= n) return;
  double s = 0.0;
  if (!upper)
    for (i64 c = 0; c < r; ++c) s += fabs(static_cast<double>(A[r + c * lda]));
  else
    for (i64 c = r + 1; c < n; ++c) s += fabs(static_cast<double>(A[r + c * lda]));
  A[r + r * lda] = static_cast<T>(s + 1.0);
}

constexpr int kProbeChains = 8;
__global__ void probe_dmma_kernel(double* out, int iters) {
  double acc[kProbeChains][2];
  for (int c = 0; c < kProbeChains; ++c) acc[c][0] = acc[c][1] = 0.0;
  const double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int c = 0; c < kProbeChains; ++c) dmma884(acc[c][0], acc[c][1], a, b);
  double s = 0;
  for (int c = 0; c < kProbeChains; ++c) s += acc[c][0] + acc[c][1];
  if (s == 12345.678) out[0] = s;
}
// FFMA2 (fma.rn.f32x2), the instruction of the fp32 GEMM: 73.8 TF/s on
// B200 against 71 for scalar FFMA (profiles/r02_fp32_ffma_roofline.txt).
__global__ void probe_ffma_kernel(float* out, int iters) {
  unsigned long long acc[kProbeChains];
  unsigned long long x, y;
  asm("mov.b64 %0, {%1, %1};" : "=l"(x) : "f"(0.999999f));
  asm("mov.b64 %0, {%1, %1};" : "=l"(y) : "f"(1e-7f));
  for (int c = 0; c < kProbeChains; ++c) {
    const float v = threadIdx.x * 1e-3f + c;
    asm("mov.b64 %0, {%1, %1};" : "=l"(acc[c]) : "f"(v));
  }
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int c = 0; c < kProbeChains; ++c) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(acc[c]) : "l"(x), "l"(y));
  float s = 0;
  for (int c = 0; c < kProbeChains; ++c) {
    float lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(acc[c]));
    s += lo + hi;
  }
  if (s == 12345.678f) out[0] = s;
}

}  // namespace

void launch_fill_uniform_f64(double* B, i64 ld, i64 rows, i64 cols, i64 col0, i64 grows,
                             uint64_t seed, cudaStream_t s) {
  if (rows <= 0 || cols <= 0) return;
  fill_uniform_kernel<double><<<8 * sm_count(), 256, 0, s>>>(B, ld, rows, cols, col0, grows, seed);
  ++launch_counter();
}
void launch_fill_uniform_f32(float* B, i64 ld, i64 rows, i64 cols, i64 col0, i64 grows,
                             uint64_t seed, cudaStream_t s) {
  if (rows <= 0 || cols <= 0) return;
  fill_uniform_kernel<float><<<8 * sm_count(), 256, 0, s>>>(B, ld, rows, cols, col0, grows, seed);
  ++launch_counter();
}
void launch_make_dominant_f64(double* A, i64 lda, i64 n, int upper, cudaStream_t s) {
  if (n <= 0) return;
  dominant_kernel<double><<<static_cast<unsigned>(ceil_div(n, 128)), 128, 0, s>>>(A, lda, n, upper);
  ++launch_counter();
}
void launch_make_dominant_f32(float* A, i64 lda, i64 n, int upper, cudaStream_t s) {
  if (n <= 0) return;
  dominant_kernel<float><<<static_cast<unsigned>(ceil_div(n, 128)), 128, 0, s>>>(A, lda, n, upper);
  ++launch_counter();
}

// Measured issue-rate peak (TFLOP/s) of DMMA.8x8x4 (kind 0) or FFMA2 (kind 1)
// on the current device: 4 CTAs x 8 warps per SM, 8 independent chains.
double probe_peak_tflops(int kind) {
  void* buf = nullptr;
  if (cudaMalloc(&buf, 64) != cudaSuccess) return -1.0;
  const int grid = 4 * sm_count(), threads = 256;
  const int iters = kind == 0 ? 4096 : 16384;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0);
    if (kind == 0) probe_dmma_kernel<<<grid, threads>>>(static_cast<double*>(buf), iters);
    else probe_ffma_kernel<<<grid, threads>>>(static_cast<float*>(buf), iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 0 && ms < best) best = ms;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(buf);
  const double per_chain = kind == 0 ? 8.0 * 8 * 4 * 2 / 32 : 4.0;  // flops per lane per step
  const double lanes = static_cast<double>(grid) * threads;
  const double flops = lanes * iters * kProbeChains * per_chain;
  return cudaGetLastError() == cudaSuccess ? flops / (best * 1e-3) / 1e12 : -1.0;
}

int smem_carveout_pct() {
  static const int pct = [] {
    const char* e = getenv("RECTRI_CU_SMEM_CARVEOUT");
    return e ? atoi(e) : static_cast<int>(cudaSharedmemCarveoutMaxShared);
  }();
  return pct;
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("RECTRI_CU_PDL");
    return !e || atoi(e) != 0;
  }();
  return on;
}

}  // namespace rectri_cu
