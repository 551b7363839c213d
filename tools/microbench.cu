// Peak-rate probes for the roofline denominators this path needs but
// MEASURED_PEAKS.json does not carry (fp64 DMMA / DFMA, fp32 FFMA), plus the
// cuBLAS anchors the north star compares against (dgemm/dtrsm/dtrmm and the
// s variants at n = m = 16384). Prints one JSON object per probe.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench
//        tools/microbench.cu -lcublas
#include <cuda_runtime.h>
#include <cublas_v2.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#define CK(x)                                                              \
  do {                                                                     \
    cudaError_t e_ = (x);                                                  \
    if (e_ != cudaSuccess) {                                               \
      std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__,               \
                   cudaGetErrorString(e_));                                \
      std::exit(1);                                                        \
    }                                                                      \
  } while (0)
#define CB(x)                                                              \
  do {                                                                     \
    cublasStatus_t s_ = (x);                                               \
    if (s_ != CUBLAS_STATUS_SUCCESS) {                                     \
      std::fprintf(stderr, "%s:%d cublas %d\n", __FILE__, __LINE__, (int)s_); \
      std::exit(1);                                                        \
    }                                                                      \
  } while (0)

constexpr int kChains = 8;

__global__ void dmma884_loop(double* out, int iters) {
  double acc[kChains][2];
  for (int c = 0; c < kChains; ++c) acc[c][0] = acc[c][1] = 0.0;
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
      asm volatile(
          "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, "
          "{%0,%1};\n"
          : "+d"(acc[c][0]), "+d"(acc[c][1])
          : "d"(a), "d"(b));
    }
  }
  double s = 0;
  for (int c = 0; c < kChains; ++c) s += acc[c][0] + acc[c][1];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma16816_loop(double* out, int iters) {
  double acc[kChains][4];
  for (int c = 0; c < kChains; ++c)
    for (int j = 0; j < 4; ++j) acc[c][j] = 0.0;
  double a[8], b[4];
  for (int j = 0; j < 8; ++j) a[j] = 1.0 + (threadIdx.x + j) * 1e-9;
  for (int j = 0; j < 4; ++j) b[j] = 1.0 - (threadIdx.x + j) * 1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
          "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
          : "+d"(acc[c][0]), "+d"(acc[c][1]), "+d"(acc[c][2]), "+d"(acc[c][3])
          : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]),
            "d"(a[6]), "d"(a[7]), "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0;
  for (int c = 0; c < kChains; ++c)
    for (int j = 0; j < 4; ++j) s += acc[c][j];
  if (s == 12345.678) out[0] = s;
}

template <typename T>
__global__ void fma_loop(T* out, int iters) {
  T acc[kChains];
  for (int c = 0; c < kChains; ++c) acc[c] = T(threadIdx.x) * T(1e-3);
  const T a = T(0.999999), b = T(1e-7);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) acc[c] = fma(acc[c], a, b);
  }
  T s = 0;
  for (int c = 0; c < kChains; ++c) s += acc[c];
  if (s == T(12345.678)) out[0] = s;
}

template <typename K>
double time_kernel(K launch, int reps = 5) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  launch();
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(e0));
    launch();
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    if (ms < best) best = ms;
  }
  CK(cudaGetLastError());
  return best * 1e-3;
}

__global__ void fill_uniform(double* p, long long n, unsigned long long seed) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  for (; i < n; i += (long long)gridDim.x * blockDim.x) {
    unsigned long long z = seed + 0x9e3779b97f4a7c15ull * (unsigned long long)(i + 1);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    z ^= z >> 31;
    p[i] = 2.0 * ((z >> 11) * 0x1.0p-53) - 1.0;
  }
}
__global__ void to_f32(const double* s, float* d, long long n) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  for (; i < n; i += (long long)gridDim.x * blockDim.x) d[i] = (float)s[i];
}
// Diagonal of a lower-stored A set to (sum of |off-diagonal row| + 1).
template <typename T>
__global__ void make_dominant_lower(T* a, long long n) {
  long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (r >= n) return;
  double s = 0;
  for (long long c = 0; c < r; ++c) s += fabs((double)a[c * n + r]);
  a[r * n + r] = (T)(s + 1.0);
}

int main(int argc, char** argv) {
  int dev = 0;
  CK(cudaSetDevice(dev));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, dev));
  const int sms = prop.multiProcessorCount;
  std::printf("{\"probe\":\"device\",\"name\":\"%s\",\"sms\":%d,\"cc\":\"%d.%d\"}\n",
              prop.name, sms, prop.major, prop.minor);
  double* dout;
  CK(cudaMalloc(&dout, 64));
  const int iters = 4096;
  for (int wpb : {4, 8}) {
    for (int bps : {1, 2, 4}) {
      const int grid = sms * bps, threads = 32 * wpb;
      double t = time_kernel([&] { dmma884_loop<<<grid, threads>>>(dout, iters); });
      double flops = double(grid) * wpb * iters * kChains * 8 * 8 * 4 * 2;
      std::printf("{\"probe\":\"dmma_m8n8k4\",\"warps_per_block\":%d,\"blocks_per_sm\":%d,"
                  "\"tflops\":%.3f}\n", wpb, bps, flops / t / 1e12);
      t = time_kernel([&] { dmma16816_loop<<<grid, threads>>>(dout, iters / 4); });
      flops = double(grid) * wpb * (iters / 4) * kChains * 16 * 8 * 16 * 2;
      std::printf("{\"probe\":\"dmma_m16n8k16\",\"warps_per_block\":%d,\"blocks_per_sm\":%d,"
                  "\"tflops\":%.3f}\n", wpb, bps, flops / t / 1e12);
    }
  }
  for (int bps : {2, 4, 8}) {
    const int grid = sms * bps, threads = 256;
    double t = time_kernel([&] { fma_loop<double><<<grid, threads>>>(dout, iters); });
    double flops = double(grid) * threads * iters * kChains * 2;
    std::printf("{\"probe\":\"dfma\",\"blocks_per_sm\":%d,\"tflops\":%.3f}\n", bps,
                flops / t / 1e12);
    t = time_kernel([&] { fma_loop<float><<<grid, threads>>>((float*)dout, iters); });
    std::printf("{\"probe\":\"ffma\",\"blocks_per_sm\":%d,\"tflops\":%.3f}\n", bps,
                flops / t / 1e12);
  }

  // cuBLAS anchors.
  cublasHandle_t h;
  CB(cublasCreate(&h));
  const bool quick = argc > 1 && std::strcmp(argv[1], "quick") == 0;
  std::vector<long long> sizes = quick ? std::vector<long long>{4096}
                                       : std::vector<long long>{4096, 8192, 16384};
  for (long long n : sizes) {
    const long long nn = n * n;
    double *A, *B, *C;
    CK(cudaMalloc(&A, nn * 8));
    CK(cudaMalloc(&B, nn * 8));
    CK(cudaMalloc(&C, nn * 8));
    fill_uniform<<<1024, 256>>>(A, nn, 1);
    fill_uniform<<<1024, 256>>>(B, nn, 2);
    const double one = 1.0;
    const double zero = 0.0;
    double t = time_kernel([&] {
      CB(cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &one, A, n, B, n, &zero, C, n));
    }, 3);
    std::printf("{\"probe\":\"cublas_dgemm\",\"n\":%lld,\"tflops\":%.3f,\"ms\":%.3f}\n", n,
                2.0 * n * n * n / t / 1e12, t * 1e3);
    t = time_kernel([&] {
      CB(cublasDtrmm(h, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N,
                     CUBLAS_DIAG_NON_UNIT, n, n, &one, A, n, B, n, C, n));
    }, 3);
    std::printf("{\"probe\":\"cublas_dtrmm_LUN\",\"n\":%lld,\"gflops_n2m\":%.1f,\"ms\":%.3f}\n",
                n, double(n) * n * n / t / 1e9, t * 1e3);
    make_dominant_lower<double><<<(n + 255) / 256, 256>>>(A, n);
    CK(cudaDeviceSynchronize());
    t = time_kernel([&] {
      CK(cudaMemcpyAsync(C, B, nn * 8, cudaMemcpyDeviceToDevice));
      CB(cublasDtrsm(h, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N,
                     CUBLAS_DIAG_NON_UNIT, n, n, &one, A, n, C, n));
    }, 3);
    double tcopy = time_kernel([&] {
      CK(cudaMemcpyAsync(C, B, nn * 8, cudaMemcpyDeviceToDevice));
    }, 3);
    std::printf("{\"probe\":\"cublas_dtrsm_LLN\",\"n\":%lld,\"gflops_n2m\":%.1f,\"ms\":%.3f,"
                "\"copy_ms\":%.3f}\n", n, double(n) * n * n / (t - tcopy) / 1e9,
                (t - tcopy) * 1e3, tcopy * 1e3);
    std::printf("{\"probe\":\"d2d_copy\",\"bytes\":%lld,\"gbs\":%.1f}\n", nn * 8,
                2.0 * nn * 8 / tcopy / 1e9);
    // fp32
    float *Af = (float*)A, *Bf = (float*)B, *Cf = (float*)C;
    // reuse buffers: regenerate in f32
    double *tmp;
    CK(cudaMalloc(&tmp, nn * 8));
    fill_uniform<<<1024, 256>>>(tmp, nn, 1);
    to_f32<<<1024, 256>>>(tmp, Af, nn);
    fill_uniform<<<1024, 256>>>(tmp, nn, 2);
    to_f32<<<1024, 256>>>(tmp, Bf, nn);
    CK(cudaFree(tmp));
    const float onef = 1.f, zerof = 0.f;
    t = time_kernel([&] {
      CB(cublasSgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &onef, Af, n, Bf, n, &zerof, Cf, n));
    }, 3);
    std::printf("{\"probe\":\"cublas_sgemm\",\"n\":%lld,\"tflops\":%.3f,\"ms\":%.3f}\n", n,
                2.0 * n * n * n / t / 1e12, t * 1e3);
    t = time_kernel([&] {
      CB(cublasStrmm(h, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N,
                     CUBLAS_DIAG_NON_UNIT, n, n, &onef, Af, n, Bf, n, Cf, n));
    }, 3);
    std::printf("{\"probe\":\"cublas_strmm_LUN\",\"n\":%lld,\"gflops_n2m\":%.1f,\"ms\":%.3f}\n",
                n, double(n) * n * n / t / 1e9, t * 1e3);
    make_dominant_lower<float><<<(n + 255) / 256, 256>>>(Af, n);
    t = time_kernel([&] {
      CK(cudaMemcpyAsync(Cf, Bf, nn * 4, cudaMemcpyDeviceToDevice));
      CB(cublasStrsm(h, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N,
                     CUBLAS_DIAG_NON_UNIT, n, n, &onef, Af, n, Cf, n));
    }, 3);
    std::printf("{\"probe\":\"cublas_strsm_LLN\",\"n\":%lld,\"gflops_n2m\":%.1f,\"ms\":%.3f}\n",
                n, double(n) * n * n / (t - tcopy / 2) / 1e9, (t - tcopy / 2) * 1e3);
    CK(cudaFree(A));
    CK(cudaFree(B));
    CK(cudaFree(C));
    std::fflush(stdout);
  }
  CB(cublasDestroy(h));
  return 0;
}
