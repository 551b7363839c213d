// mixprobe.cu -- do fp64 tensor (DMMA) and fp64 vector (DFMA) work share one
// pipe on sm_100a?  Each warp runs independent DMMA.8x8x4 chains and/or DFMA
// chains; the combined rate tells whether a GEMM could use both.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kMC = 8, kFC = 16;

template <bool DO_MMA, bool DO_FMA>
__global__ void mix(double* out, int iters) {
  double acc[kMC][2];
  double f[kFC];
  for (int c = 0; c < kMC; ++c) acc[c][0] = acc[c][1] = 0.0;
  for (int c = 0; c < kFC; ++c) f[c] = threadIdx.x * 1e-3 + c;
  const double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  const double x = 0.999999, y = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < kMC; ++c) {
      if (DO_MMA)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(acc[c][0]), "+d"(acc[c][1])
                     : "d"(a), "d"(b));
      if (DO_FMA) {
        f[2 * c] = fma(f[2 * c], x, y);
        f[2 * c + 1] = fma(f[2 * c + 1], x, y);
      }
    }
  }
  double s = 0;
  for (int c = 0; c < kMC; ++c) s += acc[c][0] + acc[c][1];
  for (int c = 0; c < kFC; ++c) s += f[c];
  if (s == 12345.678) out[0] = s;
}

template <typename K>
float timeit(K k) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    k();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  return best;
}

int main() {
  double* d;
  cudaMalloc(&d, 64);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 4096;
  for (int wpb : {4, 8, 16}) {
    const int grid = sms * 2, threads = 32 * wpb;
    const double mma_fl = double(grid) * wpb * iters * kMC * 8 * 8 * 4 * 2;
    const double fma_fl = double(grid) * threads * iters * kFC * 2;
    float t1 = timeit([&] { mix<true, false><<<grid, threads>>>(d, iters); });
    float t2 = timeit([&] { mix<false, true><<<grid, threads>>>(d, iters); });
    float t3 = timeit([&] { mix<true, true><<<grid, threads>>>(d, iters); });
    printf("{\"warps\": %d, \"dmma_only_tflops\": %.2f, \"dfma_only_tflops\": %.2f, \"mixed_ms\": %.3f, "
           "\"mixed_total_tflops\": %.2f, \"dmma_ms\": %.3f, \"dfma_ms\": %.3f}\n",
           wpb, mma_fl / t1 / 1e9, fma_fl / t2 / 1e9, t3, (mma_fl + fma_fl) / t3 / 1e9, t1, t2);
  }
  return 0;
}
