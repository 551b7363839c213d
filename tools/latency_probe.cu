// Dependent-chain latencies on this GPU (cycles per op, one warp): DFMA,
// DMUL, 64-bit SHFL, LDS.64, DFMA->SHFL round trip, and DMMA m8n8k4 chain.
// Diagnostic for the leaf's substitution chain; not a bench number.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(double* out, long long* cyc, double a, double b, int which) {
  __shared__ double sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = 1.0 + i * 1e-9;
  __syncthreads();
  double x = a + threadIdx.x * 1e-12;
  const int N = 1024;
  long long t0 = clock64();
  if (which == 0) {
#pragma unroll 16
    for (int i = 0; i < N; ++i) x = fma(x, b, a);
  } else if (which == 1) {
#pragma unroll 16
    for (int i = 0; i < N; ++i) x = x * b;
  } else if (which == 2) {
#pragma unroll 16
    for (int i = 0; i < N; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31);
  } else if (which == 3) {
    int idx = threadIdx.x;
#pragma unroll 16
    for (int i = 0; i < N; ++i) {
      x = sm[idx & 1023];
      idx = static_cast<int>(x) + i;
    }
  } else if (which == 4) {
#pragma unroll 16
    for (int i = 0; i < N; ++i) x = __shfl_sync(0xffffffffu, fma(x, b, a), i & 31);
  } else if (which == 5) {
    double c0 = x, c1 = x;
#pragma unroll 16
    for (int i = 0; i < N; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
    x = c0 + c1;
  }
  long long t1 = clock64();
  out[threadIdx.x + blockIdx.x * blockDim.x] = x;
  if (threadIdx.x == 0) cyc[blockIdx.x] = (t1 - t0);
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 20);
  cudaMalloc(&cyc, 1 << 16);
  const char* names[] = {"DFMA", "DMUL", "SHFL64", "LDS64", "DFMA+SHFL", "DMMA884"};
  for (int w = 0; w < 6; ++w) {
    k<<<1, 32>>>(out, cyc, 1.0000001, 0.9999999, w);
    k<<<1, 32>>>(out, cyc, 1.0000001, 0.9999999, w);
    long long h;
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    std::printf("{\"probe\":\"latency\",\"op\":\"%s\",\"cycles_per_op\":%.1f}\n", names[w], h / 1024.0);
  }
  return 0;
}
