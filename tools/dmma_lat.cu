// DMMA.8x8x4 latency / per-warp issue probe (sm_100a): cycles per DMMA for
// C independent accumulator chains in W warps of one CTA on one SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_lat tools/dmma_lat.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int C>
__global__ void chain(double* out, long long* cyc, int iters) {
  double acc[C][2];
#pragma unroll
  for (int c = 0; c < C; ++c) acc[c][0] = acc[c][1] = 0.0;
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < C; ++c)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[c][0]), "+d"(acc[c][1]) : "d"(a), "d"(b));
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < C; ++c) s += acc[c][0] + acc[c][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int C>
void run(int warps, double* out, long long* cyc) {
  const int iters = 4096;
  chain<C><<<1, 32 * warps>>>(out, cyc, iters);
  chain<C><<<1, 32 * warps>>>(out, cyc, iters);
  cudaDeviceSynchronize();
  long long h = 0;
  cudaMemcpy(&h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  const double per = static_cast<double>(h) / iters;
  printf("chains %2d warps %2d: %.1f cycles per iteration, %.2f cycles per DMMA per warp, SM rate %.1f FMA/clk\n",
         C, warps, per, per / C, 256.0 * C * warps / per);
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 20);
  cudaMalloc(&cyc, 1 << 12);
  for (int w : {1, 2, 4, 8, 16}) {
    run<1>(w, out, cyc);
    run<2>(w, out, cyc);
    run<4>(w, out, cyc);
    run<8>(w, out, cyc);
    run<16>(w, out, cyc);
  }
  return 0;
}
