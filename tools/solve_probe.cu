// Microbenchmark of the leaf's 32x32 diagonal-block substitution variants
// (cycles per block solve, one CTA per SM, clock64 around each solve).
// Diagnostic for leaf64.cu; not a bench number.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kRB = 32;

// (a) 4 lanes per right-hand side, rows rq + 4k, shuffle broadcast of x
__device__ void solve_shfl(double* panel, const double* Ld, const double* dg, int lane, int sw) {
  const int cc = 8 * sw + (lane >> 2), rq = lane & 3;
  const unsigned grp = lane & ~3u;
  double v[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) v[k] = panel[(rq + 4 * k) * 32 + cc];
  double ln[8], dn = dg[rq];
#pragma unroll
  for (int k = 0; k < 8; ++k) ln[k] = Ld[rq + 4 * k];
#pragma unroll
  for (int q = 0; q < kRB; ++q) {
    const int kq = q >> 2, oq = q & 3;
    double lc[8];
#pragma unroll
    for (int k = kq; k < 8; ++k) lc[k] = ln[k];
    const double dc = dn;
    if (q + 1 < kRB) {
#pragma unroll
      for (int k = (q + 1) >> 2; k < 8; ++k) ln[k] = Ld[(q + 1) * kRB + rq + 4 * k];
      if (((q + 1) & 3) == 0) dn = dg[q + 1 + rq];
    }
    double x = 0.0;
    if (rq == oq) {
      x = v[kq] * dc;
      v[kq] = x;
    }
    x = __shfl_sync(0xffffffffu, x, grp | oq);
    {
      const double nv = fma(-lc[kq], x, v[kq]);
      v[kq] = rq > oq ? nv : v[kq];
    }
#pragma unroll
    for (int k = kq + 1; k < 8; ++k) v[k] = fma(-lc[k], x, v[k]);
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) panel[(rq + 4 * k) * 32 + cc] = v[k];
}

// (b) one lane per right-hand side, 32 rows in registers (one warp: 32 rhs)
__device__ void solve_lane(double* panel, const double* Ld, const double* dg, int lane) {
  double v[kRB];
#pragma unroll
  for (int r = 0; r < kRB; ++r) v[r] = panel[r * 32 + lane];
#pragma unroll
  for (int q = 0; q < kRB; ++q) {
    const double x = v[q] * dg[q];
    v[q] = x;
#pragma unroll
    for (int r = q + 1; r < kRB; ++r) v[r] = fma(-Ld[q * kRB + r], x, v[r]);
  }
#pragma unroll
  for (int r = 0; r < kRB; ++r) panel[r * 32 + lane] = v[r];
}

__global__ void probe(long long* out, int variant, int reps) {
  __shared__ double panel[32 * 32], Ld[32 * 32], dg[32];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) {
    panel[i] = 1.0 + 1e-3 * i;
    const int q = i >> 5, r = i & 31;
    Ld[i] = q < r ? 1e-3 * (i % 7) : 0.0;
  }
  if (threadIdx.x < 32) dg[threadIdx.x] = 1.0 / (2.0 + threadIdx.x);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  long long t0 = clock64();
  for (int it = 0; it < reps; ++it) {
    if (variant == 0) solve_shfl(panel, Ld, dg, lane, warp);
    else if (warp == 0) solve_lane(panel, Ld, dg, lane);
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = (t1 - t0) / reps;
}

int main() {
  long long* d;
  cudaMalloc(&d, 1024 * sizeof(long long));
  for (int variant = 0; variant < 2; ++variant)
    for (int per_sm = 1; per_sm <= 2; ++per_sm) {
      probe<<<148 * per_sm, 128>>>(d, variant, 64);
      probe<<<148 * per_sm, 128>>>(d, variant, 64);
      cudaDeviceSynchronize();
      long long h[296];
      cudaMemcpy(h, d, 148 * per_sm * sizeof(long long), cudaMemcpyDeviceToHost);
      double s = 0;
      for (int i = 0; i < 148 * per_sm; ++i) s += h[i];
      std::printf("{\"probe\":\"diag_solve\",\"variant\":\"%s\",\"ctas_per_sm\":%d,\"cycles_per_block\":%.0f}\n",
                  variant ? "lane_per_rhs" : "4lanes_shfl", per_sm, s / (148 * per_sm));
    }
  return 0;
}
