// fp64 DMMA GEMM, configuration 8: CTA 128x64x32, warps 4x2, 3 stages.
#include "gemm_f64_kernel.cuh"

namespace rectri_cu {
void dgemm_cfg8(const GemmParams<double>& p, bool ta, bool tb, bool vec2, cudaStream_t s) {
  dgemm::Config<128, 64, 32, 4, 2, 3>::run(p, ta, tb, vec2, s);
}
}  // namespace rectri_cu
