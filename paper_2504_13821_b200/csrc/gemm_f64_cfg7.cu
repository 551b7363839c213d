// fp64 DMMA GEMM, configuration 7: CTA 64x128x32, warps 2x4, 3 stages.
#include "gemm_f64_kernel.cuh"

namespace rectri_cu {
void dgemm_cfg7(const GemmParams<double>& p, bool ta, bool tb, bool vec2, cudaStream_t s) {
  dgemm::Config<64, 128, 32, 2, 4, 3>::run(p, ta, tb, vec2, s);
}
}  // namespace rectri_cu
