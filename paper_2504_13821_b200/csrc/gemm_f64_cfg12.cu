// fp64 DMMA GEMM, configuration 12: CTA 64x128x16, warps 2x2, 4 stages.
#include "gemm_f64_kernel.cuh"

namespace rectri_cu {
void dgemm_cfg12(const GemmParams<double>& p, bool ta, bool tb, bool vec2, cudaStream_t s) {
  dgemm::Config<64, 128, 16, 2, 2, 4>::run(p, ta, tb, vec2, s);
}
}  // namespace rectri_cu
