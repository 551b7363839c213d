// fp64 DMMA GEMM, configuration 13: CTA 128x64x16, warps 2x2, 4 stages.
#include "gemm_f64_kernel.cuh"

namespace rectri_cu {
void dgemm_cfg13(const GemmParams<double>& p, bool ta, bool tb, bool vec2, cudaStream_t s) {
  dgemm::Config<128, 64, 16, 2, 2, 4>::run(p, ta, tb, vec2, s);
}
}  // namespace rectri_cu
