// fp64 DMMA GEMM, configuration 14: CTA 64x64x16, warps 2x1, 4 stages.
#include "gemm_f64_kernel.cuh"

namespace rectri_cu {
void dgemm_cfg14(const GemmParams<double>& p, bool ta, bool tb, bool vec2, cudaStream_t s) {
  dgemm::Config<64, 64, 16, 2, 1, 4>::run(p, ta, tb, vec2, s);
}
}  // namespace rectri_cu
