// fp64 DMMA GEMM, configuration 0: CTA 128x128x16, warps 2x4, 4 stages.
#include "gemm_f64_kernel.cuh"

namespace rectri_cu {
void dgemm_cfg0(const GemmParams<double>& p, bool ta, bool tb, bool vec2, cudaStream_t s) {
  dgemm::Config<128, 128, 16, 2, 4, 4>::run(p, ta, tb, vec2, s);
}
}  // namespace rectri_cu
