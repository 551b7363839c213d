// fp64 DMMA GEMM (cp.async), configuration 1: CTA 64x64x16, warps 4x2, 4 stages.
#include "gemm_f64_kernel.cuh"

namespace rectri_cu {
void dgemm_cfg1(const GemmParams<double>& p, bool ta, bool tb, bool vec2, cudaStream_t s) {
  dgemm::Config<64, 64, 16, 4, 2, 4>::run(p, ta, tb, vec2, s);
}
}  // namespace rectri_cu
