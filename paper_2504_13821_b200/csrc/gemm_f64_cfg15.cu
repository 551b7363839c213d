// fp64 DMMA GEMM, configuration 15: CTA 64x64x16, warps 2x2, 4 stages, MC layout mode 1.
#include "gemm_f64_kernel.cuh"

namespace rectri_cu {
void dgemm_cfg15(const GemmParams<double>& p, bool ta, bool tb, bool vec2, cudaStream_t s) {
  dgemm::Config<64, 64, 16, 2, 2, 4, 1>::run(p, ta, tb, vec2, s);
}
}  // namespace rectri_cu
