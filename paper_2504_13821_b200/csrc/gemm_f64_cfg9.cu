// fp64 DMMA GEMM, configuration 9: CTA 64x64x32, warps 2x2, 3 stages.
#include "gemm_f64_kernel.cuh"

namespace rectri_cu {
void dgemm_cfg9(const GemmParams<double>& p, bool ta, bool tb, bool vec2, cudaStream_t s) {
  dgemm::Config<64, 64, 32, 2, 2, 3>::run(p, ta, tb, vec2, s);
}
}  // namespace rectri_cu
