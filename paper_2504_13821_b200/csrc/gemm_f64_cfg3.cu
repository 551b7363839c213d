// fp64 DMMA GEMM, configuration 3: CTA 128x128x32, warps 4x4, 3 stages.
#include "gemm_f64_kernel.cuh"

namespace rectri_cu {
void dgemm_cfg3(const GemmParams<double>& p, bool ta, bool tb, bool vec2, cudaStream_t s) {
  dgemm::Config<128, 128, 32, 4, 4, 3>::run(p, ta, tb, vec2, s);
}
}  // namespace rectri_cu
