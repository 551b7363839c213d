// TMA DMMA GEMM configuration 2: CTA 64x64x16, consumer warps 2x2, 6 stages,
// dedicated producer warp.
#include "gemm_f64_tma_cfgs.h"

namespace rectri_cu {
bool dgemm_tma_cfg2(const GemmParams<double>& p, bool ta, bool tb, cudaStream_t s) {
  return dgemm_tma::Config<64, 64, 2, 2, 6, true>::run(p, ta, tb, s);
}
}  // namespace rectri_cu
