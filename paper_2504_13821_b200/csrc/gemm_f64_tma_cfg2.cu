// TMA DMMA GEMM configuration 2: CTA 128x128x16, consumer warps 2x4, 4 stages,
// dedicated producer warp.
#include "gemm_f64_tma_cfgs.h"

namespace rectri_cu {
bool dgemm_tma_cfg2(const GemmParams<double>& p, bool ta, bool tb, cudaStream_t s) {
  return dgemm_tma::Config<128, 128, 2, 4, 4, true>::run(p, ta, tb, s);
}
}  // namespace rectri_cu
