// TMA DMMA GEMM configuration 4: CTA 64x128x16, consumer warps 2x2, 4 stages,
// dedicated producer warp.
#include "gemm_f64_tma_cfgs.h"

namespace rectri_cu {
bool dgemm_tma_cfg4(const GemmParams<double>& p, bool ta, bool tb, cudaStream_t s) {
  return dgemm_tma::Config<64, 128, 2, 2, 4, true>::run(p, ta, tb, s);
}
}  // namespace rectri_cu
