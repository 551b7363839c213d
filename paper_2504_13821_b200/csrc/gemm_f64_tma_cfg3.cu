// TMA DMMA GEMM configuration 3: CTA 128x64x16, consumer warps 2x2, 5 stages,
// dedicated producer warp.
#include "gemm_f64_tma_cfgs.h"

namespace rectri_cu {
bool dgemm_tma_cfg3(const GemmParams<double>& p, bool ta, bool tb, cudaStream_t s) {
  return dgemm_tma::Config<128, 64, 2, 2, 5, true>::run(p, ta, tb, s);
}
}  // namespace rectri_cu
