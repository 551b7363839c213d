// TMA DMMA GEMM configuration 5: CTA 128x128x16, consumer warps 2x4, 4 stages,
// producer = lane 0 of warp 0.
#include "gemm_f64_tma_cfgs.h"

namespace rectri_cu {
bool dgemm_tma_cfg5(const GemmParams<double>& p, bool ta, bool tb, cudaStream_t s) {
  return dgemm_tma::Config<128, 128, 2, 4, 4, false>::run(p, ta, tb, s);
}
}  // namespace rectri_cu
