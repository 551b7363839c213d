// TMA DMMA GEMM configuration 0: CTA 64x64x16, consumer warps 2x2, 4 stages,
// producer = lane 0 of warp 0.
#include "gemm_f64_tma_cfgs.h"

namespace rectri_cu {
bool dgemm_tma_cfg0(const GemmParams<double>& p, bool ta, bool tb, cudaStream_t s) {
  return dgemm_tma::Config<64, 64, 2, 2, 4, false>::run(p, ta, tb, s);
}
}  // namespace rectri_cu
