// TMA DMMA GEMM configuration 3: CTA 32x32x16, consumer warps 2x2 (16x16
// each), 4 stages, dedicated producer warp -- for updates with fewer 64x64
// tiles than the GPU has SMs (small calls, the short-K bottom levels): four
// times the CTAs for the same work, each with a quarter of the latency chain.
#include "gemm_f64_tma_cfgs.h"

namespace rectri_cu {
bool dgemm_tma_cfg3(const GemmParams<double>& p, bool ta, bool tb, cudaStream_t s) {
  return dgemm_tma::Config<32, 32, 2, 2, 4, true>::run(p, ta, tb, s);
}
}  // namespace rectri_cu
