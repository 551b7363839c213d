// gemm_f64.cu -- configuration choice for the fp64 DMMA GEMM update.
//
// The kernel (gemm_f64_kernel.cuh) is instantiated per tile configuration in
// gemm_f64_cfg*.cu; this file only picks one per call.  Every configuration
// accumulates each output element over k in the same order, so the choice
// (which may depend on M, N, K) never changes a result bit -- the property
// the RHS-sharding invariant (P-GPU == 1-GPU) rests on.  Different BK values
// share that order: a k-tile of 32 is two k-tiles of 16 back to back.
#include <cstdlib>

#include "gemm_f64_kernel.cuh"
#include "gemm_f64_tma.cuh"

namespace rectri_cu {
namespace {

bool aligned16(const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15u) == 0; }

const DgemmRun kRuns[] = {
#define RECTRI_ENTRY(ID, BM, BN, BK, WM, WN, ST) dgemm_cfg##ID,
    RECTRI_DGEMM_CONFIGS(RECTRI_ENTRY)
#undef RECTRI_ENTRY
};
constexpr int kNumCfg = sizeof(kRuns) / sizeof(kRuns[0]);

int forced_config() {  // RECTRI_CU_GEMM64_CFG=<id> pins one configuration (tuning)
  static int v = [] {
    const char* e = getenv("RECTRI_CU_GEMM64_CFG");
    return e ? atoi(e) : -1;
  }();
  return v;
}

int choose(const GemmParams<double>& p) {
  const int f = forced_config();
  if (f >= 0 && f < kNumCfg) return f;
  // 64x64 CTAs: 4 warps (3 CTAs per SM) for the large levels, 8 warps (2 per
  // SM) when K <= 512 where more resident warps hide the short mainloop's
  // prologue/epilogue latency (profiles/r01_gemm_cfg_sweep.txt: round-1
  // configurations 6 and 17; the other 17 swept shapes are no longer built).
  // Both use 16-deep k-tiles: identical per-element arithmetic.
  return p.K <= 512 ? 1 : 0;
}

}  // namespace

// TMA-fed kernel configuration for a problem, or -1 for the cp.async kernel
// (identical bits either way).
// TMA config 1 (64x64 CTAs, producer warp, 4 stages) reaches 36.1-36.4 TF/s
// (97-98 % of the DMMA peak) from K = 8192 down to K = 1024 and, with the
// batched epilogue, also beats the cp.async kernels at K = 512 (29.0 vs 27.5)
// and K = 256 (19.8 vs 19.3) (profiles/r01_tma_gemm_sweep.txt).  Updates with
// fewer than ~4 64x64 tiles per SM are latency chains on a partly idle GPU:
// config 3 (32x32 CTAs) gives them four times the CTAs (fp64 TRSM n = m =
// 1024: 107.8 -> 93.3 us, n = 2048: 406.7 -> 383.5 us; profiles/r02_small_tiles.txt)
// (RECTRI_CU_GEMM64_SMALL_TILES: that threshold in 64x64 tiles, 0 = off).
// Inside a TRMM with concurrent halves (p.busy_gpu) the other half fills the
// GPU and the large tiles measured faster (n = 2048: 322.6 vs 327.4 us).
int choose_tma(const GemmParams<double>& p) {
  static const long long small = [] {
    const char* e = getenv("RECTRI_CU_GEMM64_SMALL_TILES");
    return e ? atoll(e) : 600LL;
  }();
  const long long tiles64 = ceil_div(p.M, 64) * ceil_div(p.N, 64);
  return !p.busy_gpu && tiles64 < small ? 3 : 1;
}

void launch_gemm_f64(const GemmParams<double>& p0, bool ta, bool tb, cudaStream_t s) {
  if (p0.M <= 0 || p0.N <= 0 || p0.K <= 0) return;
  GemmParams<double> p = p0;
  p.ring_check = leaf_ring_check_counter(&p.ring_plant);  // RECTRI_CU_RING_CHECK (TMA kernels)
  const int cfg = choose_tma(p);
  if (cfg == 1 && launch_gemm_f64_split(p, ta, tb, s)) return;
  if (launch_gemm_f64_tma(p, ta, tb, s, cfg)) return;
  const bool vec2 = aligned16(p.A) && aligned16(p.B) && (p.lda % 2 == 0) && (p.ldb % 2 == 0);
  kRuns[choose(p)](p, ta, tb, vec2, s);
}

}  // namespace rectri_cu
