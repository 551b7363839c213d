// gemm_f64_tma_cfgs.h -- instantiated configurations of the TMA DMMA GEMM
// (one translation unit each, gemm_f64_tma_cfg*.cu) and their launcher.
#pragma once
#include "gemm_f64_tma.cuh"

namespace rectri_cu {

bool encode_operand(CUtensorMap* map, const double* X, i64 ld, i64 O, i64 K, int BO, bool outer_contig);

namespace dgemm_tma {
template <int BM, int BN, int WARPS_M, int WARPS_N, int STAGES, bool PRODUCER>
struct Config {
  template <bool MC_A, bool MC_B>
  static bool launch(const GemmParams<double>& p, cudaStream_t s) {
    CUtensorMap ma, mb;
    if (!encode_operand(&ma, p.A, p.lda, p.M, p.K, BM, MC_A)) return false;
    if (!encode_operand(&mb, p.B, p.ldb, p.N, p.K, BN, MC_B)) return false;
    auto kern = p.ring_check ? dgemm_tma_kernel<BM, BN, WARPS_M, WARPS_N, STAGES, PRODUCER, MC_A, MC_B, true>
                             : dgemm_tma_kernel<BM, BN, WARPS_M, WARPS_N, STAGES, PRODUCER, MC_A, MC_B>;
    constexpr int slot_a = ((MC_A ? BM + 4 : BM) * kBK * 8 + 1023) / 1024 * 1024;
    constexpr int slot_b = ((MC_B ? BN + 4 : BN) * kBK * 8 + 1023) / 1024 * 1024;
    constexpr int smem = STAGES * (slot_a + slot_b) + 16 * STAGES + 1024;
    set_smem(kern, smem);
    const unsigned grid = static_cast<unsigned>(ceil_div(p.M, BM) * ceil_div(p.N, BN));
    constexpr int threads = (WARPS_M * WARPS_N + (PRODUCER ? 1 : 0)) * 32;
    launch_kernel(kern, grid, threads, smem, s, ma, mb, p);
    ++launch_counter();
    return true;
  }
  // op(A) = A is outer(m)-contiguous; op(B) = B^T is outer(n)-contiguous.
  static bool run(const GemmParams<double>& p, bool ta, bool tb, cudaStream_t s) {
    if (!ta && !tb) return launch<true, false>(p, s);
    if (ta && !tb) return launch<false, false>(p, s);
    if (!ta && tb) return launch<true, true>(p, s);
    return launch<false, true>(p, s);
  }
};
}  // namespace dgemm_tma

using DgemmTmaRun = bool (*)(const GemmParams<double>&, bool, bool, cudaStream_t);
//                              ID  BM   BN  WM WN ST producer-warp
#define RECTRI_DGEMM_TMA_CONFIGS(X) \
  X(0, 64, 64, 2, 2, 4, false)      \
  X(1, 64, 64, 2, 2, 4, true)       \
  X(2, 64, 64, 2, 2, 6, true)       \
  X(3, 32, 32, 2, 2, 4, true)
#define RECTRI_DECL(ID, BM, BN, WM, WN, ST, PR) \
  bool dgemm_tma_cfg##ID(const GemmParams<double>&, bool, bool, cudaStream_t);
RECTRI_DGEMM_TMA_CONFIGS(RECTRI_DECL)
#undef RECTRI_DECL

}  // namespace rectri_cu
