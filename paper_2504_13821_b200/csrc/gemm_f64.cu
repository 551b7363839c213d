// gemm_f64.cu -- fp64 GEMM update for the recursion on the sm_100a DMMA path.
//
// Replaces the reference's blocked CPU GEMM (src/gemm.cpp:17-216, microkernel
// src/gemm_kernels_avx2.cpp:13-67) for the off-diagonal updates
// B_dst += coeff * op(A_off) * B_src (Left) / B_src * op(A_off) (Right),
// recursion.cpp:134-143.  tcgen05 has no f64 kind, so the tensor path is
// mma.sync.m8n8k4.f64 -> SASS DMMA.8x8x4 (measured 36.9 TF/s peak on B200,
// profiles/r01_microbench_peaks.jsonl).
//
// Structure: CTA tile BM x BN x 16, STAGES-deep cp.async (LDGSTS) ring in
// shared memory (swizzled, conflict-free fragment reads), warps of WM x WN
// sub-tiles issuing DMMA from register fragments, fused epilogue
// C = fma(alpha, acc, beta * C).
#include "common.cuh"
#include "launch.h"

namespace rectri_cu {
namespace {

constexpr int kBK = 16;

// Outer-contiguous operand tile ("MC"): element (o, k) at X[o + k * ld];
// shared rows are k (kBK rows of BO doubles).
template <int BO, int NT, int VEC>
__device__ __forceinline__ void load_tile_mc(double* s, const double* X, i64 ld, i64 o0, i64 O,
                                             i64 k0, i64 K) {
  if constexpr (VEC == 2) {
    constexpr int CPR = BO / 2;
    constexpr int TOTAL = kBK * CPR;
#pragma unroll
    for (int q = threadIdx.x; q < TOTAL; q += NT) {
      const int k = q / CPR, oc = q % CPR;
      const i64 go = o0 + 2 * oc, gk = k0 + k;
      int bytes = 0;
      const double* src = X;
      if (gk < K && go < O) {
        bytes = (O - go) >= 2 ? 16 : 8;
        src = X + go + gk * ld;
      }
      cp_async16(s + k * BO + ((oc ^ ((k & 3) << 1)) << 1), src, bytes);
    }
  } else {
    constexpr int TOTAL = kBK * BO;
#pragma unroll 4
    for (int q = threadIdx.x; q < TOTAL; q += NT) {
      const int k = q / BO, o = q % BO;
      const i64 go = o0 + o, gk = k0 + k;
      const bool ok = gk < K && go < O;
      cp_async8(s + swz64(k, o, BO), ok ? X + go + gk * ld : X, ok ? 8 : 0);
    }
  }
}

// k-contiguous operand tile ("KC"): element (o, k) at X[k + o * ld]; shared
// rows are o (BO rows of kBK doubles).
template <int BO, int NT, int VEC>
__device__ __forceinline__ void load_tile_kc(double* s, const double* X, i64 ld, i64 o0, i64 O,
                                             i64 k0, i64 K) {
  if constexpr (VEC == 2) {
    constexpr int TOTAL = BO * (kBK / 2);
#pragma unroll
    for (int q = threadIdx.x; q < TOTAL; q += NT) {
      const int o = q >> 3, kc = q & 7;
      const i64 go = o0 + o, gk = k0 + 2 * kc;
      int bytes = 0;
      const double* src = X;
      if (go < O && gk < K) {
        bytes = (K - gk) >= 2 ? 16 : 8;
        src = X + gk + go * ld;
      }
      cp_async16(s + o * kBK + ((kc ^ ((o & 3) << 1)) << 1), src, bytes);
    }
  } else {
    constexpr int TOTAL = BO * kBK;
#pragma unroll 4
    for (int q = threadIdx.x; q < TOTAL; q += NT) {
      const int o = q >> 4, k = q & 15;
      const i64 go = o0 + o, gk = k0 + k;
      const bool ok = go < O && gk < K;
      cp_async8(s + swz64(o, k, kBK), ok ? X + gk + go * ld : X, ok ? 8 : 0);
    }
  }
}

template <int BM, int BN, int WARPS_M, int WARPS_N, int STAGES, bool TA, bool TB, int VEC>
__global__ void __launch_bounds__(WARPS_M * WARPS_N * 32, 1)
    dgemm_dmma_kernel(const GemmParams<double> p) {
  constexpr int NT = WARPS_M * WARPS_N * 32;
  constexpr int WM = BM / WARPS_M, WN = BN / WARPS_N;
  constexpr int TM = WM / 8, TN = WN / 8;
  static_assert(WM % 8 == 0 && WN % 8 == 0, "warp tile");

  extern __shared__ __align__(128) double smem[];
  double* sA = smem;
  double* sB = smem + STAGES * BM * kBK;

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm0 = (warp % WARPS_M) * WM, wn0 = (warp / WARPS_M) * WN;
  const i64 m0 = static_cast<i64>(blockIdx.x) * BM;
  const i64 n0 = static_cast<i64>(blockIdx.y) * BN;
  const i64 KT = ceil_div(p.K, kBK);

  auto load_stage = [&](int stage, i64 kt) {
    const i64 k0 = kt * kBK;
    double* a = sA + stage * BM * kBK;
    double* b = sB + stage * BN * kBK;
    if constexpr (TA) load_tile_kc<BM, NT, VEC>(a, p.A, p.lda, m0, p.M, k0, p.K);
    else load_tile_mc<BM, NT, VEC>(a, p.A, p.lda, m0, p.M, k0, p.K);
    if constexpr (TB) load_tile_mc<BN, NT, VEC>(b, p.B, p.ldb, n0, p.N, k0, p.K);
    else load_tile_kc<BN, NT, VEC>(b, p.B, p.ldb, n0, p.N, k0, p.K);
  };

  double acc[TM][TN][2];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < KT) load_stage(s, s);
    cp_async_commit();
  }

  for (i64 kt = 0; kt < KT; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const i64 nk = kt + STAGES - 1;
      if (nk < KT) load_stage(static_cast<int>(nk % STAGES), nk);
      cp_async_commit();
    }
    const int st = static_cast<int>(kt % STAGES);
    const double* a_s = sA + st * BM * kBK;
    const double* b_s = sB + st * BN * kBK;
#pragma unroll
    for (int kk = 0; kk < kBK / 4; ++kk) {
      const int k = kk * 4 + t;
      double af[TM], bf[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) {
        const int m = wm0 + 8 * i + g;
        af[i] = TA ? a_s[swz64(m, k, kBK)] : a_s[swz64(k, m, BM)];
      }
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        const int n = wn0 + 8 * j + g;
        bf[j] = TB ? b_s[swz64(k, n, BN)] : b_s[swz64(n, k, kBK)];
      }
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();

  const bool beta_zero = p.beta == 0.0;
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const i64 m = m0 + wm0 + 8 * i + g;
    if (m >= p.M) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const i64 n = n0 + wn0 + 8 * j + 2 * t;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        if (n + e < p.N) {
          double* c = p.C + m + (n + e) * p.ldc;
          *c = beta_zero ? p.alpha * acc[i][j][e] : fma(p.alpha, acc[i][j][e], p.beta * *c);
        }
      }
    }
  }
}

template <int BM, int BN, int WARPS_M, int WARPS_N, int STAGES, bool TA, bool TB, int VEC>
void launch_cfg(const GemmParams<double>& p, cudaStream_t s) {
  auto kern = dgemm_dmma_kernel<BM, BN, WARPS_M, WARPS_N, STAGES, TA, TB, VEC>;
  constexpr int smem = STAGES * (BM + BN) * kBK * static_cast<int>(sizeof(double));
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  dim3 grid(static_cast<unsigned>(ceil_div(p.M, BM)), static_cast<unsigned>(ceil_div(p.N, BN)));
  kern<<<grid, WARPS_M * WARPS_N * 32, smem, s>>>(p);
  ++launch_counter();
}

template <int BM, int BN, int WARPS_M, int WARPS_N, int STAGES>
void dispatch_trans(const GemmParams<double>& p, bool ta, bool tb, bool vec2, cudaStream_t s) {
#define RECTRI_CFG(TA_, TB_)                                                            \
  if (ta == TA_ && tb == TB_) {                                                         \
    if (vec2) launch_cfg<BM, BN, WARPS_M, WARPS_N, STAGES, TA_, TB_, 2>(p, s);          \
    else launch_cfg<BM, BN, WARPS_M, WARPS_N, STAGES, TA_, TB_, 1>(p, s);               \
    return;                                                                             \
  }
  RECTRI_CFG(false, false)
  RECTRI_CFG(true, false)
  RECTRI_CFG(false, true)
  RECTRI_CFG(true, true)
#undef RECTRI_CFG
}

bool aligned16(const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15u) == 0; }

}  // namespace

void launch_gemm_f64(const GemmParams<double>& p, bool ta, bool tb, cudaStream_t s) {
  if (p.M <= 0 || p.N <= 0 || p.K <= 0) return;
  const bool vec2 = aligned16(p.A) && aligned16(p.B) && (p.lda % 2 == 0) && (p.ldb % 2 == 0);
  // Tile choice only changes which CTA owns an element, never its k order.
  if (p.M >= 128 && p.N >= 128) {
    dispatch_trans<128, 128, 2, 4, 4>(p, ta, tb, vec2, s);
  } else if (p.N >= 128) {
    dispatch_trans<64, 128, 2, 4, 4>(p, ta, tb, vec2, s);
  } else if (p.M >= 128) {
    dispatch_trans<128, 64, 4, 2, 4>(p, ta, tb, vec2, s);
  } else {
    dispatch_trans<64, 64, 2, 2, 4>(p, ta, tb, vec2, s);
  }
}

}  // namespace rectri_cu
