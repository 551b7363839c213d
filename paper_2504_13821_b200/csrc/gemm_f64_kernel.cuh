// gemm_f64_kernel.cuh -- fp64 GEMM update for the recursion on the sm_100a DMMA path.
//
// Replaces the reference's blocked CPU GEMM (src/gemm.cpp:17-216, microkernel
// src/gemm_kernels_avx2.cpp:13-67) for the off-diagonal updates
// B_dst += coeff * op(A_off) * B_src (Left) / B_src * op(A_off) (Right),
// recursion.cpp:134-143.  tcgen05 has no f64 kind, so the tensor path is
// mma.sync.m16n8k4.f64 -> 2x SASS DMMA.8x8x4 (36.9 TF/s measured peak on
// B200, profiles/r01_microbench_peaks.jsonl).
//
// Structure: CTA tile BM x BN x 16; a STAGES-deep cp.async (LDGSTS) ring in
// shared memory with an XOR swizzle that makes every fragment read
// conflict-free; warps own WM x WN sub-tiles and issue DMMA from register
// fragments that are double-buffered across the four k-steps of a tile; one
// __syncthreads per k-tile, placed before the last k-step so the next tile's
// first fragments load underneath the last MMAs; fused epilogue
// C = fma(alpha, acc, beta * C) (beta == 0 never reads C).
//
// Determinism: every configuration accumulates each element over k in the
// same order (16-wide k-tiles, four m16n8k4 steps each), so the result does
// not depend on the tile shape chosen for a given M, N.
#pragma once
#include "common.cuh"
#include "launch.h"

namespace rectri_cu {
namespace dgemm {


__device__ __forceinline__ void dmma1684(double (&c)[4], double a0, double a1, double b) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
      "{%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a0), "d"(a1), "d"(b));
}

// Per-thread loader of one operand tile.  Shared rows hold CPR chunks of
// VEC doubles; thread q copies the chunks q, q + NT, ... so its chunk column
// is fixed and its row advances by NT / CPR per iteration.
//   MC: outer-contiguous source, element (o, k) at X[o + k*ld]; rows = k.
//   KC: k-contiguous source, element (o, k) at X[k + o*ld]; rows = o.
// Out-of-range elements are zero-filled by the cp.async src-size operand.
// Shared layout of an outer-contiguous (MC) tile: rows = k of BO doubles.
//   MCMODE 0: 16-byte-chunk XOR swizzle, one warp copies one row.
//   MCMODE 1: no swizzle, rows padded by 4 doubles (fragment reads stay
//             conflict-free: double-bank = 4t + g), one warp copies one row.
//   MCMODE 2: XOR swizzle, one warp copies 4 rows x 128 bytes.
// k-contiguous (KC) tiles: rows = outer, kBK doubles, XOR swizzle.
template <int BO, int MCMODE>
struct McLayout {
  static constexpr int STRIDE = MCMODE == 1 ? BO + 4 : BO;
  __host__ __device__ static constexpr int elems(int rows) { return rows * STRIDE; }
  __device__ static int idx(int row, int col) {
    return MCMODE == 1 ? row * STRIDE + col : swz64(row, col, BO);
  }
};

template <int BO, int BK, int NT, int VEC, bool KC, int MCMODE>
struct TileLoader {
  static constexpr int kBK = BK;
  static constexpr int WIDTH = KC ? kBK : BO;  // logical row width (doubles)
  static constexpr int CPR = WIDTH / VEC;
  static constexpr int ROWS = KC ? BO : kBK;
  static constexpr int IT = CPR * ROWS / NT;
  static_assert(NT % CPR == 0 || (!KC && MCMODE == 2), "loader trip count");
  static_assert((CPR * ROWS) % NT == 0, "loader trip count");
  // MCMODE 2: a warp covers RPW rows x G chunks (G chunks = 128 bytes).
  static constexpr int G = 128 / (8 * VEC);
  static constexpr int RPW = 32 / G;

  const double* base;  // X at the tile's outer origin o0 (valid dummy source)
  const double* p0;    // this thread's first chunk for k-tile 0
  i64 ld, step;        // leading dimension; global stride between its chunks
  int row0, col;       // thread's first shared row, its chunk column (elements)
  int o_lim, k_lim;    // outer extent left from o0, and K
  int fix_bytes;       // KC: per-row (outer) validity; MC: bytes of its column

  // rows advanced per iteration
  static constexpr int ROW_STEP = (!KC && MCMODE == 2) ? RPW * (NT / 32) / (CPR / G) : NT / CPR;

  __device__ void init(const double* X, i64 ld_, i64 o0, i64 O, i64 K) {
    ld = ld_;
    if (!KC && MCMODE == 2) {
      const int q = threadIdx.x;  // chunk id -> (row, chunk) in RPW x G warp tiles
      const int lane = q & 31, w = q >> 5;
      const int tiles_per_row = CPR / G;
      const int tr = w / tiles_per_row, tc = w % tiles_per_row;
      row0 = RPW * tr + lane / G;
      col = (tc * G + lane % G) * VEC;
    } else {
      row0 = threadIdx.x / CPR;
      col = (threadIdx.x % CPR) * VEC;
    }
    o_lim = static_cast<int>(O - o0 < (1 << 30) ? O - o0 : (1 << 30));
    k_lim = static_cast<int>(K < (1 << 30) ? K : (1 << 30));
    base = KC ? X + o0 * ld : X + o0;
    // Both layouts: element (row, col) of the tile at base + row*ld + col
    // (KC: row = outer, col = k; MC: row = k, col = outer).
    p0 = base + static_cast<i64>(row0) * ld + col;
    step = static_cast<i64>(ROW_STEP) * ld;
    if (!KC) {
      const int rem = o_lim - col;
      fix_bytes = rem >= VEC ? VEC * 8 : (rem > 0 ? rem * 8 : 0);
    }
  }

  __device__ __forceinline__ void load(uint32_t stage, i64 kt) const {
    const int k0 = static_cast<int>(kt * kBK);
    const double* tb = p0 + (KC ? static_cast<i64>(k0) : static_cast<i64>(k0) * ld);
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      const int row = row0 + it * ROW_STEP;
      int bytes;
      if (KC) {
        const int rem = k_lim - (k0 + col);
        bytes = row < o_lim ? (rem >= VEC ? VEC * 8 : (rem > 0 ? rem * 8 : 0)) : 0;
      } else {
        bytes = (k0 + row < k_lim) ? fix_bytes : 0;
      }
      // Hoisted per-thread pointer: k*ld would otherwise be a 64-bit multiply
      // per chunk and k-tile on outer-contiguous tiles.
      const double* g = bytes ? tb + it * step : base;
      const int e = KC ? swz64(row, col, kBK) : McLayout<BO, MCMODE>::idx(row, col);
      const uint32_t dst = stage + 8u * static_cast<uint32_t>(e);
      if constexpr (VEC == 2)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(g), "r"(bytes));
      else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(g), "r"(bytes));
    }
  }
};

template <int BM, int BN, int BK, int WARPS_M, int WARPS_N, int STAGES, bool TA, bool TB, int VEC,
          int MCMODE>
__global__ void __launch_bounds__(WARPS_M * WARPS_N * 32, 1)
    dgemm_dmma_kernel(const GemmParams<double> p) {
  pdl_wait();  // PDL: no-op unless launched programmatically (launch_kernel)
  constexpr int kBK = BK;
  constexpr int NT = WARPS_M * WARPS_N * 32;
  constexpr int WM = BM / WARPS_M, WN = BN / WARPS_N;
  constexpr int TM = WM / 16, TN = WN / 8;
  constexpr int KK = kBK / 4;
  static_assert(WM % 16 == 0 && WN % 8 == 0, "warp tile");
  using LA = McLayout<BM, MCMODE>;
  using LB = McLayout<BN, MCMODE>;
  constexpr uint32_t A_STAGE = (TA ? BM * kBK : LA::elems(kBK)) * 8;
  constexpr uint32_t B_STAGE = (TB ? LB::elems(kBK) : BN * kBK) * 8;

  extern __shared__ __align__(128) double smem[];
  const uint32_t sA = smem_u32(smem);
  const uint32_t sB = sA + STAGES * A_STAGE;

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm0 = (warp % WARPS_M) * WM, wn0 = (warp / WARPS_M) * WN;
  // Grouped rasterization of a 1-D grid: consecutive CTAs walk kGroup
  // M-tiles down one N column, then the next column, so the CTAs resident at
  // any time share A row-panels and B column-panels in L2 (an M-fastest grid
  // re-streamed all of A from DRAM for every N column).
  constexpr int kGroup = 16;
  const int tiles_m = static_cast<int>(ceil_div(p.M, BM));
  const int tiles_n = static_cast<int>(ceil_div(p.N, BN));
  const int lin = static_cast<int>(blockIdx.x);
  const int per_group = kGroup * tiles_n;
  const int grp = lin / per_group, in_grp = lin - grp * per_group;
  const int gm0 = grp * kGroup;
  const int gsize = min(kGroup, tiles_m - gm0);
  const int tm = gm0 + in_grp % gsize, tn = in_grp / gsize;
  const i64 m0 = static_cast<i64>(tm) * BM;
  const i64 n0 = static_cast<i64>(tn) * BN;
  const i64 KT = ceil_div(p.K, kBK);

  // Warm L2 with this CTA's C tile (read by the epilogue) while the
  // mainloop runs: one prefetch per 128-byte line of each column.
  if (p.beta != 0.0) {
    constexpr int LINES = BM * 8 / 128;  // lines per column
    for (int q = threadIdx.x; q < BN * LINES; q += NT) {
      const i64 n = n0 + q / LINES, m = m0 + (q % LINES) * 16;
      if (n < p.N && m < p.M)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(p.C + m + n * p.ldc));
    }
  }

  TileLoader<BM, BK, NT, VEC, TA, MCMODE> la;
  TileLoader<BN, BK, NT, VEC, !TB, MCMODE> lb;
  la.init(p.A, p.lda, m0, p.M, p.K);
  lb.init(p.B, p.ldb, n0, p.N, p.K);

  // Per-thread fragment offsets (bytes, within a stage) for k-step 0; later
  // k-steps add a constant (the swizzle depends on row & 3 only, and k-steps
  // move the k index by 4 rows in k-major layouts).
  uint32_t a_off[TM][2], b_off[TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int m = wm0 + 16 * i + 8 * h + g;
      a_off[i][h] = 8u * static_cast<uint32_t>(TA ? swz64(m, t, kBK) : LA::idx(t, m));
    }
#pragma unroll
  for (int j = 0; j < TN; ++j) {
    const int n = wn0 + 8 * j + g;
    b_off[j] = 8u * static_cast<uint32_t>(TB ? LB::idx(t, n) : swz64(n, t, kBK));
  }
  // k-major layouts: a k-step moves 4 rows and keeps (row & 3), hence the
  // swizzle; k-contiguous layouts recompute the swizzled column.
  auto a_addr = [&](uint32_t stage, int i, int h, int kk) -> uint32_t {
    if constexpr (!TA) return stage + a_off[i][h] + static_cast<uint32_t>(kk * 4 * LA::STRIDE * 8);
    const int m = wm0 + 16 * i + 8 * h + g;
    return stage + 8u * static_cast<uint32_t>(swz64(m, kk * 4 + t, kBK));
  };
  auto b_addr = [&](uint32_t stage, int j, int kk) -> uint32_t {
    if constexpr (TB) return stage + b_off[j] + static_cast<uint32_t>(kk * 4 * LB::STRIDE * 8);
    const int n = wn0 + 8 * j + g;
    return stage + 8u * static_cast<uint32_t>(swz64(n, kk * 4 + t, kBK));
  };

  double af[2][TM][2], bf[2][TN];
  auto load_frags = [&](int buf, int stage, int kk) {
    const uint32_t as = sA + stage * A_STAGE, bs = sB + stage * B_STAGE;
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int h = 0; h < 2; ++h)
        asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(af[buf][i][h]) : "r"(a_addr(as, i, h, kk)));
#pragma unroll
    for (int j = 0; j < TN; ++j)
      asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(bf[buf][j]) : "r"(b_addr(bs, j, kk)));
  };

  double acc[TM][TN][4];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[i][j][e] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < KT) {
      la.load(sA + s * A_STAGE, s);
      lb.load(sB + s * B_STAGE, s);
    }
    cp_async_commit();
  }
  cp_async_wait<STAGES - 2>();
  __syncthreads();
  load_frags(0, 0, 0);

  for (i64 kt = 0; kt < KT; ++kt) {
    {  // refill the stage of tile kt-1 (fully consumed before the last barrier)
      const i64 nk = kt + STAGES - 1;
      if (nk < KT) {
        const int ws = static_cast<int>(nk % STAGES);
        la.load(sA + ws * A_STAGE, nk);
        lb.load(sB + ws * B_STAGE, nk);
      }
      cp_async_commit();
    }
    const int rs = static_cast<int>(kt % STAGES);
#pragma unroll
    for (int kk = 0; kk < KK; ++kk) {
      const int cb = kk & 1, nb = cb ^ 1;
      if (kk < KK - 1) {
        load_frags(nb, rs, kk + 1);
      } else {
        cp_async_wait<STAGES - 2>();  // tile kt+1 has landed (this thread's part)
        __syncthreads();              // ... and everyone's; stage rs-1 is free
        if (kt + 1 < KT) load_frags(nb, static_cast<int>((kt + 1) % STAGES), 0);
      }
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) dmma1684(acc[i][j], af[cb][i][0], af[cb][i][1], bf[cb][j]);
    }
  }
  cp_async_wait<0>();

  // Epilogue, per row tile: every C read issued before the first write.
  const bool beta_zero = p.beta == 0.0;
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    double cold[2][TN][2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const i64 m = m0 + wm0 + 16 * i + 8 * h + g;
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        const i64 n = n0 + wn0 + 8 * j + 2 * t;
#pragma unroll
        for (int e = 0; e < 2; ++e)
          cold[h][j][e] = (!beta_zero && m < p.M && n + e < p.N) ? p.C[m + (n + e) * p.ldc] : 0.0;
      }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const i64 m = m0 + wm0 + 16 * i + 8 * h + g;
      if (m >= p.M) continue;
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        const i64 n = n0 + wn0 + 8 * j + 2 * t;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          if (n + e < p.N) {
            const double v = acc[i][j][2 * h + e];
            p.C[m + (n + e) * p.ldc] = beta_zero ? p.alpha * v : fma(p.alpha, v, p.beta * cold[h][j][e]);
          }
        }
      }
    }
  }
}

// Host launcher of one configuration (all four transpose forms, both copy
// widths); instantiated in gemm_f64_cfg*.cu.
template <int BM, int BN, int BK, int WARPS_M, int WARPS_N, int STAGES, int MCMODE = 0>
struct Config {
  template <bool TA, bool TB, int VEC>
  static void launch(const GemmParams<double>& p, cudaStream_t s) {
    auto kern = dgemm_dmma_kernel<BM, BN, BK, WARPS_M, WARPS_N, STAGES, TA, TB, VEC, MCMODE>;
    constexpr int pad = MCMODE == 1 ? 4 : 0;
    constexpr int smem = STAGES * (BM + BN + 2 * pad) * BK * static_cast<int>(sizeof(double));
    set_smem(kern, smem);
    const unsigned grid = static_cast<unsigned>(ceil_div(p.M, BM) * ceil_div(p.N, BN));
    launch_kernel(kern, grid, WARPS_M * WARPS_N * 32, smem, s, p);
    ++launch_counter();
  }
  static void run(const GemmParams<double>& p, bool ta, bool tb, bool vec2, cudaStream_t s) {
#define RECTRI_T(TA_, TB_)                                  \
  if (ta == TA_ && tb == TB_) {                             \
    if (vec2) launch<TA_, TB_, 2>(p, s);                    \
    else launch<TA_, TB_, 1>(p, s);                         \
    return;                                                 \
  }
    RECTRI_T(false, false)
    RECTRI_T(true, false)
    RECTRI_T(false, true)
    RECTRI_T(true, true)
#undef RECTRI_T
  }
};

}  // namespace dgemm

// Entry points of the instantiated configurations (gemm_f64_cfg*.cu).
using DgemmRun = void (*)(const GemmParams<double>&, bool, bool, bool, cudaStream_t);
#define RECTRI_DGEMM_CONFIGS(X) \
  X(0, 64, 64, 16, 2, 2, 4)     \
  X(1, 64, 64, 16, 4, 2, 4)
#define RECTRI_DECL(ID, BM, BN, BK, WM, WN, ST) \
  void dgemm_cfg##ID(const GemmParams<double>&, bool, bool, bool, cudaStream_t);
RECTRI_DGEMM_CONFIGS(RECTRI_DECL)
#undef RECTRI_DECL

}  // namespace rectri_cu
