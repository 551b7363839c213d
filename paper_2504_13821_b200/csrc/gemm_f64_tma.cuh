// gemm_f64_tma.cuh -- fp64 DMMA GEMM update fed by TMA + mbarrier pipelines.
//
// Same contract and the same per-element arithmetic as gemm_f64_kernel.cuh
// (the cp.async kernel, kept for operands TMA cannot describe): it replaces
// the reference's blocked CPU GEMM (src/gemm.cpp:155-216) for the
// recursion's off-diagonal updates (recursion.cpp:134-143).
//
// Data movement: one elected thread (a dedicated producer warp, or lane 0 of
// warp 0) issues cp.async.bulk.tensor (TMA) copies of each 16-deep k-tile of
// op(A) and op(B) into a STAGES-deep shared ring; TMA zero-fills every
// out-of-range element (exact 0, never a multiply-by-mask).  Each stage has a
// `full` mbarrier (armed with the byte count, completed by the TMA) and an
// `empty` mbarrier (one arrival per consumer warp once its last fragment read
// of the stage is done).  No __syncthreads in the mainloop, no per-thread
// address arithmetic for global loads.
//
// Shared layouts (8-byte elements) -- both conflict-free for the way the
// LSU splits a warp's request (128-bit loads: four phases of 8 consecutive
// lanes; 64-bit loads: two half-warps):
//   outer-contiguous operand (A NoTrans / B Trans): 2D box {BO + 4, 16}, so
//     a k-row is BO + 4 doubles long (the 4 extra outer elements are loaded
//     and never used; this is the padding TMA cannot otherwise express).
//     Each thread reads two adjacent outer indices with one ld.shared.v2.f64;
//     a phase (2 outer pairs x 4 k-rows) then covers 8 distinct 16-byte bank
//     groups because consecutive k-rows are shifted by 32 bytes.
//   k-contiguous operand (A Trans / B NoTrans): 2D box {16, BO} with the
//     128-byte TMA swizzle, element (o, k) at o*16 + 2*((k/2) ^ (o%8)) + k%2.
//     Fragment row g of an 8-row group is stored at outer index
//     perm(g) = 2*(g%4) + g/4, so a half-warp (g = 0..3 or 4..7) meets four
//     distinct (o%8)/2 values and its 16 loads land in 8 distinct chunks.
//
// Permutations (free: they only relabel which output row/column an mma
// lane-slot holds, never the k order): outer-contiguous A: mma row r of
// 16-row tile i is m = 16i + 2(r%8) + r/8; k-contiguous A: m = 16i +
// 8(r/8) + perm(r%8); outer-contiguous B: the 8-column mma tiles 2q, 2q+1
// interleave, column c of tile j is n = 16q + 2c + (j%2); k-contiguous B:
// n = 8j + perm(c).
//
// Determinism: each output element is accumulated over k in 16-wide k-tiles
// of four m16n8k4 steps from a zero accumulator, then C = fma(alpha, acc,
// beta*C) -- exactly the cp.async kernel's sequence, so the two kernels (and
// every tile shape) produce identical bits.
#pragma once
#include <cuda.h>

#include "common.cuh"
#include "launch.h"

namespace rectri_cu {
namespace dgemm_tma {

constexpr int kBK = 16;

__device__ __forceinline__ void dmma1684(double (&c)[4], double a0, double a1, double b) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
      "{%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a0), "d"(a1), "d"(b));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                            uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];\n" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void lds64(double& x, uint32_t a) {
  asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(x) : "r"(a));
}
__device__ __forceinline__ void lds128(double& x, double& y, uint32_t a) {
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(x), "=d"(y) : "r"(a));
}

// STAGES-deep ring; CONSUMER warps WARPS_M x WARPS_N each own WM x WN;
// PRODUCER: a dedicated 32-thread producer warp (else lane 0 of warp 0).
// MC_A: A tile outer(m)-contiguous (op(A) = A); MC_B: B tile outer(n)-contiguous
// (op(B) = B^T).
// One BM x BN output tile at (m0, n0) (the body of every TMA DGEMM kernel).
// CK: the ring checker's instantiation (RECTRI_CU_RING_CHECK): every fragment
// a consumer warp reads from a stage is compared, bit for bit, with its
// element of op(A) / op(B) in global memory (zero outside the matrix, as TMA
// fills it); a refill overtaking a stage's readers shows up as a mismatch.
template <int BM, int BN, int WARPS_M, int WARPS_N, int STAGES, bool PRODUCER, bool MC_A, bool MC_B, bool CK = false>
__device__ __forceinline__ void dgemm_tma_tile(const CUtensorMap* mapA_, const CUtensorMap* mapB_,
                                               const GemmParams<double>& p, const int m0, const int n0,
                                               unsigned char* smem_raw) {
  const CUtensorMap& mapA = *mapA_;
  const CUtensorMap& mapB = *mapB_;
  constexpr int NCW = WARPS_M * WARPS_N;  // consumer warps
  constexpr int WM = BM / WARPS_M, WN = BN / WARPS_N;
  constexpr int TM = WM / 16, TN = WN / 8;
  static_assert(WM % 16 == 0 && WN % 16 == 0, "warp tile");
  constexpr int PAD = 4;  // extra outer elements per k-row of an outer-contiguous tile
  constexpr int A_PITCH = MC_A ? BM + PAD : BM, B_PITCH = MC_B ? BN + PAD : BN;
  constexpr uint32_t A_BYTES = A_PITCH * kBK * 8, B_BYTES = B_PITCH * kBK * 8;
  // 1024-byte aligned tiles (128-byte swizzle atoms)
  constexpr uint32_t A_SLOT = (A_BYTES + 1023u) & ~1023u, B_SLOT = (B_BYTES + 1023u) & ~1023u;
  constexpr uint32_t STAGE_BYTES = A_SLOT + B_SLOT;

  // 1024-byte alignment for the 128-byte swizzle atoms.
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t sbase = (raw + 1023u) & ~1023u;
  const uint32_t bars = sbase + STAGES * STAGE_BYTES;  // full[s] at +8s, empty[s] at +8(STAGES+s)
  auto full_bar = [&](int s) { return bars + 8u * s; };
  auto empty_bar = [&](int s) { return bars + 8u * (STAGES + s); };
  auto stage_a = [&](int s) { return sbase + s * STAGE_BYTES; };
  auto stage_b = [&](int s) { return sbase + s * STAGE_BYTES + A_SLOT; };

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

  const int KT = static_cast<int>(ceil_div(p.K, kBK));

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(empty_bar(s), NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  }
  __syncthreads();

  auto issue = [&](int kf) {  // one elected thread: fill stage kf % STAGES with k-tile kf
    const int s = kf % STAGES;
    mbar_expect_tx(full_bar(s), A_BYTES + B_BYTES);
    // outer-contiguous: dims {O, K}, coords {o0, k0}; k-contiguous: {K, O}, {k0, o0}
    if (MC_A) tma_load_2d(stage_a(s), &mapA, m0, kf * kBK, full_bar(s));
    else tma_load_2d(stage_a(s), &mapA, kf * kBK, m0, full_bar(s));
    if (MC_B) tma_load_2d(stage_b(s), &mapB, n0, kf * kBK, full_bar(s));
    else tma_load_2d(stage_b(s), &mapB, kf * kBK, n0, full_bar(s));
  };

  if (PRODUCER && warp == NCW) {
    if (lane == 0) {
      for (int kf = 0; kf < KT; ++kf) {
        if (kf >= STAGES) mbar_wait(empty_bar(kf % STAGES), ((kf / STAGES) + 1) & 1);
        issue(kf);
      }
    }
    return;
  }
  constexpr int kAhead = PRODUCER ? 0 : STAGES - 1;  // inline producer keeps STAGES-1 tiles in flight
  if (!PRODUCER && threadIdx.x == 0) {
    for (int kf = 0; kf < kAhead && kf < KT; ++kf) issue(kf);
  }

  // Consumers.
  const int g = lane >> 2, t = lane & 3;
  const int wm0 = (warp % WARPS_M) * WM, wn0 = (warp / WARPS_M) * WN;
  // Byte offsets within a stage's A / B tile for k-step 0 (k-steps add a
  // constant for outer-contiguous tiles; k-contiguous tiles use xo[kk]).
  // k-contiguous swizzled element (o, k): o*128 + (((k>>1) ^ (o&7)) << 4) + (k&1)*8,
  // with o&7 == perm(g) for every fragment row/column this thread reads.
  const int pg = ((g & 3) << 1) | (g >> 2);
  uint32_t xo[4];
#pragma unroll
  for (int kk = 0; kk < 4; ++kk)
    xo[kk] = static_cast<uint32_t>(((((4 * kk + t) >> 1) ^ pg) << 4) + (t & 1) * 8);
  const uint32_t a_mc = static_cast<uint32_t>((t * A_PITCH + wm0 + 2 * g) * 8);
  const uint32_t a_kc = static_cast<uint32_t>((wm0 + pg) * 128);
  const uint32_t b_mc = static_cast<uint32_t>((t * B_PITCH + wn0 + 2 * g) * 8);
  const uint32_t b_kc = static_cast<uint32_t>((wn0 + pg) * 128);

  double af[2][TM][2], bf[2][TN];
  auto load_frags = [&](int buf, int s, int kk, int ktile) {
    const int sr = CK && p.ring_plant ? (s + 1) % STAGES : s;  // planted: the wrong stage
    const uint32_t as = stage_a(sr), bs = stage_b(sr);
#pragma unroll
    for (int i = 0; i < TM; ++i) {
      if (MC_A) {
        lds128(af[buf][i][0], af[buf][i][1], as + a_mc + (kk * 4 * A_PITCH + 16 * i) * 8);
      } else {
        lds64(af[buf][i][0], as + a_kc + xo[kk] + (16 * i) * 128);
        lds64(af[buf][i][1], as + a_kc + xo[kk] + (16 * i + 8) * 128);
      }
    }
    if (MC_B) {
#pragma unroll
      for (int q = 0; q < TN / 2; ++q)
        lds128(bf[buf][2 * q], bf[buf][2 * q + 1], bs + b_mc + (kk * 4 * B_PITCH + 16 * q) * 8);
    } else {
#pragma unroll
      for (int j = 0; j < TN; ++j) lds64(bf[buf][j], bs + b_kc + xo[kk] + (8 * j) * 128);
    }
    if constexpr (CK) {
      const i64 kg = static_cast<i64>(ktile) * kBK + 4 * kk + t;
      auto opa = [&](i64 m) {
        if (m >= p.M || kg >= p.K) return 0.0;
        return MC_A ? p.A[m + kg * p.lda] : p.A[kg + m * p.lda];
      };
      auto opb = [&](i64 n) {
        if (n >= p.N || kg >= p.K) return 0.0;
        return MC_B ? p.B[n + kg * p.ldb] : p.B[kg + n * p.ldb];
      };
      auto ne = [](double x, double y) { return __double_as_longlong(x) != __double_as_longlong(y) ? 1u : 0u; };
      unsigned bad = 0;
#pragma unroll
      for (int i = 0; i < TM; ++i) {
        const i64 m = m0 + wm0 + (MC_A ? 2 * g : pg) + 16 * i;
        bad += ne(af[buf][i][0], opa(m)) + ne(af[buf][i][1], opa(MC_A ? m + 1 : m + 8));
      }
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        const i64 n = MC_B ? n0 + wn0 + 2 * g + 16 * (j / 2) + (j & 1) : n0 + wn0 + pg + 8 * j;
        bad += ne(bf[buf][j], opb(n));
      }
      if (bad) atomicAdd(p.ring_check, static_cast<unsigned long long>(bad));
    }
  };

  const uint32_t zero = static_cast<uint32_t>(p.K >> 40);  // 0 at run time, unknown to ptxas
  double acc[TM][TN][4];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[i][j][e] = 0.0;

  if (KT > 0) {
    mbar_wait(full_bar(0), 0);
    load_frags(0, 0, 0, 0);
  }
  for (int kt = 0; kt < KT; ++kt) {
    if (!PRODUCER && threadIdx.x == 0) {
      const int kf = kt + kAhead;
      if (kf < KT) {
        if (kf >= STAGES) mbar_wait(empty_bar(kf % STAGES), ((kf / STAGES) + 1) & 1);
        issue(kf);
      }
    }
    const int s = kt % STAGES;
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      const int cb = kk & 1, nb = cb ^ 1;
      if (kk < 3) {
        load_frags(nb, s, kk + 1, kt);
      } else if (kt + 1 < KT) {
        const int s1 = (kt + 1) % STAGES;
        mbar_wait(full_bar(s1), ((kt + 1) / STAGES) & 1);
        load_frags(nb, s1, 0, kt + 1);
      }
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) dmma1684(acc[i][j], af[cb][i][0], af[cb][i][1], bf[cb][j]);
      if (kk == 3) {
        // Release stage s once its last fragment loads (this k-step's) have
        // landed: the arrive's address depends on them (slot_dep, common.cuh).
        uint32_t dep = 0;
#pragma unroll
        for (int i = 0; i < TM; ++i) dep |= slot_dep(zero, af[cb][i][0], af[cb][i][1]);
#pragma unroll
        for (int j = 0; j < TN; ++j) dep |= slot_dep(zero, bf[cb][j]);
        __syncwarp();
        if (lane == 0) mbar_arrive(empty_bar(s) + dep);
      }
    }
  }

  // Epilogue: C = fma(alpha, acc, beta*C) (beta == 0 never reads C).  Per
  // output row, every C read is issued before the first write, so the reads'
  // latency is paid once per row instead of once per element.
  const bool beta_zero = p.beta == 0.0;
  auto col_of = [&](int j, int e) -> i64 {
    const int c = 2 * t + e;
    return n0 + wn0 + (MC_B ? 16 * (j >> 1) + 2 * c + (j & 1) : 8 * j + (((c & 3) << 1) | (c >> 2)));
  };
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const i64 m = m0 + wm0 + 16 * i + (MC_A ? 2 * g + h : 8 * h + pg);
      if (m >= p.M) continue;
      double cold[TN][2];
#pragma unroll
      for (int j = 0; j < TN; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const i64 n = col_of(j, e);
          cold[j][e] = (!beta_zero && n < p.N) ? p.C[m + n * p.ldc] : 0.0;
        }
#pragma unroll
      for (int j = 0; j < TN; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const i64 n = col_of(j, e);
          if (n < p.N) {
            const double v = acc[i][j][2 * h + e];
            p.C[m + n * p.ldc] = beta_zero ? p.alpha * v : fma(p.alpha, v, p.beta * cold[j][e]);
          }
        }
    }
}

// Grouped rasterization (as the cp.async kernel): consecutive CTAs walk 16
// M-tiles down one N column so resident CTAs share panels in L2.
__device__ __forceinline__ void grouped_tile(int lin, int tiles_m, int tiles_n, int& tm, int& tn) {
  constexpr int kGroup = 16;
  const int per_group = kGroup * tiles_n;
  const int grp = lin / per_group, in_grp = lin - grp * per_group;
  const int gm0 = grp * kGroup;
  const int gsize = min(kGroup, tiles_m - gm0);
  tm = gm0 + in_grp % gsize;
  tn = in_grp / gsize;
}

template <int BM, int BN, int WARPS_M, int WARPS_N, int STAGES, bool PRODUCER, bool MC_A, bool MC_B, bool CK = false>
__global__ void __launch_bounds__((WARPS_M * WARPS_N + (PRODUCER ? 1 : 0)) * 32, 1)
    dgemm_tma_kernel(const __grid_constant__ CUtensorMap mapA,
                     const __grid_constant__ CUtensorMap mapB, const GemmParams<double> p) {
  pdl_wait();  // PDL: no-op unless launched programmatically (launch_kernel)
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  int tm, tn;
  grouped_tile(static_cast<int>(blockIdx.x), static_cast<int>(ceil_div(p.M, BM)), static_cast<int>(ceil_div(p.N, BN)),
               tm, tn);
  dgemm_tma_tile<BM, BN, WARPS_M, WARPS_N, STAGES, PRODUCER, MC_A, MC_B, CK>(&mapA, &mapB, p, tm * BM, tn * BN,
                                                                             smem_raw);
}

// Wave-tail split: the columns [0, n_main) in 64x64 tiles -- a whole number
// of waves of resident CTAs -- and the remaining columns in 32x32 tiles, four
// CTAs per 64x64 tile, so the last wave is not a few long CTAs on a mostly
// idle GPU.  Every element keeps the same k-tile order, so the result is bit
// for bit that of the uniform kernels.
template <bool MC_A, bool MC_B, bool CK = false>
__global__ void __launch_bounds__(5 * 32, 1)
    dgemm_tma_split_kernel(const __grid_constant__ CUtensorMap a64, const __grid_constant__ CUtensorMap b64,
                           const __grid_constant__ CUtensorMap a32, const __grid_constant__ CUtensorMap b32,
                           const GemmParams<double> p, const int n_main) {
  pdl_wait();  // PDL: no-op unless launched programmatically (launch_kernel)
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const int tiles_m64 = static_cast<int>(ceil_div(p.M, 64));
  const int main_tiles = tiles_m64 * (n_main / 64);
  const int b = static_cast<int>(blockIdx.x);
  if (b < main_tiles) {
    int tm, tn;
    grouped_tile(b, tiles_m64, n_main / 64, tm, tn);
    dgemm_tma_tile<64, 64, 2, 2, 4, true, MC_A, MC_B, CK>(&a64, &b64, p, tm * 64, tn * 64, smem_raw);
  } else {
    const int tiles_m32 = static_cast<int>(ceil_div(p.M, 32));
    const int r = b - main_tiles;
    dgemm_tma_tile<32, 32, 2, 2, 4, true, MC_A, MC_B, CK>(&a32, &b32, p, (r % tiles_m32) * 32,
                                                         n_main + (r / tiles_m32) * 32, smem_raw);
  }
}

}  // namespace dgemm_tma

// Returns false (nothing launched) when TMA cannot describe the operands
// (unaligned base / odd leading dimension / index range beyond int32).
bool launch_gemm_f64_tma(const GemmParams<double>& p, bool ta, bool tb, cudaStream_t s, int cfg);

}  // namespace rectri_cu
