// gemm_f64_sk.cuh -- deterministic stream-K schedule of the TMA-fed fp64
// DMMA GEMM (gemm_f64_tma.cuh).
//
// The recursion's off-diagonal updates at mid sizes launch a few hundred to a
// few thousand 64x64 tiles, i.e. 1.1-4.6 "waves" of the 3 x 148 resident
// CTAs, and the last, partial wave idles most of the GPU (n = 4096 TRMM:
// K = 1024 level 27.7 TF/s, K = 2048 33.0; profiles/r02_*).  Here a
// persistent grid of G CTAs (the resident slots) takes equal shares of the
// T x KT (tile, k-tile) iteration space, so every CTA does the same work.
// Since T > G, a share spans at least one whole tile: it is [tail of tile a]
// [whole tiles] [head of tile b], and each split tile is shared by exactly two
// neighbouring CTAs.
//
// Determinism (the basis of every bitwise property of the library): a split
// tile's accumulator is handed from the head CTA to the tail CTA in global
// memory -- exact fp64 values -- and the tail CTA CONTINUES the same chain
// from it.  So every element is still accumulated over k in 16-wide k-tiles
// of four m16n8k4 steps from a zero accumulator, in k order, then C =
// fma(alpha, acc, beta*C): bit for bit the data-parallel kernel, for any G,
// T or split point (tests/test_gpu_gemm.py).
//
// Order inside a CTA: whole tiles, then the head piece (publish the partial:
// coalesced [element][thread] stores, a named barrier among the consumer
// warps, a fence, then the flag with release semantics), then the tail piece
// (acquire-spin on the neighbour's flag, load the partial, reset the flag
// for the next launch on this stream).  Every CTA publishes before it waits,
// and CTA c only waits on CTA c - 1, so the chain cannot deadlock.
#pragma once
#include "gemm_f64_tma.cuh"

namespace rectri_cu {
namespace dgemm_tma {

struct SkPlan {
  int tiles_m, tiles_n, KT;
  long long W;  // T * KT iterations
  int G;        // CTAs
};

__device__ __forceinline__ long long sk_begin(const SkPlan& q, int c) { return q.W * c / q.G; }

template <int BM, int BN, int WARPS_M, int WARPS_N, int STAGES, bool MC_A, bool MC_B>
__global__ void __launch_bounds__((WARPS_M * WARPS_N + 1) * 32, 1)
    dgemm_sk_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                    const GemmParams<double> p, const SkPlan q, double* __restrict__ ws, int* __restrict__ flags) {
  constexpr int NCW = WARPS_M * WARPS_N;
  constexpr int WM = BM / WARPS_M, WN = BN / WARPS_N;
  constexpr int TM = WM / 16, TN = WN / 8;
  constexpr int PAD = 4;
  constexpr int A_PITCH = MC_A ? BM + PAD : BM, B_PITCH = MC_B ? BN + PAD : BN;
  constexpr uint32_t A_BYTES = A_PITCH * kBK * 8, B_BYTES = B_PITCH * kBK * 8;
  constexpr uint32_t A_SLOT = (A_BYTES + 1023u) & ~1023u, B_SLOT = (B_BYTES + 1023u) & ~1023u;
  constexpr uint32_t STAGE_BYTES = A_SLOT + B_SLOT;
  constexpr int kAcc = TM * TN * 4;  // accumulator doubles per consumer thread

  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t sbase = (raw + 1023u) & ~1023u;
  const uint32_t bars = sbase + STAGES * STAGE_BYTES;
  auto full_bar = [&](int s) { return bars + 8u * s; };
  auto empty_bar = [&](int s) { return bars + 8u * (STAGES + s); };
  auto stage_a = [&](int s) { return sbase + s * STAGE_BYTES; };
  auto stage_b = [&](int s) { return sbase + s * STAGE_BYTES + A_SLOT; };

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = static_cast<int>(blockIdx.x);
  const long long it0 = sk_begin(q, c), it1 = sk_begin(q, c + 1);
  const int KT = q.KT;
  // pieces: whole tiles [tf0, tf1), head (tile th, k-tiles [0, kh)), tail (tile tt, [kt0, KT))
  const int tt = static_cast<int>(it0 / KT), kt0 = static_cast<int>(it0 % KT);
  const bool has_tail = kt0 != 0;
  const int tf0 = has_tail ? tt + 1 : tt;
  const int th = static_cast<int>(it1 / KT), kh = static_cast<int>(it1 % KT);
  const bool has_head = kh != 0;
  const int tf1 = th;
  const int npieces = (tf1 - tf0) + (has_head ? 1 : 0) + (has_tail ? 1 : 0);
  // piece i -> (tile, k0, k1, kind): 0 whole, 1 head, 2 tail
  auto piece = [&](int i, int& tile, int& k0, int& k1) -> int {
    if (i < tf1 - tf0) {
      tile = tf0 + i;
      k0 = 0;
      k1 = KT;
      return 0;
    }
    i -= tf1 - tf0;
    if (has_head && i == 0) {
      tile = th;
      k0 = 0;
      k1 = kh;
      return 1;
    }
    tile = tt;
    k0 = kt0;
    k1 = KT;
    return 2;
  };
  constexpr int kGroup = 16;  // grouped rasterization, as the data-parallel kernel
  auto tile_mn = [&](int t, int& m0, int& n0) {
    const int per_group = kGroup * q.tiles_n;
    const int grp = t / per_group, in_grp = t - grp * per_group;
    const int gm0 = grp * kGroup;
    const int gsize = min(kGroup, q.tiles_m - gm0);
    m0 = (gm0 + in_grp % gsize) * BM;
    n0 = (in_grp / gsize) * BN;
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(empty_bar(s), NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  }
  __syncthreads();

  if (warp == NCW) {  // producer: the same piece order, one k-tile per stage
    if (lane == 0) {
      int it = 0;
      for (int pc = 0; pc < npieces; ++pc) {
        int tile, k0, k1;
        piece(pc, tile, k0, k1);
        int m0, n0;
        tile_mn(tile, m0, n0);
        for (int kf = k0; kf < k1; ++kf, ++it) {
          const int s = it % STAGES;
          if (it >= STAGES) mbar_wait(empty_bar(s), ((it / STAGES) + 1) & 1);
          mbar_expect_tx(full_bar(s), A_BYTES + B_BYTES);
          if (MC_A) tma_load_2d(stage_a(s), &mapA, m0, kf * kBK, full_bar(s));
          else tma_load_2d(stage_a(s), &mapA, kf * kBK, m0, full_bar(s));
          if (MC_B) tma_load_2d(stage_b(s), &mapB, n0, kf * kBK, full_bar(s));
          else tma_load_2d(stage_b(s), &mapB, kf * kBK, n0, full_bar(s));
        }
      }
    }
    return;
  }

  const int g = lane >> 2, t = lane & 3;
  const int wm0 = (warp % WARPS_M) * WM, wn0 = (warp / WARPS_M) * WN;
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
  auto load_frags = [&](int buf, int s, int kk) {
    const uint32_t as = stage_a(s), bs = stage_b(s);
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
      for (int qq = 0; qq < TN / 2; ++qq)
        lds128(bf[buf][2 * qq], bf[buf][2 * qq + 1], bs + b_mc + (kk * 4 * B_PITCH + 16 * qq) * 8);
    } else {
#pragma unroll
      for (int j = 0; j < TN; ++j) lds64(bf[buf][j], bs + b_kc + xo[kk] + (8 * j) * 128);
    }
  };

  double acc[TM][TN][4];
  const int ctid = threadIdx.x;  // consumer thread index (0 .. NCW*32-1)
  int it = 0;
  for (int pc = 0; pc < npieces; ++pc) {
    int tile, k0, k1;
    const int kind = piece(pc, tile, k0, k1);
    int m0, n0;
    tile_mn(tile, m0, n0);
    if (kind == 2) {
      // tail: continue the chain from the neighbour's head partial
      if (ctid == 0) {
        int v = 0;
        uint64_t t0 = 0, now = 0;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        do {
          asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(flags + (c - 1)) : "memory");
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
          // a neighbour that never publishes (not co-resident) fails the launch instead of hanging it
          if (now - t0 > 4000000000ull) __trap();
        } while (v == 0);
      }
      asm volatile("bar.sync 1, %0;\n" ::"r"(NCW * 32) : "memory");
      const double* src = ws + static_cast<size_t>(c - 1) * (NCW * 32 * kAcc);
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j)
#pragma unroll
          for (int e = 0; e < 4; ++e) acc[i][j][e] = __ldcg(src + ((i * TN + j) * 4 + e) * (NCW * 32) + ctid);
      asm volatile("bar.sync 1, %0;\n" ::"r"(NCW * 32) : "memory");
      if (ctid == 0) flags[c - 1] = 0;  // ready for the next launch on this stream
    } else {
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j)
#pragma unroll
          for (int e = 0; e < 4; ++e) acc[i][j][e] = 0.0;
    }
    for (int kt = k0; kt < k1; ++kt, ++it) {
      const int s = it % STAGES;
      mbar_wait(full_bar(s), (it / STAGES) & 1);
      load_frags(0, s, 0);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const int cb = kk & 1;
        if (kk < 3) load_frags(cb ^ 1, s, kk + 1);
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < TN; ++j) dmma1684(acc[i][j], af[cb][i][0], af[cb][i][1], bf[cb][j]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty_bar(s));
    }
    if (kind == 1) {
      // head: publish the partial accumulator for CTA c + 1
      double* dst = ws + static_cast<size_t>(c) * (NCW * 32 * kAcc);
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j)
#pragma unroll
          for (int e = 0; e < 4; ++e) __stcg(dst + ((i * TN + j) * 4 + e) * (NCW * 32) + ctid, acc[i][j][e]);
      __threadfence();
      asm volatile("bar.sync 1, %0;\n" ::"r"(NCW * 32) : "memory");
      if (ctid == 0) asm volatile("st.release.gpu.global.b32 [%0], %1;\n" ::"l"(flags + c), "r"(1) : "memory");
      continue;
    }
    // epilogue (whole tile or tail): C = fma(alpha, acc, beta*C), reads before writes
    const bool beta_zero = p.beta == 0.0;
    auto col_of = [&](int j, int e) -> i64 {
      const int cc = 2 * t + e;
      return n0 + wn0 + (MC_B ? 16 * (j >> 1) + 2 * cc + (j & 1) : 8 * j + (((cc & 3) << 1) | (cc >> 2)));
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
            const i64 nn = col_of(j, e);
            cold[j][e] = (!beta_zero && nn < p.N) ? p.C[m + nn * p.ldc] : 0.0;
          }
#pragma unroll
        for (int j = 0; j < TN; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const i64 nn = col_of(j, e);
            if (nn < p.N) {
              const double v = acc[i][j][2 * h + e];
              p.C[m + nn * p.ldc] = beta_zero ? p.alpha * v : fma(p.alpha, v, p.beta * cold[j][e]);
            }
          }
      }
  }
}

}  // namespace dgemm_tma
}  // namespace rectri_cu
