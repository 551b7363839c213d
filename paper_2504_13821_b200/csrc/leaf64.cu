// leaf64.cu -- fp64 base (leaf) kernel v2: packed triangle, register-fed
// DMMA fragments, warp-specialised GEMM / substitution overlap.
//
// Same contract and the same per-element arithmetic as leaf.cu's kernel
// (trsm_base / trmm_base, src/base_kernels.cpp:94-177, every variant reduced
// to the Left form on a virtual lower factor L' with reflected indices,
// SURVEY.md 3.6), so the two produce identical bits; leaf.cu's kernel stays
// as the fp32 leaf and as the fp64 fallback (RECTRI_CU_LEAF=1, or a stream
// without reserved scratch under capture).
//
// 1. pack_kernel (one launch per leaf call) writes the tile's L' once into a
//    per-stream scratch buffer, in consumption order and in the layouts the
//    consumer reads: off-diagonal 32x32 blocks in DMMA A-fragment order
//    ([row tile mt][lane][k-step] -- each lane's 8 values are 64 contiguous
//    bytes, each warp's 2 KB contiguous), diagonal blocks as
//    Ld[p][r] = L'(r, p) for p < r (0 elsewhere), and the reciprocal
//    diagonal (TRSM) / diagonal (TRMM), 1 for Unit.  Masked and out-of-range
//    entries are written as exact zeros by selection (never a multiply-by-
//    mask); Unit diagonals are never read.  The reflection / transposition
//    address arithmetic happens once per tile instead of once per CTA.
// 2. leaf64_kernel: one CTA owns 32 right-hand sides (panel nb x 32 in
//    shared memory, loaded once, written back once); 8 GEMM warps + 1 solver
//    warp:
//      GEMM warps: per row block I, acc = -b_I + sum_{J<I} L'_IJ X_J with
//        DMMA m8n8k4 (2 tiles per warp).  A fragments come straight from the
//        packed buffer (L2-resident, shared by every CTA) into registers,
//        prefetched kAhead blocks ahead -- no shared staging, no barrier;
//        only the last block of a row (J = I-1) waits for the solver's
//        X_{I-1}.
//      4 solver warps (one per SM sub-partition, 8 right-hand sides each,
//        4 lanes per right-hand side owning rows rq + 4k): the 32x32
//        diagonal block by warp-shuffle forward substitution (TRSM:
//        x_p = v_p * (1/d_p) on the owner lane, broadcast with shfl,
//        v_r = fma(-L'(r,p), x_p, v_r); TRMM: the masked product, no
//        chain), the diagonal block double-buffered in shared memory by
//        cp.async.bulk, so the substitution of row block I overlaps the GEMM
//        of row block I+1.
//    Hand-offs use named barriers (1: accumulators of a row block stored,
//    2: a row block solved).
#include <cstdio>
#include <cstdlib>
#include <map>
#include <vector>
#include <mutex>

#include "common.cuh"
#include "launch.h"

namespace rectri_cu {
namespace leaf64 {

constexpr int kRB = 32;                   // row block
constexpr int kNC = 32;                   // right-hand sides per CTA
constexpr int kGemmWarps = 8;
constexpr int kSolverWarps = 4;  // one per SM sub-partition; 8 right-hand sides each
constexpr int kThreads = (kGemmWarps + kSolverWarps) * 32;
constexpr int kBlk = kRB * kRB;           // doubles per packed block
constexpr int kMaxBlk = kLeafMax / kRB;   // 8 row blocks
constexpr int kMaxOff = kMaxBlk * (kMaxBlk - 1) / 2;
constexpr size_t kScratchDoubles = static_cast<size_t>(kMaxOff + kMaxBlk) * kBlk + kLeafMax;  // >= v3's

__device__ __forceinline__ int panel_idx(int r, int c) { return swz64(r, c, kNC); }

// ------------------------------------------------------------------ packing
// Scratch layout: off-diagonal blocks in consumption order (TRSM: row blocks
// ascending, TRMM descending; J ascending within a row), then the diagonal
// blocks by row block, then dg[kLeafMax].
__device__ __forceinline__ const double* lprime(const LeafParams<double>& p, int r, int j) {
  const int rr = p.reflected ? p.n - 1 - r : r;
  const int jj = p.reflected ? p.n - 1 - j : j;
  const i64 row = p.swapped ? jj : rr;
  const i64 col = p.swapped ? rr : jj;
  return p.A + row + col * p.lda;
}

__global__ void __launch_bounds__(256) pack_kernel(const LeafParams<double> p, double* __restrict__ P) {
  const int nblk = (p.n + kRB - 1) / kRB;
  const int noff = nblk * (nblk - 1) / 2;
  const int b = blockIdx.x;
  const int tid = threadIdx.x;
  if (b == noff + nblk) {  // diagonal values
    double* dg = P + static_cast<size_t>(noff + nblk) * kBlk;
    for (int r = tid; r < kLeafMax; r += blockDim.x) {
      double d = 1.0;
      if (r < p.n && !p.unit) d = *lprime(p, r, r);
      dg[r] = p.trsm ? 1.0 / d : d;
    }
    return;
  }
  if (b >= noff) {  // diagonal block I: Ld[q][r] = L'(r0 + r, r0 + q) for q < r
    const int I = b - noff, r0 = I * kRB;
    double* dst = P + static_cast<size_t>(b) * kBlk;
    for (int o = tid; o < kBlk; o += blockDim.x) {
      const int q = o >> 5, r = o & 31;
      const bool ok = q < r && r0 + r < p.n;
      dst[o] = ok ? *lprime(p, r0 + r, r0 + q) : 0.0;
    }
    return;
  }
  // off-diagonal block number b in consumption order -> (I, J)
  int I, J;
  if (p.trsm) {  // ascending rows: row I holds blocks I(I-1)/2 .. I(I+1)/2 - 1
    I = 1;
    while ((I + 1) * I / 2 <= b) ++I;
    J = b - I * (I - 1) / 2;
  } else {  // descending rows from nblk-1
    I = nblk - 1;
    int base = 0;
    while (base + I <= b) {
      base += I;
      --I;
    }
    J = b - base;
  }
  const int r0 = I * kRB, j0 = J * kRB;
  double* dst = P + static_cast<size_t>(b) * kBlk;
  for (int o = tid; o < kBlk; o += blockDim.x) {
    // A-fragment order: o = (mt*32 + lane)*8 + kk holds L'(8mt + g, 4kk + t)
    const int kk = o & 7, ln = (o >> 3) & 31, mt = o >> 8;
    const int r = 8 * mt + (ln >> 2), j = 4 * kk + (ln & 3);
    const bool ok = r0 + r < p.n;
    dst[o] = ok ? *lprime(p, r0 + r, j0 + j) : 0.0;
  }
}

// -------------------------------------------------------------- primitives
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void named_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void named_arrive(int id, int count) {
  asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}

// ------------------------------------------------------------------ kernel
struct Smem {
  double panel[kLeafMax * kNC];
  double diag[2][kBlk];
  double ys[kRB * kNC];  // TRMM off-diagonal partial sums of the row block being solved
  double dg[kLeafMax];
  unsigned long long dfull[2];
};

__global__ void __launch_bounds__(kThreads, 2) leaf64_kernel(const LeafParams<double> p,
                                                          const double* __restrict__ P) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Smem& S = *reinterpret_cast<Smem*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n = p.n;
  const int nblk = (n + kRB - 1) / kRB;
  const int rows_p = nblk * kRB;
  const int noff = nblk * (nblk - 1) / 2;
  const i64 c0 = static_cast<i64>(blockIdx.x) * kNC;
  const int ncols = static_cast<int>(min(static_cast<i64>(kNC), p.nrhs - c0));
  const bool trsm = p.trsm != 0;
  const double* Poff = P;
  const double* Pdiag = P + static_cast<size_t>(noff) * kBlk;
  const double* Pdg = P + static_cast<size_t>(noff + nblk) * kBlk;
  long long* tr = p.trace ? p.trace + static_cast<size_t>(blockIdx.x) * 48 : nullptr;
  auto stamp = [&](int k) {
    if (tr) tr[k] = clock64();
  };
  if (tid == 0) stamp(0);
  const uint32_t dfull0 = smem_u32(&S.dfull[0]);
  const uint32_t panel_u32 = smem_u32(S.panel);
  auto diag_order = [&](int bi) { return trsm ? bi : nblk - 1 - bi; };  // row block of step bi

  // Panel visitor (the GEMM warps only): Left -> each warp covers 4 rows x 8
  // right-hand sides (32-byte sectors); Right -> one row of 32 per warp.
  const i64 rstep = p.reflected ? -1 : 1;
  auto for_panel = [&](auto&& f) {
    if (!p.right) {
      const int rl = lane & 3, cl = lane >> 2;
#pragma unroll
      for (int cg = 0; cg < kNC / 8; ++cg) {
        const int c = 8 * cg + cl;
        const double* colp = p.B + (c0 + c) * p.ldb + (p.reflected ? n - 1 : 0);
        for (int rt = warp; rt < rows_p / 4; rt += kGemmWarps) {
          const int r = 4 * rt + rl;
          f(r, c, colp + r * rstep);
        }
      }
    } else {
      const int c = lane;
      for (int r = warp; r < rows_p; r += kGemmWarps) {
        const i64 sr = p.reflected ? n - 1 - r : r;
        f(r, c, p.B + sr * p.ldb + c0 + c);
      }
    }
  };

  // TRMM with alpha == 0 writes zeros without reading B (base_kernels.cpp:143-150).
  if (!trsm && p.alpha == 0.0) {
    if (warp < kGemmWarps)
      for_panel([&](int r, int c, const double* g) {
        if (r < n && c < ncols) *const_cast<double*>(g) = 0.0;
      });
    return;
  }

  if (tid == 0) {
    mbar_init(dfull0, 1);
    mbar_init(dfull0 + 8, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {  // diagonal blocks of steps 0 and 1 (+ dg with the first)
    mbar_expect_tx(dfull0, kBlk * 8 + kLeafMax * 8);
    bulk_g2s(smem_u32(S.diag[0]), Pdiag + static_cast<size_t>(diag_order(0)) * kBlk, kBlk * 8, dfull0);
    bulk_g2s(smem_u32(S.dg), Pdg, kLeafMax * 8, dfull0);
    if (nblk > 1) {
      mbar_expect_tx(dfull0 + 8, kBlk * 8);
      bulk_g2s(smem_u32(S.diag[1]), Pdiag + static_cast<size_t>(diag_order(1)) * kBlk, kBlk * 8, dfull0 + 8);
    }
  }
  if (warp < kGemmWarps)
    for_panel([&](int r, int c, const double* g) {
      const bool ok = r < n && c < ncols;
      cp_async8(S.panel + panel_idx(r, c), ok ? g : p.B, ok ? 8 : 0);
    });
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  if (tid == 0) stamp(1);
  if (trsm && p.alpha != 1.0) {  // x = alpha * b (base_kernels.cpp:76-77)
    if (warp < kGemmWarps)
      for_panel([&](int r, int c, const double*) { S.panel[panel_idx(r, c)] *= p.alpha; });
    __syncthreads();
  }

  if (warp < kGemmWarps) {
    if (p.debug_skip == 4) return;  // timing experiment: solver warps alone
    // ------------------------------------------------------- GEMM warps
    // warp w owns the m8n8 tiles (w & 3, 2*(w >> 2) + e), e = 0, 1.
    const int g = lane >> 2, t = lane & 3;
    const int mt = warp & 3, nt0 = 2 * (warp >> 2);
    uint32_t b_base[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) b_base[e] = 8u * static_cast<uint32_t>(swz64(t, 8 * (nt0 + e) + g, kNC));
    // this lane's A fragments of packed block s: 8 contiguous doubles,
    // fetched one block ahead into registers
    const double* pa_base = Poff + (mt * 32 + lane) * 8;
    double nxt[8];
    auto fetch = [&](int sblk) {
      const double2* src = reinterpret_cast<const double2*>(pa_base + static_cast<size_t>(sblk) * kBlk);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double2 v = __ldg(src + q);
        nxt[2 * q] = v.x;
        nxt[2 * q + 1] = v.y;
      }
    };
    if (noff > 0) fetch(0);
    double c[2][2];
    int s = 0;         // off-diagonal sequence index
    int x_synced = 0;  // solves this warp has waited for
    for (int bi = 0; bi < nblk; ++bi) {
      const int I = diag_order(bi);
      const int r0 = I * kRB;
      if (trsm) {
#pragma unroll
        for (int e = 0; e < 2; ++e)
#pragma unroll
          for (int h = 0; h < 2; ++h) c[e][h] = -S.panel[panel_idx(r0 + 8 * mt + g, 8 * (nt0 + e) + 2 * t + h)];
      } else {
        c[0][0] = c[0][1] = c[1][0] = c[1][1] = 0.0;
      }
      for (int J = 0; J < I; ++J, ++s) {
        double a[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = nxt[k];
        if (s + 1 < noff) fetch(s + 1);
        if (trsm && J == I - 1) {  // X_{I-1} must be solved
          named_sync(2, kThreads);
          ++x_synced;
          if (tid == 0) stamp(2 + 4 * bi + 3);
        }
        const uint32_t pb = panel_u32 + static_cast<uint32_t>(J * kRB * kNC * 8);
        if (p.debug_skip == 2) continue;  // timing experiment: no GEMM part
        // all 8 k-steps' B fragments first: one shared-memory latency per block
        double bv[kRB / 4][2];
#pragma unroll
        for (int kk = 0; kk < kRB / 4; ++kk)
#pragma unroll
          for (int e = 0; e < 2; ++e)
            asm volatile("ld.shared.f64 %0, [%1];" : "=d"(bv[kk][e]) : "r"(pb + b_base[e] + kk * 4 * kNC * 8));
#pragma unroll
        for (int kk = 0; kk < kRB / 4; ++kk)
#pragma unroll
          for (int e = 0; e < 2; ++e) dmma884(c[e][0], c[e][1], a[kk], bv[kk][e]);
      }
      if (trsm) {
        // b' = b - sum L'x into the panel rows of block I (the solver's input)
#pragma unroll
        for (int e = 0; e < 2; ++e)
#pragma unroll
          for (int h = 0; h < 2; ++h)
            S.panel[panel_idx(r0 + 8 * mt + g, 8 * (nt0 + e) + 2 * t + h)] = -c[e][h];
      } else {
        // ys was last read by the solve of step bi - 1
        if (bi >= 1) {
          named_sync(2, kThreads);
          ++x_synced;
        }
#pragma unroll
        for (int e = 0; e < 2; ++e)
#pragma unroll
          for (int h = 0; h < 2; ++h)
            S.ys[panel_idx(8 * mt + g, 8 * (nt0 + e) + 2 * t + h)] = c[e][h];
      }
      if (tid == 0) stamp(2 + 4 * bi + 2);
      named_arrive(1, kThreads);  // accumulators of row block I are stored
    }
    while (x_synced < nblk) {  // every solve done before the write-back
      named_sync(2, kThreads);
      ++x_synced;
    }
    if (tid == 0) stamp(40);
    for_panel([&](int r, int cc, const double* gp) {
      if (r < n && cc < ncols) *const_cast<double*>(gp) = S.panel[panel_idx(r, cc)];
    });
    if (tid == 0) stamp(41);
  } else {
    // ------------------------------------------------------- solver warps
    const int sw = warp - kGemmWarps;
    const int cc = 8 * sw + (lane >> 2);  // right-hand side
    const int rq = lane & 3;              // rows rq + 4k, k = 0..7
    const unsigned grp = lane & ~3u;
    for (int bi = 0; bi < nblk; ++bi) {
      const int I = diag_order(bi);
      const int r0 = I * kRB;
      const int db = bi & 1;
      mbar_wait(dfull0 + 8 * db, (bi >> 1) & 1);  // diagonal block I (and, first time, dg)
      if (p.debug_skip != 4) named_sync(1, kThreads);  // accumulators of row block I stored
      if (sw == 0 && lane == 0) stamp(2 + 4 * bi);
      double v[8];
      const double* Ld = S.diag[db];
      if (trsm) {
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = S.panel[panel_idx(r0 + rq + 4 * k, cc)];
        // L' values of step q for this lane's rows, loaded one step ahead so
        // no shared-memory latency sits on the substitution chain
        double ln[8], dn = S.dg[r0 + rq];
#pragma unroll
        for (int k = 0; k < 8; ++k) ln[k] = Ld[rq + 4 * k];
#pragma unroll
        for (int q = 0; q < kRB; ++q) {
          const int kq = q >> 2, oq = q & 3;
          double lc[8];
#pragma unroll
          for (int k = kq; k < 8; ++k) lc[k] = ln[k];
          const double dc = dn;
          if (q + 1 < kRB) {
#pragma unroll
            for (int k = (q + 1) >> 2; k < 8; ++k) ln[k] = Ld[(q + 1) * kRB + rq + 4 * k];
            if (((q + 1) & 3) == 0) dn = S.dg[r0 + q + 1 + rq];  // next owner rows rq + 4k
          }
          double x = 0.0;
          if (rq == oq) {  // owner of row q (dc = 1/d of row rq + 4kq = q)
            x = v[kq] * dc;
            v[kq] = x;
          }
          x = __shfl_sync(0xffffffffu, x, grp | oq);
          // rows rq + 4k > q: all k > kq, and k == kq when rq > oq (selected,
          // so a non-finite x never reaches a row it does not feed)
          {
            const double nv = fma(-lc[kq], x, v[kq]);
            v[kq] = rq > oq ? nv : v[kq];
          }
#pragma unroll
          for (int k = kq + 1; k < 8; ++k) v[k] = fma(-lc[k], x, v[k]);
        }
      } else {
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = S.ys[panel_idx(rq + 4 * k, cc)];
#pragma unroll
        for (int q = 0; q < kRB; ++q) {
          const double bq = S.panel[panel_idx(r0 + q, cc)];  // rows of I are written after the loop
          const int kq = q >> 2, oq = q & 3;
          {  // row rq + 4kq: diagonal when rq == oq, L' when rq > oq, untouched below
            const double coef = rq == oq ? S.dg[r0 + q] : Ld[q * kRB + rq + 4 * kq];
            const double nv = fma(coef, bq, v[kq]);
            v[kq] = rq >= oq ? nv : v[kq];
          }
#pragma unroll
          for (int k = kq + 1; k < 8; ++k) v[k] = fma(Ld[q * kRB + rq + 4 * k], bq, v[k]);
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = p.alpha * v[k];
        __syncwarp();  // the 4 lanes of a right-hand side (same warp) have read b_I
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) S.panel[panel_idx(r0 + rq + 4 * k, cc)] = v[k];
      named_sync(3, kSolverWarps * 32);  // all solver warps done with diag[db]
      if (sw == 0 && lane == 0) {
        stamp(2 + 4 * bi + 1);
        if (bi + 2 < nblk) {  // step bi + 2's diagonal block into the freed buffer
          asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
          mbar_expect_tx(dfull0 + 8 * db, kBlk * 8);
          bulk_g2s(smem_u32(S.diag[db]), Pdiag + static_cast<size_t>(diag_order(bi + 2)) * kBlk, kBlk * 8,
                   dfull0 + 8 * db);
        }
      }
      if (p.debug_skip != 4) named_arrive(2, kThreads);  // row block I solved
    }
  }
}

// ------------------------------------------------------------------ host
std::mutex g_mu;
std::map<std::pair<int, cudaStream_t>, double*> g_scratch;

double* scratch_for(cudaStream_t s, bool may_alloc) {
  if (const CallScratch* cs = call_scratch()) {  // a graph capture: the graph's own buffer
    const int k = cs->find(s);
    return k >= 0 ? cs->leaf[k] : nullptr;
  }
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(g_mu);
  auto it = g_scratch.find({dev, s});
  if (it != g_scratch.end()) return it->second;
  if (!may_alloc) return nullptr;
  double* ptr = nullptr;
  if (cudaMalloc(&ptr, kScratchDoubles * sizeof(double)) != cudaSuccess) return nullptr;
  g_scratch[{dev, s}] = ptr;
  return ptr;
}

int leaf_version_env() {
  // 3 (default): explicit-inverse diagonal blocks as DMMA products
  // (leaf64_v3.cu); 4: the same, with v5 (leaf64_v5.cu, row-block-owning
  // warps, bitwise the same) for recursion TRMM leaves with few right-hand
  // sides; 2: warp-shuffle substitution in the reference's order, bitwise
  // equal to v1 (leaf.cu).
  const char* e = getenv("RECTRI_CU_LEAF");
  return e ? atoi(e) : 3;
}

}  // namespace leaf64

int leaf_version() { return leaf64::leaf_version_env(); }

void launch_leaf_f32(const LeafParams<float>& p, cudaStream_t s) {
  if (p.n <= 0 || p.nrhs <= 0) return;
  if (p.packed) {  // triangle packed once for the whole recursion
    launch_leaf_f32_v3(p, reinterpret_cast<float*>(p.packed), s, true);
    return;
  }
  double* P = nullptr;
  if (leaf64::leaf_version_env() >= 3) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &cs);
    P = leaf64::scratch_for(s, cs == cudaStreamCaptureStatusNone);  // >= the fp32 blocks' bytes
  }
  if (P) launch_leaf_f32_v3(p, reinterpret_cast<float*>(P), s);
  else launch_leaf_f32_v1(p, s);
}

void leaf_scratch_reserve(cudaStream_t s) { leaf64::scratch_for(s, true); }

size_t leaf_scratch_bytes() { return leaf64::kScratchDoubles * sizeof(double); }

namespace {
thread_local const CallScratch* t_call_scratch = nullptr;
}
void set_call_scratch(const CallScratch* cs) { t_call_scratch = cs; }
const CallScratch* call_scratch() { return t_call_scratch; }

void launch_leaf_f64(const LeafParams<double>& p, cudaStream_t s) {
  using namespace leaf64;
  if (p.n <= 0 || p.nrhs <= 0) return;
  if (p.packed) {  // triangle packed once for the whole recursion
    launch_leaf_f64_v3(p, p.packed, s, true);
    return;
  }
  double* P = nullptr;
  if (leaf64::leaf_version_env() >= 2) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &cs);
    P = scratch_for(s, cs == cudaStreamCaptureStatusNone);
  }
  if (!P) {  // leaf.cu's kernel
    launch_leaf_f64_v1(p, s);
    return;
  }
  if (leaf64::leaf_version_env() >= 3) {
    launch_leaf_f64_v3(p, P, s);
    return;
  }
  const int nblk = (p.n + kRB - 1) / kRB;
  const int noff = nblk * (nblk - 1) / 2;
  const bool zero = !p.trsm && p.alpha == 0.0;
  LeafParams<double> pd = p;
  if (const char* e = getenv("RECTRI_CU_LEAF_DEBUG")) pd.debug_skip = atoi(e);
  if (!zero) {
    pack_kernel<<<noff + nblk + 1, 256, 0, s>>>(p, P);
    ++launch_counter();
  }
  const int smem = static_cast<int>(sizeof(Smem));
  set_smem(leaf64_kernel, smem);
  const unsigned grid = static_cast<unsigned>(ceil_div(p.nrhs, kNC));
  const char* tr = getenv("RECTRI_CU_LEAF_TRACE");
  if (tr && atoi(tr)) {  // diagnostics: per-CTA phase stamps, summary on stderr
    LeafParams<double> q = pd;
    long long* d = nullptr;
    cudaMalloc(&d, grid * 48 * sizeof(long long));
    cudaMemset(d, 0, grid * 48 * sizeof(long long));
    q.trace = d;
    leaf64_kernel<<<grid, kThreads, smem, s>>>(q, P);
    cudaStreamSynchronize(s);
    std::vector<long long> h(grid * 48);
    cudaMemcpy(h.data(), d, h.size() * sizeof(long long), cudaMemcpyDeviceToHost);
    cudaFree(d);
    const int nb = (p.n + kRB - 1) / kRB;
    double acc[48] = {0};
    for (unsigned b = 0; b < grid; ++b)
      for (int k = 1; k < 48; ++k)
        if (h[b * 48 + k]) acc[k] += static_cast<double>(h[b * 48 + k] - h[b * 48]);
    fprintf(stderr, "leaf64 trace (mean cycles from CTA start, %u CTAs): panel %.0f\n", grid, acc[1] / grid);
    for (int bi = 0; bi < nb; ++bi)
      fprintf(stderr, "  step %d: gemm x-synced %.0f  acc-stored %.0f  solver got-acc %.0f  solved %.0f\n", bi,
              acc[2 + 4 * bi + 3] / grid, acc[2 + 4 * bi + 2] / grid, acc[2 + 4 * bi] / grid,
              acc[2 + 4 * bi + 1] / grid);
    fprintf(stderr, "  writeback start %.0f end %.0f\n", acc[40] / grid, acc[41] / grid);
    ++launch_counter();
    return;
  }
  leaf64_kernel<<<grid, kThreads, smem, s>>>(pd, P);
  ++launch_counter();
}

}  // namespace rectri_cu
