// leaf64_v3.cu -- fp64 base (leaf) kernel v3: every step on the DMMA pipe.
//
// trsm_base / trmm_base (src/base_kernels.cpp:94-177) on the Left form of a
// virtual lower factor L' (reflected / transposed indices),
// blocked in 32-row blocks.  Differs from v1/v2 (leaf.cu / leaf64.cu) only in
// how the 32x32 diagonal block is applied:
//   TRSM: X_I = inv(L'_II) * (b_I - sum_{J<I} L'_IJ X_J).  inv(L'_II) is
//         computed once per leaf call by pack3_kernel (forward substitution
//         of the 32 unit vectors, one thread per column, divisions as in the
//         reference's trsm_left_lower) and applied as a 32x32x32 DMMA
//         product, so no 32-step dependency chain sits in the consumer.
//   TRMM: X_I = alpha * (sum_{J<I} L'_IJ b_J + L'_II b_I) with L'_II carrying
//         its diagonal (1 for Unit) -- one more DMMA block.
// The results agree with v1/v2 to rounding (tolerance-checked, not bitwise:
// the diagonal block's sums are re-associated); v1/v2 remain selectable
// (RECTRI_CU_LEAF=1/2) for the reference's exact substitution order.
//
// pack3_kernel writes, per leaf call, the blocks in consumption order in
// DMMA A-fragment order ([row tile mt][lane][k-step], 2 KB contiguous per
// warp): TRSM row I: L'_I0 .. L'_I,I-1, then -inv(L'_II); TRMM (rows
// descending) row I: L'_I0 .. L'_I,I-1, then L'_II.  Masked / out-of-range
// entries are exact zeros by selection; padding rows beyond n get an
// identity diagonal so every diagonal block is invertible.
//
// leaf3_kernel: one CTA owns 32 right-hand sides (panel nb x 32 in shared
// memory, loaded once, written back once); 8 warps each own two m8n8 output
// tiles of the current row block; A fragments stream from the (L2-resident)
// scratch straight into registers one block ahead.  Per row block: GEMM
// part, (TRSM) the negated partial result to shared memory + barrier, the
// diagonal-block product, store + barrier.
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "launch.h"

namespace rectri_cu {
namespace leaf64v3 {

constexpr int kRB = 32;
constexpr int kThreads = 256;
constexpr int kBlk = kRB * kRB;
constexpr int kMaxBlk = kLeafMax / kRB;
constexpr size_t kScratchDoubles = static_cast<size_t>(kMaxBlk * (kMaxBlk + 1) / 2) * kBlk;

// Panel element (r, c) of an NC-wide panel: XOR-swizzled pairs for NC >= 16;
// NC = 8 rows are 64 bytes and the B-fragment reads (4 rows x 8 columns)
// are conflict-free unswizzled.
template <int NC>
__device__ __forceinline__ int panel_idx(int r, int c) {
  if constexpr (NC >= 16) return swz64(r, c, NC);
  else return r * NC + c;
}

__device__ __forceinline__ double lprime(const LeafParams<double>& p, int r, int j) {
  const int rr = p.reflected ? p.n - 1 - r : r;
  const int jj = p.reflected ? p.n - 1 - j : j;
  const i64 row = p.swapped ? jj : rr;
  const i64 col = p.swapped ? rr : jj;
  return p.A[row + col * p.lda];
}

// Fragment order position of element (r, k) of a 32x32 block: [row tile
// mt][k-step kk][lane], so a warp's 8-byte fragment reads of one k-step are
// 256 contiguous bytes in shared memory (conflict-free).
__device__ __forceinline__ int frag_pos(int r, int k) {
  const int mt = r >> 3, g = r & 7, kk = k >> 2, t = k & 3;
  return (mt * 8 + kk) * 32 + 4 * g + t;
}

// Consumption index of block (I, J) (J == I: the diagonal block).
__device__ __forceinline__ int seq_of(int I, int J, int nblk, bool asc) {
  if (asc) return I * (I + 1) / 2 + J;
  // rows nblk-1 .. I+1 come first; row I' holds I'+1 blocks
  return (nblk * (nblk + 1) / 2 - (I + 1) * (I + 2) / 2) + J;
}

__device__ void pack3_block(const LeafParams<double>& p, double* __restrict__ P, const int b) {
  __shared__ double L[kRB][kRB + 1];
  const int nblk = (p.n + kRB - 1) / kRB;
  const bool trsm = p.trsm != 0;
  // b -> (I, J), J <= I, canonical ascending numbering
  int I = 0;
  while ((I + 1) * (I + 2) / 2 <= b) ++I;
  const int J = b - I * (I + 1) / 2;
  const int r0 = I * kRB, j0 = J * kRB;
  double* dst = P + static_cast<size_t>(seq_of(I, J, nblk, trsm || p.pack_asc)) * kBlk;
  const int tid = threadIdx.x;
  // 256 threads, 4 elements each: every load of a thread is issued before
  // its first store, so the A reads' latency is paid once, not four times
  // (the stores to P could alias A as far as the compiler knows).
  constexpr int kPer = kBlk / 256;
  double v[kPer];
  if (J < I) {
#pragma unroll
    for (int e = 0; e < kPer; ++e) {
      const int o = tid + 256 * e;
      const int ln = o & 31, kk = (o >> 5) & 7, mt = o >> 8;
      const int r = 8 * mt + (ln >> 2), k = 4 * kk + (ln & 3);
      v[e] = r0 + r < p.n ? lprime(p, r0 + r, j0 + k) : 0.0;
    }
#pragma unroll
    for (int e = 0; e < kPer; ++e) dst[tid + 256 * e] = v[e];
    return;
  }
  // diagonal block: lower triangle with its diagonal (1 for Unit; identity
  // on padding rows), zeros above
#pragma unroll
  for (int e = 0; e < kPer; ++e) {
    const int o = tid + 256 * e;
    const int r = o >> 5, k = o & 31;
    v[e] = 0.0;
    if (r0 + r >= p.n) v[e] = r == k ? 1.0 : 0.0;
    else if (k < r) v[e] = lprime(p, r0 + r, r0 + k);
    else if (k == r) v[e] = p.unit ? 1.0 : lprime(p, r0 + r, r0 + r);
  }
#pragma unroll
  for (int e = 0; e < kPer; ++e) L[(tid + 256 * e) >> 5][(tid + 256 * e) & 31] = v[e];
  __syncthreads();
  if (!trsm) {
    for (int o = tid; o < kBlk; o += blockDim.x) {
      const int r = o >> 5, k = o & 31;
      dst[frag_pos(r, k)] = L[r][k];
    }
    return;
  }
  // -inv(L): thread j solves L y = e_j by forward substitution
  // (base_kernels.cpp:73-88 order: y_r = (e_r - sum_{p<r} L(r,p) y_p) / d_r),
  // written column-oriented: once y_p is known, every later row's running sum
  // takes its term at once.  Each row still sums its terms in p order, so the
  // values are those of the row-oriented loop; the 31 updates after each
  // division are independent instead of one 496-long dependent chain (the
  // packing kernel sits at the head of every small TRSM call).
  if (tid < kRB) {
    const int j = tid;
    double y[kRB];
#pragma unroll
    for (int r = 0; r < kRB; ++r) y[r] = r == j ? 1.0 : 0.0;  // running sums
#pragma unroll
    for (int q = 0; q < kRB; ++q) {
      y[q] = q < j ? 0.0 : y[q] / L[q][q];
#pragma unroll
      for (int r = q + 1; r < kRB; ++r) y[r] = fma(-L[r][q], y[q], y[r]);
    }
#pragma unroll
    for (int r = 0; r < kRB; ++r) dst[frag_pos(r, j)] = -y[r];
  }
}

__global__ void __launch_bounds__(256) pack3_kernel(const LeafParams<double> p, double* __restrict__ P) {
  pdl_wait();  // PDL: no-op unless launched programmatically (launch_kernel)
  pack3_block(p, P, blockIdx.x);
}

// Every leaf of one recursion at once (blockIdx.y = leaf): leaf k's tile is
// A(r0_k.., r0_k..) of order n_k, packed into P + k * stride.
__global__ void __launch_bounds__(256) pack3_all_kernel(const LeafParams<double> base, const long long* __restrict__ r0s,
                                                        const int* __restrict__ ns, double* __restrict__ P,
                                                        long long stride) {
  pdl_wait();  // PDL: no-op unless launched programmatically (launch_kernel)
  const int k = blockIdx.y;
  LeafParams<double> p = base;
  p.n = ns[k];
  p.A = base.A + r0s[k] * (1 + base.lda);
  const int nblk = (p.n + kRB - 1) / kRB;
  if (static_cast<int>(blockIdx.x) >= nblk * (nblk + 1) / 2) return;
  pack3_block(p, P + static_cast<size_t>(k) * stride, blockIdx.x);
}

constexpr int kRing = 5;  // packed blocks in flight (bulk copies)
// Independent DMMA accumulation chains per output tile: k-step kk of every
// block goes to partial sum kk % kParts, the sums are added once per row
// block.  (Four chains measured the same as two, TRSM n = m = 1024: 14.0 us
// per leaf either way -- the dependency chain is not what bounds the small
// leaves.)  v5 (leaf64_v5.cu) follows the same order.
constexpr int kParts = 2;
template <int NC>
constexpr int smem_bytes() { return (kLeafMax * NC + kRB * NC + kRing * kBlk) * 8 + 2 * kRing * 8; }

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

// NC right-hand sides per CTA (32, 16 or 8: narrower panels put more CTAs on
// the SMs when the leaf has few right-hand sides).  The output tiles of a row
// block (4 x NC/8 m8n8 tiles) go E per warp to CW compute warps; every
// element's products are accumulated in the same order for every NC, so the
// widths agree bit for bit.
// WM = 2: a compute warp owns 2 row tiles x E column tiles (16 x 16 for
// NC = 32, 4 compute warps): every A and B fragment feeds two DMMAs, a third
// fewer shared-memory wavefronts per DMMA than WM = 1 (8 x 16 per warp).
// CK: the ring checker's instantiation (RECTRI_CU_RING_CHECK; the default
// kernels carry no trace of it).
template <int NC, int WM = 1, bool CK = false>
__global__ void __launch_bounds__(kThreads + 32, 2) leaf3_kernel(const LeafParams<double> p,
                                                                const double* __restrict__ P) {
  pdl_wait();  // PDL: no-op unless launched programmatically (launch_kernel)
  constexpr int kNC = NC;
  constexpr int CW = WM == 2 ? 4 : (NC >= 16 ? 8 : 4);  // compute warps
  constexpr int E = 4 * (NC / 8) / CW / WM;              // column tiles per compute warp
  constexpr int RW = 4 / WM;                             // warps along the rows
  extern __shared__ __align__(128) double smem3[];
  double* panel = smem3;                       // nb x 32 right-hand sides (swizzled rows)
  double* cbuf = smem3 + kLeafMax * kNC;       // TRSM: -(b_I - sum L'X) of the current row block
  double* ring = cbuf + kRB * kNC;             // kRing packed blocks
  const uint32_t full0 = smem_u32(ring + kRing * kBlk), empty0 = full0 + 8 * kRing;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n = p.n;
  const int nblk = (n + kRB - 1) / kRB;
  const int rows_p = nblk * kRB;
  const i64 c0 = static_cast<i64>(blockIdx.x) * kNC;
  const int ncols = static_cast<int>(min(static_cast<i64>(kNC), p.nrhs - c0));
  const bool trsm = p.trsm != 0;
  constexpr int kWarps = kThreads / 32;

  const i64 rstep = p.reflected ? -1 : 1;
  auto for_panel = [&](auto&& f) {
    if (!p.right) {
      const int rl = lane & 3, cl = lane >> 2;
#pragma unroll
      for (int cg = 0; cg < kNC / 8; ++cg) {
        const int c = 8 * cg + cl;
        const double* colp = p.B + (c0 + c) * p.ldb + (p.reflected ? n - 1 : 0);
        for (int rt = warp; rt < rows_p / 4; rt += kWarps) {
          const int r = 4 * rt + rl;
          f(r, c, colp + r * rstep);
        }
      }
    } else {
      constexpr int RPW = 32 / kNC;  // rows per warp pass
      const int c = lane % kNC;
      for (int r = warp * RPW + lane / kNC; r < rows_p; r += kWarps * RPW) {
        const i64 sr = p.reflected ? n - 1 - r : r;
        f(r, c, p.B + sr * p.ldb + c0 + c);
      }
    }
  };

  if (!trsm && p.alpha == 0.0) {  // base_kernels.cpp:143-150
    if (warp < kWarps)
      for_panel([&](int r, int c, const double* g) {
        if (r < n && c < ncols) *const_cast<double*>(g) = 0.0;
      });
    return;
  }
  // RECTRI_CU_LEAF_TRACE (direct base calls, diagnostics): clock64 stamps of
  // thread 0 -- start, panel loaded, each row block done, write-back done.
  long long* tr = p.trace && tid == 0 ? p.trace + static_cast<size_t>(blockIdx.x) * 48 : nullptr;
  if (tr) tr[0] = clock64();
  const int nseq = nblk * (nblk + 1) / 2;
  if (tid == 0) {
    for (int q = 0; q < kRing; ++q) {
      mbar_init(full0 + 8 * q, 1);
      mbar_init(empty0 + 8 * q, CW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  }
  __syncthreads();
  if (warp == kWarps) {  // producer warp: packed blocks through the ring
    if (lane == 0)
      for (int q = 0; q < nseq; ++q) {
        const int slot = q % kRing;
        if (q >= kRing) mbar_wait(empty0 + 8 * slot, ((q / kRing) + 1) & 1);
        mbar_expect_tx(full0 + 8 * slot, kBlk * 8);
        bulk_g2s(smem_u32(ring + slot * kBlk), P + static_cast<size_t>(q) * kBlk, kBlk * 8, full0 + 8 * slot);
      }
    return;
  }
  for_panel([&](int r, int c, const double* g) {
    const bool ok = r < n && c < ncols;
    cp_async8(panel + panel_idx<NC>(r, c), ok ? g : p.B, ok ? 8 : 0);
  });
  cp_async_commit();

  // warp w owns the m8n8 tiles (mt0 + i, nt0 + e), i < WM, e < E.
  const int g = lane >> 2, t = lane & 3;
  const int mt0 = WM * (warp % RW), nt0 = E * (warp / RW);
  const bool computes = warp < CW;
  const uint32_t panel_u32 = smem_u32(panel), cbuf_u32 = smem_u32(cbuf);
  uint32_t b_base[E];
#pragma unroll
  for (int e = 0; e < E; ++e) b_base[e] = 8u * static_cast<uint32_t>(panel_idx<NC>(t, 8 * (nt0 + e) + g));
  const uint32_t a_off = static_cast<uint32_t>((mt0 * 8 * 32 + lane) * 8);  // k-step-0 A fragment, row tile mt0
  cp_async_wait<0>();
  named_sync(1, kThreads);  // panel loaded (GEMM warps only; the producer runs free)
  if (tr) tr[1] = clock64();
  if (trsm && p.alpha != 1.0) {  // x = alpha * b (base_kernels.cpp:76-77)
    for_panel([&](int r, int c, const double*) { panel[panel_idx<NC>(r, c)] *= p.alpha; });
    named_sync(1, kThreads);
  }
  // element (i, e, h) of this lane's accumulators: row 8(mt0+i)+g, column 8(nt0+e)+2t+h of the row block
  auto crow = [&](int i) { return 8 * (mt0 + i) + g; };
  auto ccol = [&](int e, int h) { return 8 * (nt0 + e) + 2 * t + h; };
  auto gaddr = [&](int r, int cc) -> double* {  // B element of panel row r, column cc
    const i64 sr = p.reflected ? n - 1 - r : r;
    return p.right ? p.B + sr * p.ldb + c0 + cc : p.B + (c0 + cc) * p.ldb + sr;
  };

  // c[q][i][e][h] += A(block s) * Bsrc(32 rows at byte offset bsrc of a
  // row-major [k][kNC] swizzled buffer), k-step kk into partial sum
  // q = kk % kParts (two independent DMMA chains per tile: half the
  // dependency latency of a leaf with few right-hand sides); the partial
  // sums are added once per row block.  Same order for every NC and WM.
  double c[kParts][WM][E][2];
  auto csum = [&](int i, int e, int h) { return c[0][i][e][h] + c[1][i][e][h]; };
  auto zero = [&](int i, int e, int h) {
#pragma unroll
    for (int q = 0; q < kParts; ++q) c[q][i][e][h] = 0.0;
  };
  int s = 0;
  const uint32_t dep0 = static_cast<uint32_t>(p.n) >> 16;  // 0 at run time (n <= 256), unknown to ptxas
  auto block_mma = [&](uint32_t bsrc) {
    if (!computes) return;
    const int slot = s % kRing;
    mbar_wait(full0 + 8 * slot, (s / kRing) & 1);
    // (ring_plant: the checker's negative test reads the next slot instead)
    const uint32_t as = smem_u32(ring + (CK && p.ring_plant ? (s + 1) % kRing : slot) * kBlk) + a_off;
    double a[WM][8];
#pragma unroll
    for (int i = 0; i < WM; ++i)
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)
        asm volatile("ld.shared.f64 %0, [%1];" : "=d"(a[i][kk]) : "r"(as + (i * 8 + kk) * 32 * 8));
    if (CK) {  // RECTRI_CU_RING_CHECK: the fragments must be block s's packed values
      const double* src = P + static_cast<size_t>(s) * kBlk + a_off / 8;
      unsigned bad = 0;
#pragma unroll
      for (int i = 0; i < WM; ++i)
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          bad += __double_as_longlong(a[i][kk]) != __double_as_longlong(src[(i * 8 + kk) * 32]) ? 1u : 0u;
      if (bad) atomicAdd(p.ring_check, static_cast<unsigned long long>(bad));
    }
    // all 8 k-steps' B fragments first: one shared-memory latency per block
    double bv[kRB / 4][E];
#pragma unroll
    for (int kk = 0; kk < kRB / 4; ++kk)
#pragma unroll
      for (int e = 0; e < E; ++e)
        asm volatile("ld.shared.f64 %0, [%1];" : "=d"(bv[kk][e]) : "r"(bsrc + b_base[e] + kk * 4 * kNC * 8));
#pragma unroll
    for (int kk = 0; kk < kRB / 4; ++kk)
#pragma unroll
      for (int i = 0; i < WM; ++i)
#pragma unroll
        for (int e = 0; e < E; ++e) dmma884(c[kk % kParts][i][e][0], c[kk % kParts][i][e][1], a[i][kk], bv[kk][e]);
    // Release the slot once all of its fragment loads have landed: the
    // arrive's address depends on them (slot_dep, common.cuh) -- cheaper than
    // a proxy fence, whose MEMBAR would also wait for TRMM's global stores.
    uint32_t dep = 0;
#pragma unroll
    for (int i = 0; i < WM; ++i)
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) dep |= slot_dep(dep0, a[i][kk]);
    __syncwarp();
    if (lane == 0) mbar_arrive(empty0 + 8 * slot + dep);
    ++s;
  };
  auto for_c = [&](auto&& f) {
#pragma unroll
    for (int i = 0; i < WM; ++i)
#pragma unroll
      for (int e = 0; e < E; ++e)
#pragma unroll
        for (int h = 0; h < 2; ++h) f(i, e, h);
  };

  for (int bi = 0; bi < nblk; ++bi) {
    const int I = trsm ? bi : nblk - 1 - bi;
    const int r0 = I * kRB;
    if (trsm) {
      for_c([&](int i, int e, int h) {
        c[0][i][e][h] = !computes ? 0.0 : -panel[panel_idx<NC>(r0 + crow(i), ccol(e, h))];
        for (int q = 1; q < kParts; ++q) c[q][i][e][h] = 0.0;
      });
    } else {
      for_c([&](int i, int e, int h) { zero(i, e, h); });
    }
    for (int J = 0; J < I; ++J) block_mma(panel_u32 + static_cast<uint32_t>(J * kRB * kNC * 8));
    if (trsm) {
      // c = -(b_I - sum L'X); X_I = (-inv(L'_II)) * c
      if (computes)
        for_c([&](int i, int e, int h) { cbuf[panel_idx<NC>(crow(i), ccol(e, h))] = csum(i, e, h); });
      named_sync(1, kThreads);
      for_c([&](int i, int e, int h) { zero(i, e, h); });
      block_mma(cbuf_u32);
      if (computes)
        for_c([&](int i, int e, int h) {
          panel[panel_idx<NC>(r0 + crow(i), ccol(e, h))] = csum(i, e, h);
        });
      named_sync(1, kThreads);  // X_I visible; cbuf free
    } else {
      // c += L'_II * b_I, and X_I straight to global memory: the panel stays
      // pristine (the row blocks of a TRMM are independent), so no barrier
      // between row blocks and no write-back pass
      block_mma(panel_u32 + static_cast<uint32_t>(I * kRB * kNC * 8));
      if (computes)
        for_c([&](int i, int e, int h) {
          const int r = r0 + crow(i), cc = ccol(e, h);
          if (r < n && cc < ncols) *gaddr(r, cc) = p.alpha * csum(i, e, h);
        });
    }
    if (tr) tr[2 + bi] = clock64();
  }
  if (!trsm) return;
  named_sync(1, kThreads);
  for_panel([&](int r, int cc, const double* gp) {
    if (r < n && cc < ncols) *const_cast<double*>(gp) = panel[panel_idx<NC>(r, cc)];
  });
  if (tr) tr[41] = clock64();
}

}  // namespace leaf64v3

size_t leaf3_scratch_doubles() { return leaf64v3::kScratchDoubles; }

// Panel width for a leaf with nrhs right-hand sides: 32 while that still
// gives every SM a CTA (8192 right-hand sides: 32-wide 70 us per 16384 vs
// 16-wide 86, ncu launch list), narrower when the leaf would leave SMs idle
// (RECTRI_CU_LEAF_NC = 8 / 16 / 32 forces one).  Results do not depend on it.
int leaf3_width(long long nrhs, bool trsm) {
  const char* e = getenv("RECTRI_CU_LEAF_NC");
  const int forced = e ? atoi(e) : 0;
  if (forced == 8 || forced == 16 || forced == 32) return forced;
  if (nrhs >= 32LL * 148) return 32;  // at least one 32-wide CTA per SM (C3 panels: 8192)
  // TRSM leaves sit on the critical path (X1 -> GEMM -> X2): narrowest panels
  // up to 1024 right-hand sides; TRMM leaves overlap the other half's GEMM
  // (concurrent halves), where 16-wide ones do better (n = m = 1024: 72.5 vs
  // 84.8 us; TRSM 107.9 vs 117.9 the other way round).
  if (nrhs > (trsm ? 1024 : 512)) return 16;
  return 8;
}

void launch_leaf3_pack_all(const LeafParams<double>& base, const long long* d_r0, const int* d_n, int nleaves,
                           double* scratch, cudaStream_t s) {
  using namespace leaf64v3;
  dim3 grid(kMaxBlk * (kMaxBlk + 1) / 2, nleaves);
  launch_kernel(pack3_all_kernel, grid, 256, 0, s, base, d_r0, d_n, scratch, static_cast<long long>(kScratchDoubles));
  ++launch_counter();
}

void launch_leaf3_pack(const LeafParams<double>& p, double* dst, cudaStream_t s) {
  using namespace leaf64v3;
  const int nblk = (p.n + kRB - 1) / kRB;
  launch_kernel(pack3_kernel, nblk * (nblk + 1) / 2, 256, 0, s, p, dst);
  ++launch_counter();
}

void launch_leaf_f64_v3(const LeafParams<double>& p, double* scratch, cudaStream_t s, bool prepacked) {
  using namespace leaf64v3;
  const int nblk = (p.n + kRB - 1) / kRB;
  const bool zero = !p.trsm && p.alpha == 0.0;
  // TRMM with few right-hand sides: v5 (bitwise the same arithmetic, its
  // triangle in ascending row order) for direct base calls, and inside the
  // recursion with RECTRI_CU_LEAF >= 4 (whose packed triangles are ascending).
  const int w5 = p.trsm || zero ? 0 : leaf5_width(p.nrhs);
  const bool v5 = w5 > 0 && (prepacked ? p.pack_asc != 0 : (p.direct || leaf_trmm_asc()));
  if (!prepacked && !zero) {
    LeafParams<double> q = p;
    q.pack_asc = v5 ? 1 : 0;
    launch_kernel(pack3_kernel, nblk * (nblk + 1) / 2, 256, 0, s, q, scratch);
    ++launch_counter();
  }
  if (v5) {
    launch_leaf_f64_v5_trmm(p, scratch, w5, s);
    return;
  }
  const int nc = leaf3_width(p.nrhs, p.trsm != 0);
  const char* trv = getenv("RECTRI_CU_LEAF_TRACE");
  LeafParams<double> q = p;
  q.ring_check = leaf_ring_check_counter(&q.ring_plant);
  long long* d_tr = nullptr;
  const unsigned grid = static_cast<unsigned>(ceil_div(p.nrhs, nc));
  if (trv && atoi(trv) && !prepacked) {
    cudaMalloc(&d_tr, grid * 48 * sizeof(long long));
    cudaMemset(d_tr, 0, grid * 48 * sizeof(long long));
    q.trace = d_tr;
  }
  auto go = [&](auto kern, int width, int smem) {
    set_smem(kern, smem);
    launch_kernel(kern, static_cast<unsigned>(ceil_div(p.nrhs, width)), kThreads + 32, smem, s, q, scratch);
  };
  const char* wm = getenv("RECTRI_CU_LEAF_WM");
  if (q.ring_check) {
    if (nc == 32) go(leaf3_kernel<32, 1, true>, 32, smem_bytes<32>());
    else if (nc == 16) go(leaf3_kernel<16, 1, true>, 16, smem_bytes<16>());
    else go(leaf3_kernel<8, 1, true>, 8, smem_bytes<8>());
  } else if (nc == 32 && wm && atoi(wm) == 2) go(leaf3_kernel<32, 2>, 32, smem_bytes<32>());
  else if (nc == 32) go(leaf3_kernel<32>, 32, smem_bytes<32>());
  else if (nc == 16) go(leaf3_kernel<16>, 16, smem_bytes<16>());
  else go(leaf3_kernel<8>, 8, smem_bytes<8>());
  ++launch_counter();
  if (d_tr) {  // diagnostics: mean cycles from CTA start per phase, on stderr
    cudaStreamSynchronize(s);
    std::vector<long long> h(grid * 48);
    cudaMemcpy(h.data(), d_tr, h.size() * sizeof(long long), cudaMemcpyDeviceToHost);
    cudaFree(d_tr);
    double acc[48] = {0};
    for (unsigned b = 0; b < grid; ++b)
      for (int k = 1; k < 48; ++k)
        if (h[b * 48 + k]) acc[k] += static_cast<double>(h[b * 48 + k] - h[b * 48]);
    fprintf(stderr, "leaf3 trace (NC %d, %u CTAs, mean cycles from CTA start): panel %.0f |", nc, grid, acc[1] / grid);
    for (int bi = 0; bi < nblk; ++bi) fprintf(stderr, " %.0f", acc[2 + bi] / grid);
    fprintf(stderr, " | end %.0f\n", acc[41] / grid);
  }
}

namespace {
// Allocated by the first leaf_ring_check_read (outside any graph capture:
// the checked launches may be captured, an allocation there may not).
unsigned long long* g_ring_counter = nullptr;
}  // namespace

unsigned long long* leaf_ring_check_counter(int* plant) {
  const char* e = getenv("RECTRI_CU_RING_CHECK");
  const int mode = e ? atoi(e) : 0;
  *plant = mode == 2 ? 1 : 0;
  if (mode != 1 && mode != 2) return nullptr;
  if (!g_ring_counter) fprintf(stderr, "RECTRI_CU_RING_CHECK: call rectri_cu_debug_ring_check first; not checking\n");
  return g_ring_counter;
}

long long leaf_ring_check_read(bool reset) {
  cudaDeviceSynchronize();
  if (!g_ring_counter) {
    if (cudaMalloc(&g_ring_counter, sizeof(unsigned long long)) != cudaSuccess) {
      g_ring_counter = nullptr;
      return -1;
    }
    cudaMemset(g_ring_counter, 0, sizeof(unsigned long long));
    cudaDeviceSynchronize();
  }
  unsigned long long h = 0;
  cudaMemcpy(&h, g_ring_counter, sizeof(h), cudaMemcpyDeviceToHost);
  if (reset) {
    cudaMemset(g_ring_counter, 0, sizeof(h));
    cudaDeviceSynchronize();
  }
  return static_cast<long long>(h);
}

}  // namespace rectri_cu
