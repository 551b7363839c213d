// leaf64_v5.cu -- fp64 TRMM base (leaf) kernel for few right-hand sides:
// row-block-owning warps.
//
// trmm_base (src/base_kernels.cpp:94-156) on the Left form of a virtual
// lower factor L': X_I = alpha * sum_{J <= I} L'_IJ b_J.
// Every row block of a TRMM leaf is independent of the others (the result
// goes to global memory, the panel stays pristine in shared memory), so the
// leaf need not run its 8 row blocks one after the other: compute warp w
// owns the row blocks {w, nblk-1-w} of all NC columns, and the longest chain
// of a CTA is nblk + 1 packed blocks instead of the nblk (nblk + 1) / 2 of
// v3 (TRMM n = 256: 9 blocks instead of 36).  That is what matters
// when the leaf has few right-hand sides (a 256 x 2048 leaf fills 128 CTAs)
// and the GPU waits on the chain rather than on the tensor pipe.
//
// Arithmetic: per element exactly v3's (leaf64_v3.cu) -- J ascending with the
// diagonal block L'_II last, DMMA.8x8x4 k-steps alternating between two
// partial sums kk % 2, X = alpha * (c0 + c1) -- so v5 and v3 agree bit for bit and
// the launcher may pick either by right-hand-side count.
//
// Where it is used: direct trmm_base calls (a 256 x 2048 leaf: 13.6 us vs
// v3's 26 us, ncu); inside the recursion only with RECTRI_CU_LEAF=4, because
// there the leaf runs beside the other right-hand-side stream's GEMMs and
// v3's smaller shared-memory footprint measured faster (fp64 TRMM n = 4096:
// 2202 us v3, 2226-2248 us v5; profiles/r02_leaf_v5.txt).
//
// Blocks stream from the packed triangle (pack3_kernel, ascending row order:
// row I's blocks are contiguous) through a ring of STEPS: step s holds, for
// each compute warp, the s-th block of its sequence (row w's blocks, then
// row nblk-1-w's), filled by a producer warp with bulk copies (full
// mbarrier: the bytes of the step; empty mbarrier: one arrival per compute
// warp).
#include <cstdlib>

#include "common.cuh"
#include "launch.h"

namespace rectri_cu {
namespace leaf64v5 {

constexpr int kRB = 32;
constexpr int kBlk = kRB * kRB;
constexpr int kCW = 4;  // compute warps: row pairs of an order-256 leaf

template <int NC>
__device__ __forceinline__ int pidx(int r, int c) {
  if constexpr (NC >= 16) return swz64(r, c, NC);
  else return r * NC + c;
}

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

// Block (I, J) of warp w's sequence at step s, or false when w has finished.
__device__ __forceinline__ bool step_block(int w, int s, int nblk, int& I, int& J) {
  const int r1 = w, r2 = nblk - 1 - w;
  if (r1 > r2) return false;  // no row for this warp
  if (s <= r1) {
    I = r1;
    J = s;
    return true;
  }
  if (r2 == r1) return false;
  const int s2 = s - (r1 + 1);
  if (s2 > r2) return false;
  I = r2;
  J = s2;
  return true;
}

template <int NC, int STAGES>
constexpr int smem_bytes() { return (kLeafMax * NC + STAGES * kCW * kBlk) * 8 + 2 * STAGES * 8; }

template <int NC, int STAGES, int MINB>
__global__ void __launch_bounds__(kCW * 32 + 32, MINB) leaf5_trmm_kernel(const LeafParams<double> p,
                                                                      const double* __restrict__ P) {
  pdl_wait();  // PDL: no-op unless launched programmatically (launch_kernel)
  constexpr int E = NC / 8;  // 8-column tiles per warp
  extern __shared__ __align__(128) double smem5[];
  double* panel = smem5;                   // kLeafMax x NC (swizzled rows)
  double* ring = smem5 + kLeafMax * NC;    // STAGES steps x kCW blocks
  const uint32_t full0 = smem_u32(ring + STAGES * kCW * kBlk), empty0 = full0 + 8 * STAGES;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n = p.n;
  const int nblk = (n + kRB - 1) / kRB;
  const int rows_p = nblk * kRB;
  const i64 c0 = static_cast<i64>(blockIdx.x) * NC;
  const int ncols = static_cast<int>(min(static_cast<i64>(NC), p.nrhs - c0));
  const int nsteps = nblk == 1 ? 1 : nblk + 1;

  if (tid == 0) {
    for (int q = 0; q < STAGES; ++q) {
      mbar_init(full0 + 8 * q, 1);
      mbar_init(empty0 + 8 * q, kCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  }
  __syncthreads();
  if (warp == kCW) {  // producer warp
    if (lane == 0)
      for (int s = 0; s < nsteps; ++s) {
        const int slot = s % STAGES;
        if (s >= STAGES) mbar_wait(empty0 + 8 * slot, ((s / STAGES) + 1) & 1);
        uint32_t bytes = 0;
        int IJ[kCW][2];
        bool has[kCW];
        for (int w = 0; w < kCW; ++w) {
          has[w] = step_block(w, s, nblk, IJ[w][0], IJ[w][1]);
          if (has[w]) bytes += kBlk * 8;
        }
        mbar_expect_tx(full0 + 8 * slot, bytes);  // bytes == 0 completes the phase at once
        for (int w = 0; w < kCW; ++w)
          if (has[w])
            bulk_g2s(smem_u32(ring + (slot * kCW + w) * kBlk),
                     P + static_cast<size_t>(IJ[w][0] * (IJ[w][0] + 1) / 2 + IJ[w][1]) * kBlk, kBlk * 8,
                     full0 + 8 * slot);
      }
    return;
  }

  auto gaddr = [&](int r, int c) -> double* {  // panel element (r, c) in B
    const i64 sr = p.reflected ? n - 1 - r : r;
    return p.right ? p.B + sr * p.ldb + c0 + c : p.B + (c0 + c) * p.ldb + sr;
  };
  // The whole panel, cooperatively (every warp reads rows of other warps).
  if (!p.right) {
    const int rl = lane & 3, cl = lane >> 2;  // 4 rows x 8 columns per instruction
    for (int cg = 0; cg < E; ++cg) {
      const int c = 8 * cg + cl;
      for (int rt = warp; rt < rows_p / 4; rt += kCW) {
        const int r = 4 * rt + rl;
        const bool ok = r < n && c < ncols;
        cp_async8(panel + pidx<NC>(r, c), ok ? gaddr(r, c) : p.B, ok ? 8 : 0);
      }
    }
  } else {
    constexpr int RPP = 32 / NC >= 1 ? 32 / NC : 1;  // rows per pass
    constexpr int CPP = NC < 32 ? NC : 32;
    for (int cb = 0; cb < NC; cb += CPP)
      for (int r = warp * RPP + lane / CPP; r < rows_p; r += kCW * RPP) {
        const int c = cb + lane % CPP;
        const bool ok = r < n && c < ncols;
        cp_async8(panel + pidx<NC>(r, c), ok ? gaddr(r, c) : p.B, ok ? 8 : 0);
      }
  }
  cp_async_commit();
  cp_async_wait<0>();
  named_sync(1, kCW * 32);

  const int g = lane >> 2, t = lane & 3;
  const uint32_t panel_u32 = smem_u32(panel);
  uint32_t b_base[E];
#pragma unroll
  for (int e = 0; e < E; ++e) b_base[e] = panel_u32 + 8u * static_cast<uint32_t>(pidx<NC>(t, 8 * e + g));
  constexpr uint32_t kRowBytes = NC * 8;

  constexpr int kParts = 2;  // as leaf64_v3.cu
  double c[kParts][4][E][2];
  auto zero_c = [&]() {
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int e = 0; e < E; ++e)
#pragma unroll
        for (int q = 0; q < kParts; ++q) c[q][mt][e][0] = c[q][mt][e][1] = 0.0;
  };
  zero_c();
  const uint32_t dep0 = static_cast<uint32_t>(n) >> 16;  // 0 at run time (n <= 256), unknown to ptxas
  for (int s = 0; s < nsteps; ++s) {
    const int slot = s % STAGES;
    int I = 0, J = 0;
    const bool has = step_block(warp, s, nblk, I, J);
    mbar_wait(full0 + 8 * slot, (s / STAGES) & 1);
    if (has) {
      const uint32_t as = smem_u32(ring + (slot * kCW + warp) * kBlk) + 8u * lane;
      const uint32_t bs = static_cast<uint32_t>(J * kRB) * kRowBytes;
      double a[2][4], bv[2][E];
      auto load = [&](int buf, int kk) {
#pragma unroll
        for (int mt = 0; mt < 4; ++mt)
          asm volatile("ld.shared.f64 %0, [%1];" : "=d"(a[buf][mt]) : "r"(as + (mt * 8 + kk) * 256));
#pragma unroll
        for (int e = 0; e < E; ++e)
          asm volatile("ld.shared.f64 %0, [%1];" : "=d"(bv[buf][e]) : "r"(b_base[e] + bs + 4u * kk * kRowBytes));
      };
      load(0, 0);
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        if (kk < 7) load((kk + 1) & 1, kk + 1);
#pragma unroll
        for (int mt = 0; mt < 4; ++mt)
#pragma unroll
          for (int e = 0; e < E; ++e)
            dmma884(c[kk % kParts][mt][e][0], c[kk % kParts][mt][e][1], a[kk & 1][mt], bv[kk & 1][e]);
      }
    }
    // release the slot once its fragment loads have landed: the arrive's
    // address depends on accumulators that every A fragment of the block fed
    // (slot_dep, common.cuh)
    uint32_t dep = 0;
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) dep |= slot_dep(dep0, c[0][mt][0][0], c[1][mt][0][0]);
    __syncwarp();
    if (lane == 0) mbar_arrive(empty0 + 8 * slot + dep);
    if (has && J == I) {  // row block I complete: X_I = alpha * (c0 + c1) straight to global
      const int r0 = I * kRB;
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int e = 0; e < E; ++e)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int r = r0 + 8 * mt + g, cc = 8 * e + 2 * t + h;
            if (r < n && cc < ncols)
              *gaddr(r, cc) = p.alpha * (c[0][mt][e][h] + c[1][mt][e][h]);
          }
      zero_c();
    }
  }
}

template <int NC, int STAGES, int MINB>
void go(const LeafParams<double>& p, const double* P, cudaStream_t s) {
  auto kern = leaf5_trmm_kernel<NC, STAGES, MINB>;
  constexpr int smem = smem_bytes<NC, STAGES>();
  set_smem(kern, smem);
  launch_kernel(kern, static_cast<unsigned>(ceil_div(p.nrhs, NC)), kCW * 32 + 32, smem, s, p, P);
  ++launch_counter();
}

}  // namespace leaf64v5

// Panel width of the v5 TRMM leaf for nrhs right-hand sides, 0 = not v5
// (RECTRI_CU_LEAF5_NC forces 8 / 16 / 32; RECTRI_CU_LEAF5_MAX: the largest
// nrhs it is used for, default 4096).
int leaf5_width(long long nrhs) {
  const char* mx = getenv("RECTRI_CU_LEAF5_MAX");
  const long long maxr = mx ? atoll(mx) : 4096;
  if (nrhs > maxr) return 0;
  const char* e = getenv("RECTRI_CU_LEAF5_NC");
  const int forced = e ? atoi(e) : 0;
  if (forced == 8 || forced == 16 || forced == 32) return forced;
  return nrhs <= 1024 ? 8 : 16;
}

void launch_leaf_f64_v5_trmm(const LeafParams<double>& p, const double* packed, int width, cudaStream_t s) {
  using namespace leaf64v5;
  if (width == 8) go<8, 3, 2>(p, packed, s);
  else if (width == 16) go<16, 3, 1>(p, packed, s);
  else go<32, 2, 1>(p, packed, s);
}

}  // namespace rectri_cu
