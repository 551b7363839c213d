// leaf64_v4.cu -- fp64 base (leaf) kernel v4: column-owning warps.
//
// trsm_base / trmm_base (src/base_kernels.cpp:94-177) on the Left form of a
// virtual lower factor L', with the SAME per-element
// arithmetic as v3 (leaf64_v3.cu): 32-row blocks, the packed triangle of
// pack3_kernel (diagonal blocks as -inv(L'_II) for TRSM, L'_II for TRMM),
// DMMA.8x8x4 products whose k-steps alternate between two partial sums added
// once per row block, TRSM initial value -alpha*b_I.  So v4 and v3 agree bit
// for bit (tests/test_gpu_leaf.py), and the choice between them -- by the
// number of right-hand sides -- never changes a result.
//
// What changes is the work distribution.  Right-hand sides are independent,
// so each compute warp owns CW whole columns of the CTA's NC-wide panel and
// walks all row blocks of them by itself:
//   * no CTA-wide barrier anywhere in the solve (v3: two named barriers per
//     row block, every warp waiting for the slowest) -- a warp only
//     __syncwarp()s between writing a row block and reading it back;
//   * the panel arrives row block by row block (one cp.async group each) and
//     row block I starts as soon as its own rows are in, so the HBM load of
//     the panel overlaps the first blocks' DMMAs;
//   * each X_I goes to global memory from registers as soon as it is final
//     (TRMM keeps the panel pristine -- its row blocks are independent, so
//     they run ascending like TRSM's and the panel load pipelines for both);
//   * per k-step a warp reads 4 A fragments (32 rows) and CW/8 B fragments
//     for 4*CW/8 DMMAs (v3: 1 A + E B for E DMMAs, 8 rows per warp).
// The packed blocks stream from L2 through a RING-deep bulk-copy ring shared
// by the W = NC/CW compute warps (producer warp, full/empty mbarriers; a slot
// is released only after the DMMAs that consumed it were issued).
#include <cstdlib>

#include "common.cuh"
#include "launch.h"

namespace rectri_cu {
namespace leaf64v4 {

constexpr int kRB = 32;
constexpr int kBlk = kRB * kRB;

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
// cp.async.wait_group with a run-time count (at most 7 groups pending).
__device__ __forceinline__ void cp_async_wait_dyn(int pending) {
  switch (pending) {
    case 0: cp_async_wait<0>(); break;
    case 1: cp_async_wait<1>(); break;
    case 2: cp_async_wait<2>(); break;
    case 3: cp_async_wait<3>(); break;
    case 4: cp_async_wait<4>(); break;
    case 5: cp_async_wait<5>(); break;
    case 6: cp_async_wait<6>(); break;
    default: cp_async_wait<7>(); break;
  }
}

template <int NC, int CW, int RING>
constexpr int smem_bytes() { return (kLeafMax * NC + RING * kBlk) * 8 + 2 * RING * 8; }

template <int NC, int CW, int RING, int MINB>
__global__ void __launch_bounds__((NC / CW) * 32 + 32, MINB) leaf4_kernel(const LeafParams<double> p,
                                                                       const double* __restrict__ P) {
  constexpr int W = NC / CW;  // compute warps
  constexpr int E = CW / 8;   // 8-column tiles per warp
  static_assert(CW % 8 == 0 && NC % CW == 0 && (NC >= 16 || NC == 8), "panel geometry");
  extern __shared__ __align__(128) double smem4[];
  double* panel = smem4;                  // kLeafMax x NC (swizzled rows)
  double* ring = smem4 + kLeafMax * NC;   // RING packed 32x32 blocks
  const uint32_t full0 = smem_u32(ring + RING * kBlk), empty0 = full0 + 8 * RING;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n = p.n;
  const int nblk = (n + kRB - 1) / kRB;
  const i64 c0 = static_cast<i64>(blockIdx.x) * NC;
  const int ncols = static_cast<int>(min(static_cast<i64>(NC), p.nrhs - c0));
  const bool trsm = p.trsm != 0;
  const int nseq = nblk * (nblk + 1) / 2;

  if (tid == 0) {
    for (int q = 0; q < RING; ++q) {
      mbar_init(full0 + 8 * q, 1);
      mbar_init(empty0 + 8 * q, W);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  }
  __syncthreads();
  if (warp == W) {  // producer warp: the packed blocks, ascending rows, through the ring
    if (lane == 0)
      for (int q = 0; q < nseq; ++q) {
        const int slot = q % RING;
        if (q >= RING) mbar_wait(empty0 + 8 * slot, ((q / RING) + 1) & 1);
        mbar_expect_tx(full0 + 8 * slot, kBlk * 8);
        bulk_g2s(smem_u32(ring + slot * kBlk), P + static_cast<size_t>(q) * kBlk, kBlk * 8, full0 + 8 * slot);
      }
    return;
  }

  // This warp's columns [cw0, cw0 + CW) of the panel: every row block is one
  // cp.async group, issued up front.
  const int cw0 = warp * CW;
  auto gaddr = [&](int r, int c) -> const double* {  // panel element (r, c) in B
    const i64 sr = p.reflected ? n - 1 - r : r;
    return p.right ? p.B + sr * p.ldb + c0 + c : p.B + (c0 + c) * p.ldb + sr;
  };
  for (int I = 0; I < nblk; ++I) {
    if (!p.right) {
      const int rl = lane & 3, cl = lane >> 2;  // 4 rows x 8 columns per instruction
#pragma unroll
      for (int cg = 0; cg < E; ++cg) {
        const int c = cw0 + 8 * cg + cl;
#pragma unroll
        for (int rt = 0; rt < kRB / 4; ++rt) {
          const int r = I * kRB + 4 * rt + rl;
          const bool ok = r < n && c < ncols;
          cp_async8(panel + pidx<NC>(r, c), ok ? gaddr(r, c) : p.B, ok ? 8 : 0);
        }
      }
    } else {
      constexpr int RPP = 32 / CW;  // rows per pass (CW contiguous columns)
#pragma unroll
      for (int rr = 0; rr < kRB; rr += RPP) {
        const int r = I * kRB + rr + lane / CW, c = cw0 + lane % CW;
        const bool ok = r < n && c < ncols;
        cp_async8(panel + pidx<NC>(r, c), ok ? gaddr(r, c) : p.B, ok ? 8 : 0);
      }
    }
    cp_async_commit();
  }

  const int g = lane >> 2, t = lane & 3;
  const uint32_t panel_u32 = smem_u32(panel);
  // B fragment of k-step kk of row block J, column tile e: panel row 32J + 4kk + t
  // (row & 3 == t, so the swizzle is that of row t), column cw0 + 8e + g.
  uint32_t b_base[E];
#pragma unroll
  for (int e = 0; e < E; ++e) b_base[e] = panel_u32 + 8u * static_cast<uint32_t>(pidx<NC>(t, cw0 + 8 * e + g));
  constexpr uint32_t kRowBytes = NC * 8;

  double c[2][4][E][2];
  int s = 0;
  auto block_mma = [&](int Jrow) {  // c += (next packed block) * panel rows [32 Jrow, 32 Jrow + 32)
    const int slot = s % RING;
    mbar_wait(full0 + 8 * slot, (s / RING) & 1);
    const uint32_t as = smem_u32(ring + slot * kBlk) + 8u * lane;
    double a[4][8];
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)
        asm volatile("ld.shared.f64 %0, [%1];" : "=d"(a[mt][kk]) : "r"(as + (mt * 8 + kk) * 256));
    double bv[8][E];
#pragma unroll
    for (int kk = 0; kk < 8; ++kk)
#pragma unroll
      for (int e = 0; e < E; ++e)
        asm volatile("ld.shared.f64 %0, [%1];"
                     : "=d"(bv[kk][e])
                     : "r"(b_base[e] + (static_cast<uint32_t>(Jrow * kRB + 4 * kk)) * kRowBytes));
#pragma unroll
    for (int kk = 0; kk < 8; ++kk)
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int e = 0; e < E; ++e) dmma884(c[kk & 1][mt][e][0], c[kk & 1][mt][e][1], a[mt][kk], bv[kk][e]);
    __syncwarp();
    if (lane == 0) {
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // generic reads before the async refill
      mbar_arrive(empty0 + 8 * slot);
    }
    ++s;
  };
  // element (mt, e, h) of this lane's accumulators: row 8 mt + g, column cw0 + 8 e + 2 t + h of the row block
  auto for_c = [&](auto&& f) {
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int e = 0; e < E; ++e) f(mt, e);
  };
  auto store_x = [&](int r, int cc, double x) {
    if (r < n && cc < ncols) *const_cast<double*>(gaddr(r, cc)) = x;
  };

  for (int I = 0; I < nblk; ++I) {
    cp_async_wait_dyn(nblk - 1 - I);  // this lane's copies of row blocks 0..I have landed
    __syncwarp();                     // ... and every lane's
    const int r0 = I * kRB;
    if (trsm) {
      for_c([&](int mt, int e) {
        const int r = r0 + 8 * mt + g, cc = cw0 + 8 * e + 2 * t;
        const double2 b = *reinterpret_cast<const double2*>(panel + pidx<NC>(r, cc));
        c[0][mt][e][0] = p.alpha != 1.0 ? -(p.alpha * b.x) : -b.x;
        c[0][mt][e][1] = p.alpha != 1.0 ? -(p.alpha * b.y) : -b.y;
        c[1][mt][e][0] = c[1][mt][e][1] = 0.0;
      });
    } else {
      for_c([&](int mt, int e) { c[0][mt][e][0] = c[0][mt][e][1] = c[1][mt][e][0] = c[1][mt][e][1] = 0.0; });
    }
    for (int J = 0; J < I; ++J) block_mma(J);
    if (trsm) {
      // c = -(b_I - sum L'X) into the panel rows of block I; X_I = (-inv(L'_II)) * c
      for_c([&](int mt, int e) {
        const int r = r0 + 8 * mt + g, cc = cw0 + 8 * e + 2 * t;
        *reinterpret_cast<double2*>(panel + pidx<NC>(r, cc)) =
            make_double2(c[0][mt][e][0] + c[1][mt][e][0], c[0][mt][e][1] + c[1][mt][e][1]);
        c[0][mt][e][0] = c[0][mt][e][1] = c[1][mt][e][0] = c[1][mt][e][1] = 0.0;
      });
      __syncwarp();
      block_mma(I);
      __syncwarp();  // every lane has read c before X_I replaces it
      for_c([&](int mt, int e) {
        const int r = r0 + 8 * mt + g, cc = cw0 + 8 * e + 2 * t;
        const double x0 = c[0][mt][e][0] + c[1][mt][e][0], x1 = c[0][mt][e][1] + c[1][mt][e][1];
        *reinterpret_cast<double2*>(panel + pidx<NC>(r, cc)) = make_double2(x0, x1);
        store_x(r, cc, x0);
        store_x(r, cc + 1, x1);
      });
    } else {
      block_mma(I);  // c += L'_II * b_I (the panel stays pristine: X goes straight out)
      for_c([&](int mt, int e) {
        const int r = r0 + 8 * mt + g, cc = cw0 + 8 * e + 2 * t;
        store_x(r, cc, p.alpha * (c[0][mt][e][0] + c[1][mt][e][0]));
        store_x(r, cc + 1, p.alpha * (c[0][mt][e][1] + c[1][mt][e][1]));
      });
    }
  }
}

template <int NC, int CW, int RING, int MINB>
void go(const LeafParams<double>& p, const double* P, cudaStream_t s) {
  auto kern = leaf4_kernel<NC, CW, RING, MINB>;
  constexpr int smem = smem_bytes<NC, CW, RING>();
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  kern<<<static_cast<unsigned>(ceil_div(p.nrhs, NC)), (NC / CW) * 32 + 32, smem, s>>>(p, P);
  ++launch_counter();
}

int config_env() {
  const char* e = getenv("RECTRI_CU_LEAF4_CFG");
  return e ? atoi(e) : 0;
}

}  // namespace leaf64v4

// v4 is used for leaves with at least this many right-hand sides
// (RECTRI_CU_LEAF4_MIN, default 2048; v3 below, bitwise the same results).
long long leaf4_min_rhs() {
  const char* e = getenv("RECTRI_CU_LEAF4_MIN");
  return e ? atoll(e) : 2048;
}

bool leaf4_use(long long nrhs) { return leaf_version() >= 4 && nrhs >= leaf4_min_rhs(); }

void launch_leaf_f64_v4(const LeafParams<double>& p, const double* packed, cudaStream_t s) {
  using namespace leaf64v4;
  switch (config_env()) {
    case 1: go<64, 16, 8, 1>(p, packed, s); break;
    case 2: go<32, 8, 5, 2>(p, packed, s); break;
    case 3: go<64, 8, 8, 1>(p, packed, s); break;
    case 4: go<32, 16, 5, 2>(p, packed, s); break;
    default: go<32, 8, 5, 2>(p, packed, s); break;
  }
}

}  // namespace rectri_cu
