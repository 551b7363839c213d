// leaf32_v3.cu -- fp32 base (leaf) kernel v3: the fp64 v3 design
// (leaf64_v3.cu) on the FFMA pipe.
//
// trsm_base / trmm_base (src/base_kernels.cpp:94-177) on the Left form of a
// virtual lower factor L' in 32-row blocks:
//   * pack32_kernel writes, per leaf call, the blocks in consumption order as
//     [k][row] fp32 tiles (TRSM row I: L'_I0 .. L'_I,I-1, then -inv(L'_II);
//     TRMM rows descending: ..., then L'_II with its diagonal).  The inverse
//     is computed in fp64 by substitution (one thread per column) and rounded
//     once; masked / out-of-range entries are exact zeros by selection and
//     padding rows get an identity diagonal.
//   * leaf32_kernel: one CTA owns 32 right-hand sides (panel nb x 32 floats
//     in shared memory); a producer warp streams the packed blocks through an
//     8-deep cp.async.bulk ring (mbarrier full/empty); 8 compute warps each
//     own 4 rows x 1 right-hand side (lane) of the current 32x32 row block and
//     accumulate with packed FFMA2 (fma.rn.f32x2: two rows per instruction);
//     per 4 k-steps a lane reads its 4 right-hand-side values as one
//     ld.shared.v4 (column-major padded panel) and the 4 x 4 L' values as
//     four broadcast ld.shared.v4.
// Results agree with leaf.cu (v1, RECTRI_CU_LEAF=1) to rounding.
#include <cstdlib>

#include "common.cuh"
#include "launch.h"

namespace rectri_cu {
namespace leaf32v3 {

constexpr int kRB = 32;
constexpr int kBlk = kRB * kRB;  // floats per packed block
constexpr int kRing = 8;
// Panel and partial-result buffers are column-major per right-hand side
// ([c][r]) with padded strides, so a lane reads 4 consecutive rows of its
// column as one conflict-free ld.shared.v4 (bank = 4c + r mod 32).
constexpr int kPS = kLeafMax + 4;  // panel column stride (floats)
constexpr int kCS = kRB + 4;       // cbuf column stride
template <int NC>
constexpr int smem_bytes() { return (NC * kPS + NC * kCS + kRing * kBlk) * 4 + 2 * kRing * 8; }

__device__ __forceinline__ float lprime(const LeafParams<float>& p, int r, int j) {
  const int rr = p.reflected ? p.n - 1 - r : r;
  const int jj = p.reflected ? p.n - 1 - j : j;
  const i64 row = p.swapped ? jj : rr;
  const i64 col = p.swapped ? rr : jj;
  return p.A[row + col * p.lda];
}

__device__ __forceinline__ int seq_of(int I, int J, int nblk, bool asc) {
  if (asc) return I * (I + 1) / 2 + J;
  return (nblk * (nblk + 1) / 2 - (I + 1) * (I + 2) / 2) + J;
}

__device__ void pack32_block(const LeafParams<float>& p, float* __restrict__ P, const int b) {
  __shared__ double L[kRB][kRB + 1];
  const int nblk = (p.n + kRB - 1) / kRB;
  const bool trsm = p.trsm != 0;
  int I = 0;
  while ((I + 1) * (I + 2) / 2 <= b) ++I;
  const int J = b - I * (I + 1) / 2;
  const int r0 = I * kRB, j0 = J * kRB;
  float* dst = P + static_cast<size_t>(seq_of(I, J, nblk, trsm)) * kBlk;
  const int tid = threadIdx.x;
  if (J < I) {  // [k][r]
    for (int o = tid; o < kBlk; o += blockDim.x) {
      const int k = o >> 5, r = o & 31;
      dst[o] = r0 + r < p.n ? lprime(p, r0 + r, j0 + k) : 0.f;
    }
    return;
  }
  for (int o = tid; o < kBlk; o += blockDim.x) {
    const int r = o >> 5, k = o & 31;
    double v = 0.0;
    if (r0 + r >= p.n) v = r == k ? 1.0 : 0.0;
    else if (k < r) v = lprime(p, r0 + r, r0 + k);
    else if (k == r) v = p.unit ? 1.0 : lprime(p, r0 + r, r0 + r);
    L[r][k] = v;
  }
  __syncthreads();
  if (!trsm) {
    for (int o = tid; o < kBlk; o += blockDim.x) {
      const int k = o >> 5, r = o & 31;
      dst[o] = static_cast<float>(L[r][k]);
    }
    return;
  }
  if (tid < kRB) {  // -inv(L), column j = tid, in fp64 (column-oriented: leaf64_v3.cu)
    const int j = tid;
    double y[kRB];
#pragma unroll
    for (int r = 0; r < kRB; ++r) y[r] = r == j ? 1.0 : 0.0;
#pragma unroll
    for (int q = 0; q < kRB; ++q) {
      y[q] = q < j ? 0.0 : y[q] / L[q][q];
#pragma unroll
      for (int r = q + 1; r < kRB; ++r) y[r] = fma(-L[r][q], y[q], y[r]);
    }
#pragma unroll
    for (int r = 0; r < kRB; ++r) dst[j * kRB + r] = static_cast<float>(-y[r]);  // [k = j][r]
  }
}

__global__ void __launch_bounds__(256) pack32_kernel(const LeafParams<float> p, float* __restrict__ P) {
  pdl_wait();  // PDL: no-op unless launched programmatically (launch_kernel)
  pack32_block(p, P, blockIdx.x);
}

// Every leaf of one recursion (blockIdx.y = leaf k: order ns[k] at
// A(r0s[k], r0s[k])) into P + k * stride.
__global__ void __launch_bounds__(256) pack32_all_kernel(const LeafParams<float> base, const long long* __restrict__ r0s,
                                                         const int* __restrict__ ns, float* __restrict__ P,
                                                         long long stride) {
  pdl_wait();  // PDL: no-op unless launched programmatically (launch_kernel)
  const int k = blockIdx.y;
  LeafParams<float> p = base;
  p.n = ns[k];
  p.A = base.A + r0s[k] * (1 + base.lda);
  const int nblk = (p.n + kRB - 1) / kRB;
  if (static_cast<int>(blockIdx.x) >= nblk * (nblk + 1) / 2) return;
  pack32_block(p, P + static_cast<size_t>(k) * stride, blockIdx.x);
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

// NC right-hand sides per CTA (32, 16 or 8): 8 row groups x NC columns of
// compute threads as 8 row groups x NC/2 column pairs (NC / 8 warps) plus the
// producer warp; each thread keeps 4 rows x 2 right-hand sides (one A read
// feeds both columns) and the same k order for every NC, so the widths
// agree bit for bit.
// CK: the ring checker's instantiation (RECTRI_CU_RING_CHECK, as in leaf64_v3.cu).
template <int NC, bool CK = false>
__global__ void __launch_bounds__(4 * NC + 32, 4) leaf32_kernel(const LeafParams<float> p,
                                                                const float* __restrict__ P) {
  pdl_wait();  // PDL: no-op unless launched programmatically (launch_kernel)
  constexpr int kNC = NC;
  constexpr int kWarps = NC / 8;
  constexpr int kThreads = kWarps * 32;
  constexpr int kCP = NC / 2;  // column pairs
  extern __shared__ __align__(128) float smem32[];
  float* panel = smem32;                  // [c][r], stride kPS
  float* cbuf = panel + kNC * kPS;        // [c][r], stride kCS
  float* ring = cbuf + kNC * kCS;         // kRing blocks [k][r]
  const uint32_t full0 = smem_u32(ring + kRing * kBlk), empty0 = full0 + 8 * kRing;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n = p.n;
  const int nblk = (n + kRB - 1) / kRB;
  const int rows_p = nblk * kRB;
  const i64 c0 = static_cast<i64>(blockIdx.x) * kNC;
  const int ncols = static_cast<int>(min(static_cast<i64>(kNC), p.nrhs - c0));
  const bool trsm = p.trsm != 0;

  // Panel visitor (compute warps): Left -> each warp covers 4 rows x 8
  // right-hand sides; Right -> one row of 32 per warp.
  const i64 rstep = p.reflected ? -1 : 1;
  auto for_panel = [&](auto&& f) {
    if (!p.right) {
      const int rl = lane & 3, cl = lane >> 2;
#pragma unroll
      for (int cg = 0; cg < kNC / 8; ++cg) {
        const int c = 8 * cg + cl;
        const float* colp = p.B + (c0 + c) * p.ldb + (p.reflected ? n - 1 : 0);
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

  if (!trsm && p.alpha == 0.f) {  // base_kernels.cpp:143-150
    if (warp < kWarps)
      for_panel([&](int r, int c, const float* g) {
        if (r < n && c < ncols) *const_cast<float*>(g) = 0.f;
      });
    return;
  }
  const int nseq = nblk * (nblk + 1) / 2;
  if (tid == 0) {
    for (int q = 0; q < kRing; ++q) {
      mbar_init(full0 + 8 * q, 1);
      mbar_init(empty0 + 8 * q, kWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  }
  __syncthreads();
  if (warp == kWarps) {  // producer warp
    if (lane == 0)
      for (int q = 0; q < nseq; ++q) {
        const int slot = q % kRing;
        if (q >= kRing) mbar_wait(empty0 + 8 * slot, ((q / kRing) + 1) & 1);
        mbar_expect_tx(full0 + 8 * slot, kBlk * 4);
        bulk_g2s(smem_u32(ring + slot * kBlk), P + static_cast<size_t>(q) * kBlk, kBlk * 4, full0 + 8 * slot);
      }
    return;
  }
  for_panel([&](int r, int c, const float* g) {
    const bool ok = r < n && c < ncols;
    cp_async4(panel + c * kPS + r, ok ? g : p.B, ok ? 4 : 0);
  });
  cp_async_commit();
  cp_async_wait<0>();
  named_sync(1, kThreads);
  if (trsm && p.alpha != 1.f) {  // x = alpha * b (base_kernels.cpp:76-77)
    for_panel([&](int r, int c, const float*) { panel[c * kPS + r] *= p.alpha; });
    named_sync(1, kThreads);
  }

  // Thread (row group g, column pair q): rows 4g .. 4g+3 of the row block,
  // right-hand sides q and q + NC/2 (lanes: q fastest, so a warp's x reads
  // hit consecutive columns -- 8 distinct bank groups per 8 lanes).
  const int tq = warp * 32 + lane;
  const int rw = 4 * (tq / kCP), cc = tq % kCP;
  unsigned long long acc[2][2];  // [column][row pair]: (4g, 4g+1), (4g+2, 4g+3)
  int s = 0;
  const uint32_t dep0 = static_cast<uint32_t>(n) >> 16;  // 0 at run time (n <= 256), unknown to ptxas
  // acc[j] += block(s) * src_j (32 consecutive rows of column j)
  auto block_mma = [&](const float* src0, const float* src1) {
    const int slot = s % kRing;
    mbar_wait(full0 + 8 * slot, (s / kRing) & 1);
    const float* blk = ring + (CK && p.ring_plant ? (s + 1) % kRing : slot) * kBlk;
    unsigned bad = 0;
#pragma unroll
    for (int kb = 0; kb < kRB; kb += 4) {
      const float4 x0 = *reinterpret_cast<const float4*>(src0 + kb);
      const float4 x1 = *reinterpret_cast<const float4*>(src1 + kb);
      const float xs[2][4] = {{x0.x, x0.y, x0.z, x0.w}, {x1.x, x1.y, x1.z, x1.w}};
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const float4 a = *reinterpret_cast<const float4*>(blk + (kb + kk) * kRB + rw);  // broadcast
        if (CK) {  // RECTRI_CU_RING_CHECK: block s's packed values, bit for bit
          const float4 g = *reinterpret_cast<const float4*>(P + static_cast<size_t>(s) * kBlk + (kb + kk) * kRB + rw);
          bad += (__float_as_uint(a.x) != __float_as_uint(g.x)) + (__float_as_uint(a.y) != __float_as_uint(g.y)) +
                 (__float_as_uint(a.z) != __float_as_uint(g.z)) + (__float_as_uint(a.w) != __float_as_uint(g.w));
        }
        unsigned long long a01, a23;
        asm("mov.b64 %0, {%1, %2};" : "=l"(a01) : "f"(a.x), "f"(a.y));
        asm("mov.b64 %0, {%1, %2};" : "=l"(a23) : "f"(a.z), "f"(a.w));
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          unsigned long long xx;
          asm("mov.b64 %0, {%1, %1};" : "=l"(xx) : "f"(xs[j][kk]));
          asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc[j][0]) : "l"(a01), "l"(xx));
          asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc[j][1]) : "l"(a23), "l"(xx));
        }
      }
    }
    // release the slot once its fragment loads have landed: the arrive's
    // address depends on the accumulators every loaded A value fed
    // (slot_dep, common.cuh; FFMA2 latency only, no proxy-fence MEMBAR)
    const uint32_t dep = slot_dep(dep0, acc[0][0], acc[0][1]);
    if (CK && bad) atomicAdd(p.ring_check, static_cast<unsigned long long>(bad));
    __syncwarp();
    if (lane == 0) mbar_arrive(empty0 + 8 * slot + dep);
    ++s;
  };
  auto unpack = [&](int j, float (&v)[4]) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(v[0]), "=f"(v[1]) : "l"(acc[j][0]));
    asm("mov.b64 {%0, %1}, %2;" : "=f"(v[2]), "=f"(v[3]) : "l"(acc[j][1]));
  };
  auto pack = [&](int j, const float (&v)[4]) {
    asm("mov.b64 %0, {%1, %2};" : "=l"(acc[j][0]) : "f"(v[0]), "f"(v[1]));
    asm("mov.b64 %0, {%1, %2};" : "=l"(acc[j][1]) : "f"(v[2]), "f"(v[3]));
  };

  float* pcol[2] = {panel + cc * kPS, panel + (cc + kCP) * kPS};  // rows contiguous
  float* ccol[2] = {cbuf + cc * kCS, cbuf + (cc + kCP) * kCS};
  for (int bi = 0; bi < nblk; ++bi) {
    const int I = trsm ? bi : nblk - 1 - bi;
    const int r0 = I * kRB;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const float4 b4 = *reinterpret_cast<const float4*>(pcol[j] + r0 + rw);
      const float v[4] = {trsm ? -b4.x : 0.f, trsm ? -b4.y : 0.f, trsm ? -b4.z : 0.f, trsm ? -b4.w : 0.f};
      pack(j, v);
    }
    for (int J = 0; J < I; ++J) block_mma(pcol[0] + J * kRB, pcol[1] + J * kRB);
    if (trsm) {
      // acc = -(b_I - sum L'X); X_I = (-inv(L'_II)) * acc
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        float v[4];
        unpack(j, v);
        *reinterpret_cast<float4*>(ccol[j] + rw) = make_float4(v[0], v[1], v[2], v[3]);
        acc[j][0] = acc[j][1] = 0ull;
      }
      named_sync(1, kThreads);
      block_mma(ccol[0], ccol[1]);
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        float v[4];
        unpack(j, v);
        *reinterpret_cast<float4*>(pcol[j] + r0 + rw) = make_float4(v[0], v[1], v[2], v[3]);
      }
      named_sync(1, kThreads);  // X_I visible; cbuf free
    } else {
      // + L'_II * b_I, then X_I straight to global memory: later (lower)
      // row blocks read only panel blocks J < I, so b_I stays intact in
      // shared memory and no barrier is needed per row block
      block_mma(pcol[0] + I * kRB, pcol[1] + I * kRB);
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int c = cc + j * kCP;
        if (c >= ncols) continue;
        float v[4];
        unpack(j, v);
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int r = r0 + rw + t;
          if (r >= n) break;
          const i64 sr = p.reflected ? n - 1 - r : r;
          float* gp = p.right ? p.B + sr * p.ldb + c0 + c : p.B + (c0 + c) * p.ldb + sr;
          *gp = p.alpha * v[t];
        }
      }
    }
  }
  if (!trsm) return;
  named_sync(1, kThreads);
  for_panel([&](int r, int c, const float* g) {
    if (r < n && c < ncols) *const_cast<float*>(g) = panel[c * kPS + r];
  });
}

}  // namespace leaf32v3

void launch_leaf32_pack_all(const LeafParams<float>& base, const long long* d_r0, const int* d_n, int nleaves,
                            float* scratch, long long stride, cudaStream_t s) {
  using namespace leaf32v3;
  constexpr int kMaxBlk = kLeafMax / kRB;
  dim3 grid(kMaxBlk * (kMaxBlk + 1) / 2, nleaves);
  launch_kernel(pack32_all_kernel, grid, 256, 0, s, base, d_r0, d_n, scratch, stride);
  ++launch_counter();
}

void launch_leaf_f32_v3(const LeafParams<float>& p, float* scratch, cudaStream_t s, bool prepacked) {
  using namespace leaf32v3;
  const int nblk = (p.n + kRB - 1) / kRB;
  if (!prepacked && (p.trsm || p.alpha != 0.f)) {
    launch_kernel(pack32_kernel, nblk * (nblk + 1) / 2, 256, 0, s, p, scratch);
    ++launch_counter();
  }
  auto go = [&](auto kern, int width, int smem) {
    set_smem(kern, smem);
    launch_kernel(kern, static_cast<unsigned>(ceil_div(p.nrhs, width)), 4 * width + 32, smem, s, p, scratch);
  };
  const int nc = leaf3_width(p.nrhs, p.trsm != 0);
  LeafParams<float> q = p;
  q.ring_check = leaf_ring_check_counter(&q.ring_plant);
  if (q.ring_check) {
    auto gc = [&](auto kern, int width, int smem) {
      set_smem(kern, smem);
      launch_kernel(kern, static_cast<unsigned>(ceil_div(p.nrhs, width)), 4 * width + 32, smem, s, q, scratch);
    };
    if (nc == 32) gc(leaf32_kernel<32, true>, 32, smem_bytes<32>());
    else if (nc == 16) gc(leaf32_kernel<16, true>, 16, smem_bytes<16>());
    else gc(leaf32_kernel<8, true>, 8, smem_bytes<8>());
  } else if (nc == 32) go(leaf32_kernel<32>, 32, smem_bytes<32>());
  else if (nc == 16) go(leaf32_kernel<16>, 16, smem_bytes<16>());
  else go(leaf32_kernel<8>, 8, smem_bytes<8>());
  ++launch_counter();
}

}  // namespace rectri_cu
