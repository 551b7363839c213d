// common.cuh -- shared device helpers for the sm_100a TRMM/TRSM kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

namespace rectri_cu {

using i64 = int64_t;

// ---------------------------------------------------------------------------
// cp.async (LDGSTS).  `src_bytes` < cp size zero-fills the remainder, which is
// how every out-of-range element of a tile becomes an exact 0 (never a
// multiply-by-mask: NaN must not leak from outside a view).
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(smem)),
               "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, int src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(smem)),
               "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem, int src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(smem_u32(smem)),
               "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// ---------------------------------------------------------------------------
// Releasing a ring slot that bulk copies / TMA refill.  ptxas schedules an
// mbarrier.arrive by its register inputs only, so it may issue the arrive
// while shared loads of the slot are still in flight (SYNCS.ARRIVE does not
// wait on the load scoreboard); the producer can then refill the slot under
// those loads.  Making the arrive's address depend on the loaded values
// forces the wait: slot_dep() folds bits of the fragments into a value that
// is zero at run time (`zero` comes from a kernel parameter ptxas cannot
// see, e.g. K >> 40), and the arrive goes to bar + slot_dep(...).  Shared
// loads of a warp complete in order (the DEPBAR.LE counting ptxas itself
// relies on), so depending on the last loads of the slot covers all of them.
// This replaces fence.proxy.async before the arrive, which compiles to a
// MEMBAR.ALL.CTA that also waits for the thread's outstanding global stores.
__device__ __forceinline__ uint32_t dep_bits(double v) { return static_cast<uint32_t>(__double2hiint(v)); }
__device__ __forceinline__ uint32_t dep_bits(float v) { return __float_as_uint(v); }
__device__ __forceinline__ uint32_t dep_bits(unsigned long long v) { return static_cast<uint32_t>(v); }
template <typename... V>
__device__ __forceinline__ uint32_t slot_dep(uint32_t zero, V... v) {
  return (0u | ... | dep_bits(v)) & zero;
}

// ---------------------------------------------------------------------------
// fp64 tensor-core MMA: D(8x8) += A(8x4, row) * B(4x8, col), lowered to SASS
// DMMA.8x8x4 on sm_100a (tcgen05 has no f64 kind).  Fragment ownership
// (lane = 4*g + t): a = A[g][t], b = B[t][g], c{0,1} = C[g][2t + {0,1}].
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// ---------------------------------------------------------------------------
// Swizzled shared-memory tile addressing for 8-byte elements.  A tile row of
// `width` doubles (width % 16 == 0) is split into 16-byte chunks; the chunk
// index is XORed with 2*(row & 3).  With the m8n8k4 fragment pattern (8
// consecutive outer indices x 4 consecutive k) every half-warp then touches 16
// distinct 8-byte banks whether the tile is stored k-major or outer-major, and
// 16-byte cp.async chunks stay intact.
__device__ __forceinline__ int swz64(int row, int col, int width) {
  return row * width + ((((col >> 1) ^ ((row & 3) << 1))) << 1) + (col & 1);
}

__host__ __device__ __forceinline__ i64 ceil_div(i64 a, i64 b) { return (a + b - 1) / b; }

// Opts a kernel into `bytes` of dynamic shared memory and asks for the
// largest shared-memory carveout of the SM's unified L1/shared storage, so
// as many CTAs fit per SM as their shared memory allows (without it the
// driver may pick a smaller carveout: ncu showed the 70 KB DGEMM CTA limited
// to 2 per SM).  RECTRI_CU_SMEM_CARVEOUT overrides the percentage (-1: leave
// the driver's choice).
int smem_carveout_pct();
template <typename Kern>
inline void set_smem(Kern kern, int bytes) {
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  const int pct = smem_carveout_pct();
  if (pct >= 0) cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
}

// ---------------------------------------------------------------------------
// Programmatic dependent launch (PDL).  The recursion is a chain of short
// kernels per right-hand-side stream (leaf -> update -> leaf ...).  Launched
// with cudaLaunchAttributeProgrammaticStreamSerialization (launch_kernel), a
// kernel may be set up before its predecessor has fully retired and waits in
// griddepcontrol.wait until the predecessor has completed and its memory is
// visible, so part of the launch latency leaves the critical path while the
// ordering stays the stream's.  Every kernel launched through launch_kernel
// calls pdl_wait() before touching global memory; without the
// attribute it is a no-op.  No kernel triggers its dependents early
// (griddepcontrol.launch_dependents): measured, an early trigger (at kernel
// start, or after the main loop) parks the next kernel's CTAs on SMs the
// other right-hand-side stream needs -- TRSM n = 1024 91 -> 101-121 us --
// while the implicit trigger at completion gains 1-2 % on small problems
// (TRSM n = 1024 93.1 -> 91.3 us, fp32 TRSM n = 4096 1910 -> 1881 us;
// profiles/r02_pdl.txt).  RECTRI_CU_PDL=0 launches without the attribute.
__device__ __forceinline__ void pdl_wait() {
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
}
bool pdl_enabled();
template <typename... KArgs, typename... Args>
inline cudaError_t launch_kernel(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                                 Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

}  // namespace rectri_cu
