// sgemm_tf32x3.cu -- fp32 GEMM update on the 5th-generation tensor cores
// (tcgen05.mma kind::tf32, accumulators in TMEM) with the 3xTF32 split.
//
// An opt-in fp32 variant (RECTRI_CU_FP32_TF32X3 / backend flag), reported
// separately from the default exact-FFMA path (gemm_f32.cu) under its own
// tolerance, as the north star allows.  Each fp32 operand x is split into
// hi = x with the low 13 mantissa bits cleared (exactly a TF32 value) and
// lo = x - hi (exact in fp32; its own TF32 truncation is the method's
// ~2^-22 relative error), and op(A) op(B) is accumulated in fp32 as
// A_lo B_hi + A_hi B_lo + A_hi B_hi (small terms first; A_lo B_lo dropped).
//
// Structure: a split kernel writes hi/lo copies of op(A)'s and B's views
// (packed, column-major); the GEMM kernel then runs one 128 x 256 output tile
// per CTA with 6 warps:
//   warp 0 lane 0 -- TMA producer: 4 tensor copies per 32-deep k-tile (A_hi,
//     A_lo, B_hi, B_lo, 128-byte swizzle) into a 2-stage ring, `full`
//     mbarriers armed with the byte count;
//   warp 1 -- allocates 256 TMEM columns; lane 0 issues 3 x 4
//     tcgen05.mma.cta_group::1.kind::tf32 (M = 128, N = 256, K = 8) per
//     k-tile and commits each stage's `empty` mbarrier and, at the end, the
//     accumulator barrier;
//   warps 2-5 -- epilogue: tcgen05.ld.32x32b of their TMEM lane quadrant,
//     C = alpha * acc + beta * C with column-major coalesced stores.
// Operands may be K-major (k-contiguous: A Trans, B NoTrans; 128-byte
// swizzle, 8-row x 128-byte atoms, SBO = 1 KB, +32 bytes per 8-deep k-step)
// or MN-major (outer-contiguous: A NoTrans, B Trans; for 32-bit types the
// tensor core only accepts SWIZZLE_128B_BASE32B -- TMA's 128B_ATOM_32B --
// with 32-element x 4-row atoms: LBO = 4 KB between 32-element chunks,
// SBO = 512 B between 4-row k-groups, +1 KB per 8-deep k-step).
#include <cuda.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>

#include "common.cuh"
#include "launch.h"

namespace rectri_cu {
namespace tf32x3 {

constexpr int BM = 128, BN = 256;
constexpr int kThreads = 192;
constexpr int kRingBytes = 192 * 1024;  // operand ring: 2 stages of 32-deep or 4 of 16-deep k-tiles
template <int BK>
struct Geo {
  static constexpr uint32_t A_TILE = BM * BK * 4;
  static constexpr uint32_t B_TILE = BN * BK * 4;
  static constexpr uint32_t STAGE = 2 * A_TILE + 2 * B_TILE;
  static constexpr int STAGES = kRingBytes / STAGE;
  static constexpr int SMEM = STAGES * STAGE + 1024 + 256;
  // K-major tiles: rows of BK fp32 = BK*4 bytes, 128B (BK 32) / 64B (BK 16) swizzle
  static constexpr uint32_t K_SBO = 8 * BK * 4;
  static constexpr uint32_t K_LAYOUT = BK == 32 ? 2u : 4u;
  // MN-major tiles: 32-element chunks of BK k-rows of 128 bytes
  static constexpr uint32_t MN_CHUNK = BK * 128;
};

// ------------------------------------------------------------------ split
// dst_hi/dst_lo (rows x cols, ld = rows) from a strided view.
__global__ void split_kernel(const float* __restrict__ X, i64 ld, i64 rows, i64 cols, float* __restrict__ hi,
                             float* __restrict__ lo) {
  const i64 r = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (r >= rows) return;
  for (i64 c = blockIdx.y; c < cols; c += gridDim.y) {
    const float x = X[r + c * ld];
    const float h = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
    hi[r + c * rows] = h;
    lo[r + c * rows] = x - h;
  }
}

// --------------------------------------------------------------- helpers
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok = 0;
  long long spins = 0;
  while (!ok) {
    if (++spins > (1ll << 26)) __trap();  // a lost arrival aborts the kernel instead of hanging the GPU
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void tma_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];\n" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
// UMMA shared-memory descriptor, version 1 (sm_100).  layout: 2 =
// SWIZZLE_128B (K-major tiles), 1 = SWIZZLE_128B_BASE32B (the only layout
// the tensor core accepts for MN-major 32-bit operands).
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((addr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
  d |= static_cast<uint64_t>(1) << 46;  // version
  d |= static_cast<uint64_t>(layout) << 61;
  return d;
}
__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(bar)
               : "memory");
}

// Instruction descriptor: F32 accumulate, TF32 A/B, majors, N, M.
__host__ __device__ constexpr uint32_t instr_desc(bool a_mn, bool b_mn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) |
         (static_cast<uint32_t>(BN >> 3) << 17) | (static_cast<uint32_t>(BM >> 4) << 24);
}

// A_MN: op(A) m-contiguous (A NoTrans); B_MN: op(B) n-contiguous (B Trans).
template <bool A_MN, bool B_MN, int BK>
__global__ void __launch_bounds__(kThreads, 1)
    tf32x3_kernel(const __grid_constant__ CUtensorMap mAh, const __grid_constant__ CUtensorMap mAl,
                  const __grid_constant__ CUtensorMap mBh, const __grid_constant__ CUtensorMap mBl,
                  const GemmParams<float> p, const uint32_t p_lbo_mn, const uint32_t p_sbo_mn) {
  using G = Geo<BK>;
  constexpr int STAGES = G::STAGES;
  constexpr uint32_t STAGE = G::STAGE, A_TILE = G::A_TILE, B_TILE = G::B_TILE;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const uint32_t sbase = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t bars = sbase + STAGES * STAGE;  // full[s], empty[s], accum
  const uint32_t tmem_slot = bars + 8 * (2 * STAGES + 1);
  auto full_bar = [&](int s) { return bars + 8u * s; };
  auto empty_bar = [&](int s) { return bars + 8u * (STAGES + s); };
  const uint32_t accum_bar = bars + 8u * (2 * STAGES);
  auto tile_a = [&](int s, int lo) { return sbase + s * STAGE + lo * A_TILE; };
  auto tile_b = [&](int s, int lo) { return sbase + s * STAGE + 2 * A_TILE + lo * B_TILE; };

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // Grouped rasterization: consecutive CTAs walk 8 M-tiles down one N column,
  // so the CTAs resident at a time share A row panels and B column panels in L2.
  constexpr int kGroup = 8;
  const int tiles_m = static_cast<int>(ceil_div(p.M, BM));
  const int tiles_n = static_cast<int>(ceil_div(p.N, BN));
  const int lin = static_cast<int>(blockIdx.x);
  const int grp = lin / (kGroup * tiles_n), in_grp = lin - grp * kGroup * tiles_n;
  const int gsize = min(kGroup, tiles_m - grp * kGroup);
  const int m0 = (grp * kGroup + in_grp % gsize) * BM;
  const int n0 = (in_grp / gsize) * BN;
  const int KT = static_cast<int>(ceil_div(p.K, BK));

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(empty_bar(s), 1);
    }
    mbar_init(accum_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  }
  if (warp == 1) {  // TMEM: 128 lanes x 256 fp32 columns
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(tmem_slot), "n"(BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  uint32_t tmem_base;
  asm volatile("ld.shared.b32 %0, [%1];\n" : "=r"(tmem_base) : "r"(tmem_slot));

  if (warp == 0) {
    if (lane == 0) {
      for (int kt = 0; kt < KT; ++kt) {
        const int s = kt % STAGES;
        if (kt >= STAGES) mbar_wait(empty_bar(s), ((kt / STAGES) + 1) & 1);
        mbar_expect_tx(full_bar(s), STAGE);
        const int k0 = kt * BK;
        for (int lo = 0; lo < 2; ++lo) {
          const CUtensorMap* ma = lo ? &mAl : &mAh;
          const CUtensorMap* mb = lo ? &mBl : &mBh;
          if (A_MN) {  // [m-chunk of 32][k BK][32 m] : box {32, BK}
#pragma unroll
            for (int c = 0; c < BM / 32; ++c)
              tma_2d(tile_a(s, lo) + c * G::MN_CHUNK, ma, m0 + 32 * c, k0, full_bar(s));
          } else {  // [m 128][k BK] : box {BK, 128}
            tma_2d(tile_a(s, lo), ma, k0, m0, full_bar(s));
          }
          if (B_MN) {
#pragma unroll
            for (int c = 0; c < BN / 32; ++c)
              tma_2d(tile_b(s, lo) + c * G::MN_CHUNK, mb, n0 + 32 * c, k0, full_bar(s));
          } else {
            tma_2d(tile_b(s, lo), mb, k0, n0, full_bar(s));
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = instr_desc(A_MN, B_MN);
      for (int kt = 0; kt < KT; ++kt) {
        const int s = kt % STAGES;
        mbar_wait(full_bar(s), (kt / STAGES) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;\n");
#pragma unroll
        for (int ks = 0; ks < BK / 8; ++ks) {
          // K-major: +32 bytes per 8-deep k-step inside the swizzle row;
          // MN-major: +1 KB (8 k-rows of 128 bytes).
          const uint32_t ak = A_MN ? ks * 1024u : ks * 32u;
          const uint32_t bk = B_MN ? ks * 1024u : ks * 32u;
          const uint32_t a_lbo = A_MN ? p_lbo_mn : 16u, b_lbo = B_MN ? p_lbo_mn : 16u;
          const uint32_t a_sbo = A_MN ? p_sbo_mn : G::K_SBO, b_sbo = B_MN ? p_sbo_mn : G::K_SBO;
          const uint32_t a_lay = A_MN ? 1u : G::K_LAYOUT, b_lay = B_MN ? 1u : G::K_LAYOUT;
          const uint64_t ah = smem_desc(tile_a(s, 0) + ak, a_lbo, a_sbo, a_lay);
          const uint64_t al = smem_desc(tile_a(s, 1) + ak, a_lbo, a_sbo, a_lay);
          const uint64_t bh = smem_desc(tile_b(s, 0) + bk, b_lbo, b_sbo, b_lay);
          const uint64_t bl = smem_desc(tile_b(s, 1) + bk, b_lbo, b_sbo, b_lay);
          const uint32_t acc0 = (kt > 0 || ks > 0) ? 1u : 0u;
          umma_tf32(tmem_base, al, bh, idesc, acc0);
          umma_tf32(tmem_base, ah, bl, idesc, 1u);
          umma_tf32(tmem_base, ah, bh, idesc, 1u);
        }
        umma_commit(empty_bar(s));  // stage s free once these MMAs complete
      }
      umma_commit(accum_bar);
    }
  } else {
    // Epilogue: warp w reads TMEM lanes 32*(w % 4) .. +31 (= tile rows).
    const int quad = warp & 3;
    const int row = quad * 32 + lane;
    mbar_wait(accum_bar, 0);
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const i64 m = m0 + row;
    const bool beta_zero = p.beta == 0.f;
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 32) {
      uint32_t v[32];
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(quad * 32) << 16) + static_cast<uint32_t>(c0);
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
          "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];\n"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
            "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
            "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]),
            "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),
            "=r"(v[30]), "=r"(v[31])
          : "r"(taddr));
      // all 32 C reads in flight before the first write (one latency per chunk)
      float cold[32];
      const i64 nlim = p.N - (n0 + c0);
      const bool row_ok = m < p.M;
#pragma unroll
      for (int j = 0; j < 32; ++j)
        cold[j] = (row_ok && !beta_zero && j < nlim) ? __ldg(p.C + m + (n0 + c0 + j) * p.ldc) : 0.f;
      __syncwarp();
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");  // warp-converged (.aligned)
      if (row_ok) {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          if (j < nlim) {
            const float acc = __uint_as_float(v[j]);
            p.C[m + (n0 + c0 + j) * p.ldc] = beta_zero ? p.alpha * acc : fmaf(p.alpha, acc, p.beta * cold[j]);
          }
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem_base), "n"(BN));
  }
}

// ------------------------------------------------------------------ host
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeFn encoder() {
  static EncodeFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<EncodeFn>(nullptr);
    return reinterpret_cast<EncodeFn>(f);
  }();
  return fn;
}

// Packed column-major X (rows x cols): outer-contiguous operands (MN-major)
// are (o, k) = X[o + k*rows], box {32, 32}; k-contiguous (K-major) operands
// are (o, k) = X[k + o*rows], box {32, BO}.
bool encode(CUtensorMap* map, const float* X, i64 rows, i64 cols, bool mn, int BO, int BK) {
  EncodeFn enc = encoder();
  if (!enc) return false;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(cols)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(rows) * 4};
  const cuuint32_t box[2] = {mn ? 32u : static_cast<cuuint32_t>(BK), mn ? static_cast<cuuint32_t>(BK)
                                                                          : static_cast<cuuint32_t>(BO)};
  const cuuint32_t estr[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(X), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE,
             mn ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : (BK == 32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B),
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Per-stream scratch for the hi/lo operand copies (grows as needed; the
// recursion's GEMMs run in stream order, so one buffer per stream suffices).
std::mutex g_mu;
struct Scratch {
  float* p = nullptr;
  size_t n = 0;
};
std::map<std::pair<int, cudaStream_t>, Scratch> g_scratch;

float* scratch(cudaStream_t s, size_t floats) {
  if (const CallScratch* cs = call_scratch()) {  // a graph capture: the graph's own buffer
    const int k = cs->find(s);
    return k >= 0 && cs->split_floats[k] >= floats ? cs->split[k] : nullptr;
  }
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(g_mu);
  Scratch& sc = g_scratch[{dev, s}];
  if (sc.n < floats) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &cs);
    if (cs != cudaStreamCaptureStatusNone) return nullptr;  // no allocation inside a capture
    if (sc.p) {
      cudaStreamSynchronize(s);
      cudaFree(sc.p);
    }
    sc.p = nullptr;
    sc.n = 0;
    if (cudaMalloc(&sc.p, floats * sizeof(float)) != cudaSuccess) return nullptr;
    sc.n = floats;
  }
  return sc.p;
}

void split(const float* X, i64 ld, i64 rows, i64 cols, float* hi, float* lo, cudaStream_t s) {
  const dim3 grid(static_cast<unsigned>(ceil_div(rows, 256)),
                  static_cast<unsigned>(std::min<i64>(cols, std::max<i64>(1, 148 * 32 / ceil_div(rows, 256)))));
  split_kernel<<<grid, 256, 0, s>>>(X, ld, rows, cols, hi, lo);
  ++launch_counter();
}

template <bool A_MN, bool B_MN, int BK>
void launch(const CUtensorMap* maps, const GemmParams<float>& p, cudaStream_t s) {
  auto kern = tf32x3_kernel<A_MN, B_MN, BK>;
  constexpr int smem = Geo<BK>::SMEM;
  set_smem(kern, smem);
  const unsigned grid = static_cast<unsigned>(ceil_div(p.M, BM) * ceil_div(p.N, BN));
  // MN-major descriptor offsets: LBO = 32-element chunk stride, SBO = 4-row k-group stride
  const uint32_t lbo = Geo<BK>::MN_CHUNK, sbo = 512;
  kern<<<grid, kThreads, smem, s>>>(maps[0], maps[1], maps[2], maps[3], p, lbo, sbo);
  ++launch_counter();
}

int k_depth() {
  const char* e = getenv("RECTRI_CU_TF32X3_BK");  // 16 (default, 4 stages) or 32 (2 stages)
  return e && atoi(e) == 32 ? 32 : 16;
}

template <int BK>
void launch_bk(bool a_mn, bool b_mn, const CUtensorMap* maps, const GemmParams<float>& p, cudaStream_t s) {
  if (a_mn && b_mn) launch<true, true, BK>(maps, p, s);
  else if (a_mn) launch<true, false, BK>(maps, p, s);
  else if (b_mn) launch<false, true, BK>(maps, p, s);
  else launch<false, false, BK>(maps, p, s);
}

}  // namespace tf32x3

void tf32x3_reserve(cudaStream_t s, size_t floats) { tf32x3::scratch(s, floats); }

namespace {
thread_local bool t_tf32x3 = false;  // the calling thread's current call asked for it
}
void tf32x3_set_call(bool on) { t_tf32x3 = on; }

bool tf32x3_enabled() {
  if (t_tf32x3) return true;
  const char* e = getenv("RECTRI_CU_FP32_TF32X3");
  return e && atoi(e) != 0;
}

// C <- alpha op(A) op(B) + beta C via the 3xTF32 split on tcgen05; false if
// the scratch cannot be provided (caller falls back to the FFMA kernel).
bool launch_gemm_f32_tf32x3(const GemmParams<float>& p, bool ta, bool tb, cudaStream_t s) {
  using namespace tf32x3;
  const i64 M = p.M, N = p.N, K = p.K;
  // Packed hi/lo copies: op(A) as stored (A: M x K or K x M), B as stored.
  const i64 ar = ta ? K : M, ac = ta ? M : K, br = tb ? N : K, bc = tb ? K : N;
  if (ar % 4 != 0 || br % 4 != 0) return false;  // TMA row pitch must be a multiple of 16 bytes
  const size_t need = 2 * static_cast<size_t>(ar * ac + br * bc);
  float* sc = scratch(s, need);
  if (!sc || !encoder()) return false;
  float* ah = sc;
  float* al = ah + ar * ac;
  float* bh = al + ar * ac;
  float* bl = bh + br * bc;
  split(p.A, p.lda, ar, ac, ah, al, s);
  split(p.B, p.ldb, br, bc, bh, bl, s);
  const i64 arp = ar, brp = br;
  const bool a_mn = !ta, b_mn = tb;
  CUtensorMap maps[4];
  const int bk = k_depth();
  if (!encode(&maps[0], ah, arp, ac, a_mn, BM, bk) || !encode(&maps[1], al, arp, ac, a_mn, BM, bk) ||
      !encode(&maps[2], bh, brp, bc, b_mn, BN, bk) || !encode(&maps[3], bl, brp, bc, b_mn, BN, bk))
    return false;
  if (bk == 32) launch_bk<32>(a_mn, b_mn, maps, p, s);
  else launch_bk<16>(a_mn, b_mn, maps, p, s);
  return true;
}

}  // namespace rectri_cu
