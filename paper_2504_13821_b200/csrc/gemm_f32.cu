// gemm_f32.cu -- fp32 GEMM update for the recursion on the FFMA path.
//
// Replaces the reference's CPU GEMM (src/gemm.cpp:17-216; f32 microkernel
// src/gemm_kernels_avx2.cpp:13-40) for fp32.  The north star keeps fp32 on
// exact FFMA (TF32 would change the numerics), so this is a SIMT kernel:
// CTA tile BM x BN x 16, each thread an 8 x 8 register tile (two 4x4
// quadrants per dimension so fragment reads are 128-bit and conflict-free),
// STAGES-deep cp.async ring.  Operands that are contiguous along k are
// transposed on the fly by 4-byte cp.async into the k-major shared layout.
// Accumulation is a k-ascending fma chain per element, independent of the
// tile configuration.
#include "common.cuh"
#include "launch.h"

namespace rectri_cu {
namespace {

constexpr int kBK = 16;
constexpr int kPad = 4;  // floats of row padding (keeps 16-byte alignment)

// Per-thread loader of one operand tile.  Shared layout for both operands:
// [k][o] rows of BO + kPad floats.
//   MC (outer-contiguous source, element (o, k) at X[o + k*ld]): VEC-float
//     chunks along o; the thread's o is fixed, its k advances by NT / CPR.
//   KC (k-contiguous source, element (o, k) at X[k + o*ld]): transposed by
//     4-byte copies, consecutive threads walk k (contiguous global
//     addresses); the thread's k is fixed, its o advances by NT / kBK.
// The thread's global pointer is computed once and advanced per k-tile.
template <int BO, int NT, int VEC, bool KC>
struct FLoader {
  static constexpr int RS = BO + kPad;
  static constexpr int CPR = KC ? kBK : BO / VEC;  // copies per shared row (KC: per o)
  static constexpr int IT = kBK * BO / VEC / NT;
  static constexpr int STEP = NT / CPR;            // MC: k rows, KC: o rows per iteration
  static_assert(!KC || VEC == 1, "KC copies are 4-byte transposes");
  static_assert(NT % CPR == 0 && (kBK * BO / VEC) % NT == 0, "loader trip count");

  const float* base;
  const float* p0;
  i64 ld, step;
  int k_first, o_first;
  int o_lim, k_lim, fix_bytes;

  __device__ void init(const float* X, i64 ld_, i64 o0, i64 O, i64 K) {
    ld = ld_;
    const int q = threadIdx.x;
    if (KC) {
      k_first = q % kBK;
      o_first = q / kBK;
    } else {
      o_first = (q % CPR) * VEC;
      k_first = q / CPR;
    }
    o_lim = static_cast<int>(O - o0 < (1 << 30) ? O - o0 : (1 << 30));
    k_lim = static_cast<int>(K < (1 << 30) ? K : (1 << 30));
    base = KC ? X + o0 * ld : X + o0;
    p0 = KC ? base + static_cast<i64>(o_first) * ld + k_first : base + o_first + static_cast<i64>(k_first) * ld;
    step = static_cast<i64>(STEP) * ld;
    const int rem = o_lim - o_first;
    fix_bytes = rem >= VEC ? VEC * 4 : (rem > 0 ? rem * 4 : 0);
  }

  __device__ __forceinline__ void load(float* s, i64 kt) const {
    const int k0 = static_cast<int>(kt * kBK);
    const float* tb = p0 + (KC ? static_cast<i64>(k0) : static_cast<i64>(k0) * ld);
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      const int o = o_first + (KC ? it * STEP : 0);
      const int k = k_first + (KC ? 0 : it * STEP);
      int bytes;
      if (KC) bytes = (o < o_lim && k0 + k < k_lim) ? 4 : 0;
      else bytes = (k0 + k < k_lim) ? fix_bytes : 0;
      const float* g = bytes ? tb + it * step : base;
      float* dst = s + k * RS + o;
      if constexpr (VEC == 4) cp_async16(dst, g, bytes);
      else cp_async4(dst, g, bytes);
    }
  }
};

template <int BM, int BN, int STAGES, bool TA, bool TB, int VA, int VB>
__global__ void __launch_bounds__((BM / 8) * (BN / 8), 2)
    sgemm_ffma_kernel(const GemmParams<float> p) {
  constexpr int TX = BN / 8, TY = BM / 8, NT = TX * TY;
  constexpr int RSA = BM + kPad, RSB = BN + kPad;
  extern __shared__ __align__(128) float fsmem[];
  float* sA = fsmem;
  float* sB = fsmem + STAGES * kBK * RSA;

  const int tx = threadIdx.x % TX, ty = threadIdx.x / TX;
  const i64 m0 = static_cast<i64>(blockIdx.x) * BM;
  const i64 n0 = static_cast<i64>(blockIdx.y) * BN;
  const i64 KT = ceil_div(p.K, kBK);

  FLoader<BM, NT, TA ? 1 : VA, TA> la;
  FLoader<BN, NT, TB ? VB : 1, !TB> lb;
  la.init(p.A, p.lda, m0, p.M, p.K);
  lb.init(p.B, p.ldb, n0, p.N, p.K);
  auto load_stage = [&](int stage, i64 kt) {
    la.load(sA + stage * kBK * RSA, kt);
    lb.load(sB + stage * kBK * RSB, kt);
  };

  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < KT) load_stage(s, s);
    cp_async_commit();
  }
  for (i64 kt = 0; kt < KT; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const i64 nk = kt + STAGES - 1;
      if (nk < KT) load_stage(static_cast<int>(nk % STAGES), nk);
      cp_async_commit();
    }
    const int st = static_cast<int>(kt % STAGES);
    const float* a_s = sA + st * kBK * RSA;
    const float* b_s = sB + st * kBK * RSB;
#pragma unroll
    for (int k = 0; k < kBK; ++k) {
      const float4 a0 = *reinterpret_cast<const float4*>(a_s + k * RSA + ty * 4);
      const float4 a1 = *reinterpret_cast<const float4*>(a_s + k * RSA + BM / 2 + ty * 4);
      const float4 b0 = *reinterpret_cast<const float4*>(b_s + k * RSB + tx * 4);
      const float4 b1 = *reinterpret_cast<const float4*>(b_s + k * RSB + BN / 2 + tx * 4);
      const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
  }
  cp_async_wait<0>();

  const bool beta_zero = p.beta == 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const i64 n = n0 + (j < 4 ? tx * 4 + j : BN / 2 + tx * 4 + j - 4);
    if (n >= p.N) continue;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const i64 m = m0 + (i < 4 ? ty * 4 + i : BM / 2 + ty * 4 + i - 4);
      if (m < p.M) {
        float* c = p.C + m + n * p.ldc;
        *c = beta_zero ? p.alpha * acc[i][j] : fmaf(p.alpha, acc[i][j], p.beta * *c);
      }
    }
  }
}

template <int BM, int BN, int STAGES, bool TA, bool TB, int VA, int VB>
void launch_cfg(const GemmParams<float>& p, cudaStream_t s) {
  auto kern = sgemm_ffma_kernel<BM, BN, STAGES, TA, TB, VA, VB>;
  constexpr int smem = STAGES * kBK * (BM + BN + 2 * kPad) * static_cast<int>(sizeof(float));
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  dim3 grid(static_cast<unsigned>(ceil_div(p.M, BM)), static_cast<unsigned>(ceil_div(p.N, BN)));
  kern<<<grid, (BM / 8) * (BN / 8), smem, s>>>(p);
  ++launch_counter();
}

bool aligned16(const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15u) == 0; }

template <int BM, int BN, int STAGES>
void dispatch(const GemmParams<float>& p, bool ta, bool tb, cudaStream_t s) {
  // The vector width only applies to outer-contiguous operands (A when !ta,
  // B when tb); it needs 16-byte aligned columns.
  const bool va = !ta && aligned16(p.A) && p.lda % 4 == 0;
  const bool vb = tb && aligned16(p.B) && p.ldb % 4 == 0;
#define RECTRI_CFG(TA_, TB_)                                                   \
  if (ta == TA_ && tb == TB_) {                                                \
    if (va && vb) launch_cfg<BM, BN, STAGES, TA_, TB_, 4, 4>(p, s);            \
    else if (va) launch_cfg<BM, BN, STAGES, TA_, TB_, 4, 1>(p, s);             \
    else if (vb) launch_cfg<BM, BN, STAGES, TA_, TB_, 1, 4>(p, s);             \
    else launch_cfg<BM, BN, STAGES, TA_, TB_, 1, 1>(p, s);                     \
    return;                                                                    \
  }
  RECTRI_CFG(false, false)
  RECTRI_CFG(true, false)
  RECTRI_CFG(false, true)
  RECTRI_CFG(true, true)
#undef RECTRI_CFG
}

}  // namespace

void launch_gemm_f32(const GemmParams<float>& p, bool ta, bool tb, cudaStream_t s) {
  if (p.M <= 0 || p.N <= 0 || p.K <= 0) return;
  if (p.M >= 128 && p.N >= 128) dispatch<128, 128, 3>(p, ta, tb, s);
  else if (p.N >= 128) dispatch<64, 128, 3>(p, ta, tb, s);
  else if (p.M >= 128) dispatch<128, 64, 3>(p, ta, tb, s);
  else dispatch<64, 64, 3>(p, ta, tb, s);
}

}  // namespace rectri_cu
