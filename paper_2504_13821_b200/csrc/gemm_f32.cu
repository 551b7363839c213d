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

// Shared layout for both operands: [k][o] with row stride BO + kPad.
// Outer-contiguous source: element (o, k) at X[o + k * ld].
template <int BO, int NT, int VEC>
__device__ __forceinline__ void load_mc(float* s, const float* X, i64 ld, i64 o0, i64 O, i64 k0,
                                        i64 K) {
  constexpr int RS = BO + kPad;
  if constexpr (VEC == 4) {
    constexpr int CPR = BO / 4;
#pragma unroll
    for (int q = threadIdx.x; q < kBK * CPR; q += NT) {
      const int k = q / CPR, oc = q % CPR;
      const i64 go = o0 + 4 * oc, gk = k0 + k;
      int bytes = 0;
      const float* src = X;
      if (gk < K && go < O) {
        const i64 rem = O - go;
        bytes = rem >= 4 ? 16 : static_cast<int>(rem) * 4;
        src = X + go + gk * ld;
      }
      cp_async16(s + k * RS + 4 * oc, src, bytes);
    }
  } else {
#pragma unroll 4
    for (int q = threadIdx.x; q < kBK * BO; q += NT) {
      const int k = q / BO, o = q % BO;
      const i64 go = o0 + o, gk = k0 + k;
      const bool ok = gk < K && go < O;
      cp_async4(s + k * RS + o, ok ? X + go + gk * ld : X, ok ? 4 : 0);
    }
  }
}

// k-contiguous source: element (o, k) at X[k + o * ld]; transposed by 4-byte
// copies (consecutive threads walk k, i.e. contiguous global addresses).
template <int BO, int NT>
__device__ __forceinline__ void load_kc(float* s, const float* X, i64 ld, i64 o0, i64 O, i64 k0,
                                        i64 K) {
  constexpr int RS = BO + kPad;
#pragma unroll 4
  for (int q = threadIdx.x; q < kBK * BO; q += NT) {
    const int k = q & (kBK - 1), o = q / kBK;
    const i64 go = o0 + o, gk = k0 + k;
    const bool ok = gk < K && go < O;
    cp_async4(s + k * RS + o, ok ? X + gk + go * ld : X, ok ? 4 : 0);
  }
}

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

  auto load_stage = [&](int stage, i64 kt) {
    const i64 k0 = kt * kBK;
    float* a = sA + stage * kBK * RSA;
    float* b = sB + stage * kBK * RSB;
    if constexpr (TA) load_kc<BM, NT>(a, p.A, p.lda, m0, p.M, k0, p.K);
    else load_mc<BM, NT, VA>(a, p.A, p.lda, m0, p.M, k0, p.K);
    if constexpr (TB) load_mc<BN, NT, VB>(b, p.B, p.ldb, n0, p.N, k0, p.K);
    else load_kc<BN, NT>(b, p.B, p.ldb, n0, p.N, k0, p.K);
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
