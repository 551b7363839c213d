// gemm_f32.cu -- fp32 GEMM update for the recursion on the FFMA path.
//
// Replaces the reference's CPU GEMM (src/gemm.cpp:17-216; f32 microkernel
// src/gemm_kernels_avx2.cpp:13-40) for fp32.  The north star keeps fp32 on
// exact FFMA (TF32 would change the numerics), so this is a SIMT kernel:
// CTA tile BM x BN x 16, 256 threads, each an 8 x 8 register tile, STAGES-deep
// cp.async ring.  The two operand layouts get their own shared layout and
// fragment pattern:
//   outer-contiguous source (A for op N, B for op T): shared [k][o], 16-byte
//     copies; a thread's 8 outer indices are two runs of 4 (o = 4t.., BO/2+4t..)
//     read as two LDS.128 per k;
//   k-contiguous source (A for op T, B for op N): shared [o][k + 2], 8-byte
//     copies (no transposition); a thread's 8 outer indices are t + 16j, read
//     as LDS.64 pairs covering two k-steps (row stride 18 floats: the 16
//     lanes of a phase hit distinct bank pairs).
// Accumulation is a k-ascending fma chain per element, independent of the
// tile configuration.
//
// That is v1 (RECTRI_CU_SGEMM=1).  v2 (sgemm_ffma2_kernel, the default) keeps
// the tile but stores every operand as [k][o], double-buffers one k-step of
// fragments in registers, uses 32-deep k-tiles for op-N A and a float4
// epilogue; see its comment.  B200, 8192x16384x8192 (v1 -> v2):
// NN 50.4 -> 55.1 TF/s, TN 41.1 -> 50.7, NT 53.7 -> 56.7 (FFMA peak 71);
// K = 256 levels 18 -> 23 TF/s.
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "launch.h"

namespace rectri_cu {
namespace {

constexpr int kBK = 16;
constexpr int kPadMC = 4;  // [k][o] rows: BO + 4 floats (16-byte aligned rows)
constexpr int kPadKC = 2;  // [o][k] rows: 16 + 2 floats (8-byte aligned rows)
constexpr int kRowKC = kBK + kPadKC;

template <int BO, bool KC>
struct FLayout {
  static constexpr int ELEMS = KC ? BO * kRowKC : kBK * (BO + kPadMC);
};

// Per-thread loader.  MC: (o, k) at X[o + k*ld], chunks of VEC floats along
// o into [k][o]; KC: (o, k) at X[k + o*ld], chunks of VEC floats along k into
// [o][k].  The thread's chunk column is fixed, its row advances by STEP.
template <int BO, int NT, int VEC, bool KC, int BKT = kBK>
struct FLoader {
  static constexpr int WIDTH = KC ? BKT : BO;  // source run length per row
  static constexpr int CPR = WIDTH / VEC;
  static constexpr int ROWS = KC ? BO : BKT;
  static constexpr int IT = CPR * ROWS / NT;
  static constexpr int STEP = NT / CPR;
  static_assert(NT % CPR == 0 && (CPR * ROWS) % NT == 0, "loader trip count");

  const float* base;
  const float* p0;
  i64 ld, step;
  int row0, col;
  int o_lim, k_lim, fix_bytes, soff;

  __device__ void init(const float* X, i64 ld_, i64 o0, i64 O, i64 K) {
    ld = ld_;
    row0 = threadIdx.x / CPR;
    col = (threadIdx.x % CPR) * VEC;
    o_lim = static_cast<int>(O - o0 < (1 << 30) ? O - o0 : (1 << 30));
    k_lim = static_cast<int>(K < (1 << 30) ? K : (1 << 30));
    base = KC ? X + o0 * ld : X + o0;
    p0 = base + static_cast<i64>(row0) * ld + col;  // (row, col) at base + row*ld + col
    step = static_cast<i64>(STEP) * ld;
    const int rem = o_lim - col;
    fix_bytes = rem >= VEC ? VEC * 4 : (rem > 0 ? rem * 4 : 0);
    soff = KC ? row0 * kRowKC + col : row0 * (BO + kPadMC) + col;
  }

  __device__ __forceinline__ void load(float* s, i64 kt) const {
    const int k0 = static_cast<int>(kt * BKT);
    const float* tb = p0 + (KC ? static_cast<i64>(k0) : static_cast<i64>(k0) * ld);
    // interior tiles (the vast majority): no per-copy bounds, the source
    // pointer advanced by one add per copy instead of a multiply
    const bool inside = KC ? (k0 + BKT <= k_lim && o_lim >= BO) : (k0 + BKT <= k_lim && fix_bytes == VEC * 4);
    if (inside) {
      const float* g = tb;
#pragma unroll
      for (int it = 0; it < IT; ++it, g += step) {
        float* dst = s + soff + it * STEP * (KC ? kRowKC : BO + kPadMC);
        if constexpr (VEC == 4) cp_async16(dst, g, 16);
        else if constexpr (VEC == 2) cp_async8(dst, g, 8);
        else cp_async4(dst, g, 4);
      }
      return;
    }
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      const int row = row0 + it * STEP;
      int bytes;
      if (KC) {
        const int rem = k_lim - (k0 + col);
        bytes = row < o_lim ? (rem >= VEC ? VEC * 4 : (rem > 0 ? rem * 4 : 0)) : 0;
      } else {
        bytes = (k0 + row < k_lim) ? fix_bytes : 0;
      }
      const float* g = bytes ? tb + it * step : base;
      float* dst = KC ? s + row * kRowKC + col : s + row * (BO + kPadMC) + col;
      if constexpr (VEC == 4) cp_async16(dst, g, bytes);
      else if constexpr (VEC == 2) cp_async8(dst, g, bytes);
      else cp_async4(dst, g, bytes);
    }
  }
};

// The thread's 8 outer indices of an operand and how to read them.
template <int BO, bool KC>
struct FFrag {
  // index j (0..7) of thread t (0..15 along this operand)
  __device__ static int outer(int t, int j) {
    return KC ? t + 16 * j : (j < 4 ? 4 * t + j : BO / 2 + 4 * t + j - 4);
  }
  // values for k-steps k and k+1: v[0][j] (k), v[1][j] (k+1)
  __device__ static void read(const float* s, int t, int k, float (&v)[2][8]) {
    if constexpr (KC) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float2 x = *reinterpret_cast<const float2*>(s + (t + 16 * j) * kRowKC + k);
        v[0][j] = x.x;
        v[1][j] = x.y;
      }
    } else {
      constexpr int RS = BO + kPadMC;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const float4 a = *reinterpret_cast<const float4*>(s + (k + h) * RS + 4 * t);
        const float4 b = *reinterpret_cast<const float4*>(s + (k + h) * RS + BO / 2 + 4 * t);
        v[h][0] = a.x; v[h][1] = a.y; v[h][2] = a.z; v[h][3] = a.w;
        v[h][4] = b.x; v[h][5] = b.y; v[h][6] = b.z; v[h][7] = b.w;
      }
    }
  }
};

template <int BM, int BN, int STAGES, bool TA, bool TB, int VA, int VB>
__global__ void __launch_bounds__((BM / 8) * (BN / 8), 2)
    sgemm_ffma_kernel(const GemmParams<float> p) {
  pdl_wait();  // PDL: no-op unless launched programmatically (launch_kernel)
  constexpr int TX = BN / 8, TY = BM / 8, NT = TX * TY;
  static_assert(TX == 16 && TY == 16, "16 x 16 thread grid");
  constexpr bool A_KC = TA, B_KC = !TB;  // k-contiguous sources
  constexpr int A_EL = FLayout<BM, A_KC>::ELEMS, B_EL = FLayout<BN, B_KC>::ELEMS;
  extern __shared__ __align__(128) float fsmem[];
  float* sA = fsmem;
  float* sB = fsmem + STAGES * A_EL;

  const int tx = threadIdx.x % TX, ty = threadIdx.x / TX;
  const i64 m0 = static_cast<i64>(blockIdx.x) * BM;
  const i64 n0 = static_cast<i64>(blockIdx.y) * BN;
  const i64 KT = ceil_div(p.K, kBK);

  FLoader<BM, NT, VA, A_KC> la;
  FLoader<BN, NT, VB, B_KC> lb;
  la.init(p.A, p.lda, m0, p.M, p.K);
  lb.init(p.B, p.ldb, n0, p.N, p.K);

  // A outer-contiguous (op N): the thread's m values come in adjacent pairs
  // (LDS.128), so accumulators are packed as m-pairs and updated with the
  // packed FFMA2 (fma.rn.f32x2, B value broadcast as a scalar operand): two
  // independent round-to-nearest FMAs per instruction, bitwise the same as
  // two fmaf, at half the issue slots and register-bank reads per FMA.
  // A k-contiguous (op T): scalar FFMA.
  constexpr bool kPacked = !A_KC;
  float acc[8][8];
  unsigned long long acc2[4][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc2[i][j] = 0ull;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < KT) {
      la.load(sA + s * A_EL, s);
      lb.load(sB + s * B_EL, s);
    }
    cp_async_commit();
  }
  for (i64 kt = 0; kt < KT; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const i64 nk = kt + STAGES - 1;
      if (nk < KT) {
        const int ws = static_cast<int>(nk % STAGES);
        la.load(sA + ws * A_EL, nk);
        lb.load(sB + ws * B_EL, nk);
      }
      cp_async_commit();
    }
    const int st = static_cast<int>(kt % STAGES);
    const float* a_s = sA + st * A_EL;
    const float* b_s = sB + st * B_EL;
#pragma unroll
    for (int k = 0; k < kBK; k += 2) {
      float av[2][8], bv[2][8];
      FFrag<BM, A_KC>::read(a_s, ty, k, av);
      FFrag<BN, B_KC>::read(b_s, tx, k, bv);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if constexpr (kPacked) {
#pragma unroll
          for (int ip = 0; ip < 4; ++ip) {
            unsigned long long ap;
            asm("mov.b64 %0, {%1, %2};" : "=l"(ap) : "f"(av[h][2 * ip]), "f"(av[h][2 * ip + 1]));
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              unsigned long long bb;
              asm("mov.b64 %0, {%1, %1};" : "=l"(bb) : "f"(bv[h][j]));
              asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc2[ip][j]) : "l"(ap), "l"(bb));
            }
          }
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(av[h][i], bv[h][j], acc[i][j]);
        }
      }
    }
  }
  cp_async_wait<0>();
  if constexpr (kPacked) {
#pragma unroll
    for (int ip = 0; ip < 4; ++ip)
#pragma unroll
      for (int j = 0; j < 8; ++j)
        asm("mov.b64 {%0, %1}, %2;" : "=f"(acc[2 * ip][j]), "=f"(acc[2 * ip + 1][j]) : "l"(acc2[ip][j]));
  }

  // Epilogue, per column: every C read of the column issued before the writes.
  const bool beta_zero = p.beta == 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const i64 n = n0 + FFrag<BN, B_KC>::outer(tx, j);
    if (n >= p.N) continue;
    float cold[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const i64 m = m0 + FFrag<BM, A_KC>::outer(ty, i);
      cold[i] = (!beta_zero && m < p.M) ? p.C[m + n * p.ldc] : 0.f;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const i64 m = m0 + FFrag<BM, A_KC>::outer(ty, i);
      if (m < p.M) p.C[m + n * p.ldc] = beta_zero ? p.alpha * acc[i][j] : fmaf(p.alpha, acc[i][j], p.beta * cold[i]);
    }
  }
}

// ---- v2: one shared layout for every transposition case.  k-contiguous
// sources are transposed into [k][o] by 4-byte copies (lane -> 8 k x 4 o, so
// a warp reads four 32-byte sectors and writes 32 distinct banks), so both
// operands are read as two LDS.128 per k-step, one k-step of fragments is
// double-buffered in registers across the k loop (and across tiles: the
// next tile's first fragments are read right after its barrier), and every
// case accumulates with FFMA2 on m-pairs.  Same k-ascending fma chain per
// element as v1, so the two kernels agree bit for bit.
template <int BO, int NT, int BK = kBK>
struct TLoaderKC {
  static constexpr int RS = BO + kPadMC;
  static_assert(NT == 256 && BO % 32 == 0, "8 k x 32 o per pass");
  const float* base;
  const float* p0;
  i64 step32;
  int kl, ol, o_lim, k_lim, soff;

  __device__ void init(const float* X, i64 ld, i64 o0, i64 O, i64 K) {
    kl = threadIdx.x % 8;
    ol = threadIdx.x / 8;
    soff = kl * RS + ol;  // this thread's element of a stage, constant offsets from here
    o_lim = static_cast<int>(O - o0 < (1 << 30) ? O - o0 : (1 << 30));
    k_lim = static_cast<int>(K < (1 << 30) ? K : (1 << 30));
    base = X + o0 * ld;
    p0 = base + static_cast<i64>(ol) * ld + kl;
    step32 = 32 * ld;
  }
  __device__ __forceinline__ void load(float* s, i64 kt) const {
    const int k0 = static_cast<int>(kt * BK);
    if (k0 + BK <= k_lim && o_lim >= BO) {  // interior tile: no per-copy bounds
      const float* g = p0 + k0;
      float* d = s + soff;
#pragma unroll
      for (int ob = 0; ob < BO / 32; ++ob, g += step32)
#pragma unroll
        for (int h = 0; h < BK / 8; ++h) cp_async4(d + 8 * h * RS + 32 * ob, g + 8 * h, 4);
      return;
    }
#pragma unroll
    for (int h = 0; h < BK / 8; ++h)
#pragma unroll
      for (int ob = 0; ob < BO / 32; ++ob) {
        const int k = kl + 8 * h, o = ol + 32 * ob;
        const bool ok = k0 + k < k_lim && o < o_lim;
        cp_async4(s + k * RS + o, ok ? p0 + ob * step32 + k0 + 8 * h : base, ok ? 4 : 0);
      }
  }
};

// Thread t's CN values of k-step k: CN / 4 float4 runs, at 4t + q * BO / (CN / 4).
template <int BO, int CN = 8>
__device__ __forceinline__ void read_k(const float* s, int t, int k, float (&v)[CN]) {
  constexpr int RS = BO + kPadMC, Q = CN / 4;
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const float4 a = *reinterpret_cast<const float4*>(s + k * RS + q * (BO / Q) + 4 * t);
    v[4 * q] = a.x; v[4 * q + 1] = a.y; v[4 * q + 2] = a.z; v[4 * q + 3] = a.w;
  }
}
// Outer index (row of A / column of B within the tile) of value j of thread t.
template <int BO, int CN = 8>
__device__ __forceinline__ int outer_k(int t, int j) { return (j / 4) * (BO / (CN / 4)) + 4 * t + (j & 3); }

// BN = 128: 16 x 16 threads of 8 x 8 (two CTAs per SM); BN = 256: 8 x 16
// per thread (one CTA per SM): per k-step a warp issues 6 LDS.128 for 64
// FFMA2 instead of 4 for 32 -- the shared-memory wavefronts, not the FMA
// pipe, bound the 8 x 8 tile (ncu: 76 % of shared bandwidth at 85 % FMA).
// Same k-ascending chain per element either way: bitwise equal.
// CK: the ring checker's instantiation (RECTRI_CU_RING_CHECK): each k-step's
// fragments are compared, bit for bit, with their op(A) / op(B) elements in
// global memory (zero outside the matrix, as the loaders fill them) before
// they are used; ring_plant reads the wrong stage (the negative test).
template <int BM, int BN, int STAGES, bool TA, bool TB, int VA, int VB, int BK = kBK, bool CK = false>
__global__ void __launch_bounds__(256, BN == 128 ? 2 : 1) sgemm_ffma2_kernel(const GemmParams<float> p) {
  pdl_wait();  // PDL: no-op unless launched programmatically (launch_kernel)
  constexpr int TX = 16, NT = 256;
  constexpr int CN = BN / 16;  // columns per thread
  static_assert(BM == 128 && (BN == 128 || BN == 256), "16 x 16 threads of 8 x CN");
  constexpr bool A_KC = TA, B_KC = !TB;
  constexpr int A_EL = BK * (BM + kPadMC), B_EL = BK * (BN + kPadMC);
  using LA = std::conditional_t<A_KC, TLoaderKC<BM, NT, BK>, FLoader<BM, NT, VA, false, BK>>;
  using LB = std::conditional_t<B_KC, TLoaderKC<BN, NT, BK>, FLoader<BN, NT, VB, false, BK>>;
  extern __shared__ __align__(128) float fsmem[];
  float* sA = fsmem;
  float* sB = fsmem + STAGES * A_EL;

  const int tx = threadIdx.x % TX, ty = threadIdx.x / TX;
  const i64 m0 = static_cast<i64>(blockIdx.x) * BM;
  const i64 n0 = static_cast<i64>(blockIdx.y) * BN;
  const i64 KT = ceil_div(p.K, BK);
  LA la;
  LB lb;
  la.init(p.A, p.lda, m0, p.M, p.K);
  lb.init(p.B, p.ldb, n0, p.N, p.K);

  unsigned long long acc2[4][CN];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < CN; ++j) acc2[i][j] = 0ull;

  // Stage s holds k-tile j with j % STAGES == s.  full[s]: every thread's
  // cp.async copies of the tile have landed (cp.async.mbarrier.arrive.noinc,
  // 256 arrivals); empty[s]: all 8 warps have read the tile.  Instead of a
  // CTA barrier per k-tile, the refill of a stage is issued one tile later
  // than it could be -- at the end of tile kt the stage of tile kt - 1 gets
  // tile kt + STAGES - 1 -- so the empty wait is normally already satisfied
  // and warps drift apart freely; the refill still has a whole tile of
  // compute to land in.
  static_assert(STAGES >= 3, "the deferred refill needs three stages");
  __shared__ __align__(8) unsigned long long bars[2 * STAGES];
  const uint32_t full0 = smem_u32(&bars[0]), empty0 = smem_u32(&bars[STAGES]);
  if (threadIdx.x == 0) {
    for (int q = 0; q < STAGES; ++q) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(full0 + 8 * q), "r"(NT));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(empty0 + 8 * q), "r"(NT / 32));
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  auto bar_wait = [](uint32_t bar, uint32_t parity) {
    uint32_t ok = 0;
    while (!ok)
      asm volatile(
          "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
          " selp.u32 %0, 1, 0, p;\n}\n"
          : "=r"(ok)
          : "r"(bar), "r"(parity)
          : "memory");
  };
  auto fill = [&](int stage, i64 tile) {  // this thread's copies of k-tile `tile`, then its arrival
    la.load(sA + stage * A_EL, tile);
    lb.load(sB + stage * B_EL, tile);
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(full0 + 8 * stage) : "memory");
  };

#pragma unroll
  for (int s = 0; s < STAGES; ++s)
    if (s < KT) fill(s, s);
  float fa[2][8], fb[2][CN];
  // stage a consumer reads (CK && ring_plant: the next one, the planted mix-up)
  auto rs_of = [&](int stage) { return CK && p.ring_plant ? (stage + 1) % STAGES : stage; };
  bar_wait(full0, 0);
  read_k<BM>(sA + rs_of(0) * A_EL, ty, 0, fa[0]);
  read_k<BN, CN>(sB + rs_of(0) * B_EL, tx, 0, fb[0]);
  int st = 0;
  const uint32_t dep0 = static_cast<uint32_t>(p.K >> 40);  // 0 at run time, unknown to ptxas
  for (i64 kt = 0; kt < KT; ++kt) {
    const int cur = st;
    const float* a_s = sA + rs_of(st) * A_EL;
    const float* b_s = sB + rs_of(st) * B_EL;
#pragma unroll
    for (int k = 0; k < BK; ++k) {
      const int cb = k & 1;
      if (k + 1 < BK) {
        read_k<BM>(a_s, ty, k + 1, fa[cb ^ 1]);
        read_k<BN, CN>(b_s, tx, k + 1, fb[cb ^ 1]);
      } else {
        // refill the stage of tile kt - 1 (released after its last FFMAs) with tile kt + STAGES - 1
        const i64 nt = kt + STAGES - 1;
        if (kt >= 1 && nt < KT) {
          const int rs = static_cast<int>((kt - 1) % STAGES);
          bar_wait(empty0 + 8 * rs, static_cast<uint32_t>(((kt - 1) / STAGES) & 1));
          fill(rs, nt);
        }
        st = st + 1 == STAGES ? 0 : st + 1;
        if (kt + 1 < KT) {
          bar_wait(full0 + 8 * st, static_cast<uint32_t>(((kt + 1) / STAGES) & 1));
          read_k<BM>(sA + rs_of(st) * A_EL, ty, 0, fa[cb ^ 1]);
          read_k<BN, CN>(sB + rs_of(st) * B_EL, tx, 0, fb[cb ^ 1]);
        }
      }
      if constexpr (CK) {  // RECTRI_CU_RING_CHECK: fragments of (kt, k) vs op(A) / op(B)
        const i64 kg = kt * BK + k;
        unsigned bad = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const i64 m = m0 + outer_k<BM>(ty, j);
          const float e = m < p.M && kg < p.K ? (TA ? p.A[kg + m * p.lda] : p.A[m + kg * p.lda]) : 0.f;
          bad += __float_as_uint(fa[cb][j]) != __float_as_uint(e) ? 1u : 0u;
        }
#pragma unroll
        for (int j = 0; j < CN; ++j) {
          const i64 n = n0 + outer_k<BN, CN>(tx, j);
          const float e = n < p.N && kg < p.K ? (TB ? p.B[n + kg * p.ldb] : p.B[kg + n * p.ldb]) : 0.f;
          bad += __float_as_uint(fb[cb][j]) != __float_as_uint(e) ? 1u : 0u;
        }
        if (bad) atomicAdd(p.ring_check, static_cast<unsigned long long>(bad));
      }
#pragma unroll
      for (int ip = 0; ip < 4; ++ip) {
        unsigned long long ap;
        asm("mov.b64 %0, {%1, %2};" : "=l"(ap) : "f"(fa[cb][2 * ip]), "f"(fa[cb][2 * ip + 1]));
#pragma unroll
        for (int j = 0; j < CN; ++j) {
          unsigned long long bb;
          asm("mov.b64 %0, {%1, %1};" : "=l"(bb) : "f"(fb[cb][j]));
          asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc2[ip][j]) : "l"(ap), "l"(bb));
        }
      }
    }
    // release the stage once this warp's last reads of tile kt have landed:
    // the arrive's address depends on accumulators every one of those
    // fragments fed (slot_dep, common.cuh: ptxas may otherwise issue the
    // arrive while the loads are in flight)
    uint32_t dep = 0;
#pragma unroll
    for (int ip = 0; ip < 4; ++ip) dep |= slot_dep(dep0, acc2[ip][0]);
#pragma unroll
    for (int j = 1; j < CN; ++j) dep |= slot_dep(dep0, acc2[0][j]);
    __syncwarp();
    if ((threadIdx.x & 31) == 0)
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(empty0 + 8 * cur + dep) : "memory");
  }
  cp_async_wait<0>();

  const bool beta_zero = p.beta == 0.f;
  // Full-height tile with a 16-byte aligned C: each column's 8 values are two
  // float4 runs (rows 4ty.., BM/2 + 4ty..), and the reads of 4 columns are
  // issued before their writes -- two dependent round trips per thread
  // instead of eight (short-K updates stall on exactly these reads).
  const bool vec = m0 + BM <= p.M && (reinterpret_cast<uintptr_t>(p.C) & 15) == 0 && p.ldc % 4 == 0;
  if (vec) {
#pragma unroll
    for (int jb = 0; jb < CN; jb += 4) {
      float4 cv[4][2];
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) {
        const i64 n = n0 + outer_k<BN, CN>(tx, jb + jj);
        const float* cp = p.C + m0 + 4 * ty + n * p.ldc;
        const bool rd = !beta_zero && n < p.N;
        cv[jj][0] = rd ? *reinterpret_cast<const float4*>(cp) : make_float4(0.f, 0.f, 0.f, 0.f);
        cv[jj][1] = rd ? *reinterpret_cast<const float4*>(cp + BM / 2) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) {
        const int j = jb + jj;
        const i64 n = n0 + outer_k<BN, CN>(tx, j);
        if (n >= p.N) continue;
        float a[8];
#pragma unroll
        for (int ip = 0; ip < 4; ++ip)
          asm("mov.b64 {%0, %1}, %2;" : "=f"(a[2 * ip]), "=f"(a[2 * ip + 1]) : "l"(acc2[ip][j]));
        const float co[8] = {cv[jj][0].x, cv[jj][0].y, cv[jj][0].z, cv[jj][0].w,
                             cv[jj][1].x, cv[jj][1].y, cv[jj][1].z, cv[jj][1].w};
        float o[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) o[i] = beta_zero ? p.alpha * a[i] : fmaf(p.alpha, a[i], p.beta * co[i]);
        float* cp = p.C + m0 + 4 * ty + n * p.ldc;
        *reinterpret_cast<float4*>(cp) = make_float4(o[0], o[1], o[2], o[3]);
        *reinterpret_cast<float4*>(cp + BM / 2) = make_float4(o[4], o[5], o[6], o[7]);
      }
    }
    return;
  }
#pragma unroll
  for (int j = 0; j < CN; ++j) {
    const i64 n = n0 + outer_k<BN, CN>(tx, j);
    if (n >= p.N) continue;
    float accj[8], cold[8];
#pragma unroll
    for (int ip = 0; ip < 4; ++ip)
      asm("mov.b64 {%0, %1}, %2;" : "=f"(accj[2 * ip]), "=f"(accj[2 * ip + 1]) : "l"(acc2[ip][j]));
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const i64 m = m0 + FFrag<BM, false>::outer(ty, i);
      cold[i] = (!beta_zero && m < p.M) ? p.C[m + n * p.ldc] : 0.f;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const i64 m = m0 + FFrag<BM, false>::outer(ty, i);
      if (m < p.M) p.C[m + n * p.ldc] = beta_zero ? p.alpha * accj[i] : fmaf(p.alpha, accj[i], p.beta * cold[i]);
    }
  }
}

template <int BM, int BN, int STAGES, bool TA, bool TB, int VA, int VB, int BK = kBK>
void launch_cfg2(const GemmParams<float>& p, cudaStream_t s) {
  // the checker instantiation only for the vectorised copies (RECTRI_CU_RING_CHECK)
  constexpr bool kCk = VA == 4 && VB == 4;
  auto kern = kCk && p.ring_check ? sgemm_ffma2_kernel<BM, BN, STAGES, TA, TB, VA, VB, BK, kCk>
                                  : sgemm_ffma2_kernel<BM, BN, STAGES, TA, TB, VA, VB, BK>;
  constexpr int smem = STAGES * BK * (BM + BN + 2 * kPadMC) * static_cast<int>(sizeof(float));
  set_smem(kern, smem);
  dim3 grid(static_cast<unsigned>(ceil_div(p.M, BM)), static_cast<unsigned>(ceil_div(p.N, BN)));
  launch_kernel(kern, grid, 256, smem, s, p);
  ++launch_counter();
}

template <int BM, int BN, int STAGES, bool TA, bool TB, int VA, int VB>
void launch_cfg(const GemmParams<float>& p, cudaStream_t s) {
  auto kern = sgemm_ffma_kernel<BM, BN, STAGES, TA, TB, VA, VB>;
  constexpr int smem =
      STAGES * (FLayout<BM, TA>::ELEMS + FLayout<BN, !TB>::ELEMS) * static_cast<int>(sizeof(float));
  set_smem(kern, smem);
  dim3 grid(static_cast<unsigned>(ceil_div(p.M, BM)), static_cast<unsigned>(ceil_div(p.N, BN)));
  launch_kernel(kern, grid, (BM / 8) * (BN / 8), smem, s, p);
  ++launch_counter();
}

bool aligned(const void* ptr, unsigned b) { return (reinterpret_cast<uintptr_t>(ptr) & (b - 1)) == 0; }

// Copy width per operand: outer-contiguous sources use 16-byte chunks when
// 16-byte aligned (else 4-byte); k-contiguous sources use 8-byte chunks when
// 8-byte aligned (else 4-byte).
template <int BM, int BN, int STAGES>
void dispatch(const GemmParams<float>& p, bool ta, bool tb, cudaStream_t s) {
  const bool a_kc = ta, b_kc = !tb;
  const bool va = a_kc ? (aligned(p.A, 8) && p.lda % 2 == 0) : (aligned(p.A, 16) && p.lda % 4 == 0);
  const bool vb = b_kc ? (aligned(p.B, 8) && p.ldb % 2 == 0) : (aligned(p.B, 16) && p.ldb % 4 == 0);
#define RECTRI_CFG(TA_, TB_)                                                              \
  if (ta == TA_ && tb == TB_) {                                                           \
    constexpr int WA = TA_ ? 2 : 4, WB = TB_ ? 4 : 2;                                     \
    if (va && vb) launch_cfg<BM, BN, STAGES, TA_, TB_, WA, WB>(p, s);                     \
    else if (va) launch_cfg<BM, BN, STAGES, TA_, TB_, WA, 1>(p, s);                       \
    else if (vb) launch_cfg<BM, BN, STAGES, TA_, TB_, 1, WB>(p, s);                       \
    else launch_cfg<BM, BN, STAGES, TA_, TB_, 1, 1>(p, s);                                \
    return;                                                                               \
  }
  RECTRI_CFG(false, false)
  RECTRI_CFG(true, false)
  RECTRI_CFG(false, true)
  RECTRI_CFG(true, true)
#undef RECTRI_CFG
}

// v2: only outer-contiguous sources have a copy width (16-byte chunks when
// 16-byte aligned); k-contiguous sources are always copied 4 bytes at a time.
template <int BM, int BN, int STAGES, int BK = kBK>
void dispatch2(const GemmParams<float>& p, bool ta, bool tb, cudaStream_t s) {
  const bool va = ta || (aligned(p.A, 16) && p.lda % 4 == 0);
  const bool vb = !tb || (aligned(p.B, 16) && p.ldb % 4 == 0);
#define RECTRI_CFG2(TA_, TB_)                                                             \
  if (ta == TA_ && tb == TB_) {                                                           \
    if (va && vb) launch_cfg2<BM, BN, STAGES, TA_, TB_, 4, 4, BK>(p, s);                  \
    else if (va) launch_cfg2<BM, BN, STAGES, TA_, TB_, 4, 1, BK>(p, s);                   \
    else if (vb) launch_cfg2<BM, BN, STAGES, TA_, TB_, 1, 4, BK>(p, s);                   \
    else launch_cfg2<BM, BN, STAGES, TA_, TB_, 1, 1, BK>(p, s);                           \
    return;                                                                               \
  }
  RECTRI_CFG2(false, false)
  RECTRI_CFG2(true, false)
  RECTRI_CFG2(false, true)
  RECTRI_CFG2(true, true)
#undef RECTRI_CFG2
}

int sgemm_version() {
  const char* e = getenv("RECTRI_CU_SGEMM");
  return e && atoi(e) == 1 ? 1 : 2;
}

}  // namespace

void launch_gemm_f32(const GemmParams<float>& p0, bool ta, bool tb, cudaStream_t s) {
  if (p0.M <= 0 || p0.N <= 0 || p0.K <= 0) return;
  GemmParams<float> p = p0;
  p.ring_check = leaf_ring_check_counter(&p.ring_plant);  // RECTRI_CU_RING_CHECK (v2 kernels)
  if (tf32x3_enabled() && launch_gemm_f32_tf32x3(p, ta, tb, s)) return;
  // k-tile depth: 32 for op-N A (fewer barriers; NN +2 %, NT +5 % at
  // 8192x16384x8192), 16 for op-T A (two transposed operands at 32 spill).
  // RECTRI_CU_SGEMM_BK = 16 / 32 forces one.  Results do not depend on it.
  const char* e = getenv("RECTRI_CU_SGEMM_BK");
  const int forced = e ? atoi(e) : 0;
  const int bk = forced == 16 || forced == 32 ? forced : (ta ? 16 : 32);
  // 128 x 256 tiles (8 x 16 per thread, one CTA per SM) for updates with at
  // least a wave of them: +3-8 % on the long updates (fewer shared
  // wavefronts per FMA), but a quarter of the 128 x 128 CTAs per SM slot
  // would starve the short ones (fp32 TRSM n = 4096 1925 -> 2105 us if
  // forced everywhere).  Threshold sweep 592 / 444 / 296 / 148 tiles: 148
  // best (n = 8192 -1 %, 16384 -0.5 %, smaller n unchanged).
  // RECTRI_CU_SGEMM_WIDE = 0 / 1 forces it off / on.
  const char* w = getenv("RECTRI_CU_SGEMM_WIDE");
  const i64 wide_tiles = ceil_div(p.M, 128) * ceil_div(p.N, 256);
  const char* wm = getenv("RECTRI_CU_SGEMM_WIDE_MIN");  // tuning: tile-count threshold
  const bool wide = w ? atoi(w) == 1 : wide_tiles >= (wm ? atoll(wm) : 148);
  if (sgemm_version() == 2 && wide && bk == 32) dispatch2<128, 256, 3, 32>(p, ta, tb, s);
  else if (sgemm_version() == 2 && wide) dispatch2<128, 256, 3>(p, ta, tb, s);
  else if (sgemm_version() == 2 && bk == 32) dispatch2<128, 128, 3, 32>(p, ta, tb, s);
  else if (sgemm_version() == 2) dispatch2<128, 128, 3>(p, ta, tb, s);
  else dispatch<128, 128, 3>(p, ta, tb, s);
}

}  // namespace rectri_cu
