// leaf.cu -- the base (leaf) kernels trsm_base / trmm_base on sm_100a.
//
// Replaces src/base_kernels.cpp:94-177 (trsm_left_lower, trmm_left, and the
// Right-as-transposed-Left reduction of :35-47, :152-155, :172-176).
//
// Every variant is reduced, as in the reference, to the Left form on a
// virtual lower-triangular factor L' with reflected row indices
// (SURVEY.md 3.6).  One CTA owns kNC right-hand sides for the whole tile:
//   1. the B panel (n x kNC) is copied once into shared memory with cp.async
//      (each warp covers 4 rows x 8 right-hand sides: 32-byte sectors from
//      global, conflict-free in shared memory);
//   2. the tile is walked in 32-row blocks.  The off-diagonal part of a block
//      row is a small GEMM against already-final blocks (DMMA m8n8k4 for fp64,
//      FFMA for fp32); the 32x32 blocks of L' are streamed by cp.async into a
//      double buffer, block J+1 in flight while block J is multiplied, and the
//      diagonal block is prefetched underneath the whole GEMM part;
//   3. the 32x32 diagonal block is applied by 8 lanes per right-hand side,
//      4 rows each, broadcasting each resolved value with a warp shuffle
//      (TRSM: forward substitution with the reciprocal diagonal; TRMM: the
//      masked lower-triangular product);
//   4. the panel is written back once.
// Entries outside the stored triangle are never loaded: masked positions are
// zero-filled by cp.async (src-size 0) and the diagonal block's strict upper
// half is skipped by predicate, so NaN there never reaches the output
// (test_recursion.cpp:304-326).  Unit diagonals are never read.
// The per-element arithmetic order depends only on the tile, never on the
// number of right-hand sides, so results are bitwise independent of how the
// right-hand sides are sharded.
#include <cstdlib>

#include "common.cuh"
#include "launch.h"

namespace rectri_cu {
namespace {

constexpr int kRB = 32;        // row block
constexpr int kNC = 32;        // right-hand sides per CTA
constexpr int kThreads = 256;  // 8 warps

template <typename T>
struct Layout;

// fp64: panel rows of kNC doubles with the 16-byte-chunk XOR swizzle (DMMA
// fragment reads, 4x8 sub-tile copies and the 8-lane diagonal pattern are all
// conflict-free); staged L' blocks k-major with the same swizzle.
template <>
struct Layout<double> {
  static constexpr int kPanelStride = kNC;
  __device__ static int panel(int r, int c) { return swz64(r, c, kNC); }
  __device__ static int lblk(int r, int j) { return swz64(j, r, kRB); }
};
// fp32: panel rows padded to 33 floats (row-wise and column-wise lane
// patterns both conflict-free); staged L' blocks k-major, rows contiguous
// (float4 broadcast reads).
template <>
struct Layout<float> {
  static constexpr int kPanelStride = kNC + 1;
  __device__ static int panel(int r, int c) { return r * (kNC + 1) + c; }
  __device__ static int lblk(int r, int j) { return j * kRB + r; }
};

// One element by cp.async; `ok == false` zero-fills (src-size 0) and the
// caller passes a valid base address that is not read.
template <typename T>
__device__ __forceinline__ void cp_async_elem(T* dst, const T* src, bool ok) {
  if constexpr (sizeof(T) == 8)
    cp_async8(dst, src, ok ? 8 : 0);
  else
    cp_async4(dst, src, ok ? 4 : 0);
}

template <typename T>
__device__ __forceinline__ const T* lprime_ptr(const LeafParams<T>& p, int r, int j) {
  const int rr = p.reflected ? p.n - 1 - r : r;
  const int jj = p.reflected ? p.n - 1 - j : j;
  const i64 row = p.swapped ? jj : rr;
  const i64 col = p.swapped ? rr : jj;
  return p.A + row + col * p.lda;
}

// Off-diagonal block-row GEMM: acc(block I) += Ls(32 x 32) * panel(block J).
// TRSM accumulates the NEGATED right-hand side (acc = -b + sum L'x) and
// negates on store: with round-to-nearest every intermediate is the exact
// negation of the b - sum L'x chain, so no per-element sign is needed.
// fp64: warp w owns the m8n8 tiles (w & 3, 2*(w >> 2) + e), e = 0, 1;
// fragment addresses are fixed per thread (row & 3 is invariant).
struct GemmPart64 {
  double c[2][2];
  int mt, nt0, g, t;
  uint32_t a_base, b_base[2];  // shared byte offsets for k-step 0
  __device__ void init(int lane, int warp) {
    g = lane >> 2;
    t = lane & 3;
    mt = warp & 3;
    nt0 = 2 * (warp >> 2);
    a_base = 8u * static_cast<uint32_t>(swz64(t, 8 * mt + g, kRB));
#pragma unroll
    for (int e = 0; e < 2; ++e) b_base[e] = 8u * static_cast<uint32_t>(swz64(t, 8 * (nt0 + e) + g, kNC));
  }
  __device__ void load(const double* panel, int r0, bool negate) {
#pragma unroll
    for (int e = 0; e < 2; ++e)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const double x = panel[Layout<double>::panel(r0 + 8 * mt + g, 8 * (nt0 + e) + 2 * t + h)];
        c[e][h] = negate ? -x : x;
      }
  }
  __device__ void zero() {
#pragma unroll
    for (int e = 0; e < 2; ++e) c[e][0] = c[e][1] = 0.0;
  }
  // ls_u32 / panel_u32: shared addresses of the staged block and the panel.
  __device__ void mma(uint32_t ls_u32, uint32_t panel_u32, int j0) {
    double a[2], b[2][2];
    const uint32_t pb = panel_u32 + static_cast<uint32_t>(j0 * kNC * 8);
    auto ld = [&](int buf, int kk) {
      asm volatile("ld.shared.f64 %0, [%1];" : "=d"(a[buf]) : "r"(ls_u32 + a_base + kk * 4 * kRB * 8));
#pragma unroll
      for (int e = 0; e < 2; ++e)
        asm volatile("ld.shared.f64 %0, [%1];" : "=d"(b[buf][e]) : "r"(pb + b_base[e] + kk * 4 * kNC * 8));
    };
    ld(0, 0);
#pragma unroll
    for (int kk = 0; kk < kRB / 4; ++kk) {
      if (kk + 1 < kRB / 4) ld((kk + 1) & 1, kk + 1);
#pragma unroll
      for (int e = 0; e < 2; ++e) dmma884(c[e][0], c[e][1], a[kk & 1], b[kk & 1][e]);
    }
  }
  __device__ void store(double* dst, int r0, bool negate) const {
#pragma unroll
    for (int e = 0; e < 2; ++e)
#pragma unroll
      for (int h = 0; h < 2; ++h)
        dst[Layout<double>::panel(r0 + 8 * mt + g, 8 * (nt0 + e) + 2 * t + h)] = negate ? -c[e][h] : c[e][h];
  }
};

// fp32: lane = right-hand side, warp w owns rows 4w .. 4w+3 of the block.
struct GemmPart32 {
  float c[4];
  int lane, w;
  __device__ void init(int lane_, int warp) {
    lane = lane_;
    w = warp;
  }
  __device__ void load(const float* panel, int r0, bool negate) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float x = panel[Layout<float>::panel(r0 + 4 * w + i, lane)];
      c[i] = negate ? -x : x;
    }
  }
  __device__ void zero() {
#pragma unroll
    for (int i = 0; i < 4; ++i) c[i] = 0.f;
  }
  __device__ void mma(uint32_t ls_u32, uint32_t panel_u32, int j0) {
    const float* ls = reinterpret_cast<const float*>(__cvta_shared_to_generic(ls_u32));
    const float* panel = reinterpret_cast<const float*>(__cvta_shared_to_generic(panel_u32));
#pragma unroll 8
    for (int k = 0; k < kRB; ++k) {
      const float b = panel[Layout<float>::panel(j0 + k, lane)];
      const float4 a = *reinterpret_cast<const float4*>(ls + k * kRB + 4 * w);
      c[0] = fmaf(a.x, b, c[0]);
      c[1] = fmaf(a.y, b, c[1]);
      c[2] = fmaf(a.z, b, c[2]);
      c[3] = fmaf(a.w, b, c[3]);
    }
  }
  __device__ void store(float* dst, int r0, bool negate) const {
#pragma unroll
    for (int i = 0; i < 4; ++i) dst[Layout<float>::panel(r0 + 4 * w + i, lane)] = negate ? -c[i] : c[i];
  }
};

template <typename T>
struct GemmPartOf;
template <>
struct GemmPartOf<double> {
  using type = GemmPart64;
};
template <>
struct GemmPartOf<float> {
  using type = GemmPart32;
};

constexpr int kRing = 4;  // depth of the staged-block ring

template <typename T>
struct LeafSmem {
  static constexpr int panel = kLeafMax * Layout<T>::kPanelStride;
  static constexpr int blk = kRB * kRB;
  static constexpr int ys = kRB * Layout<T>::kPanelStride;
  static constexpr int total = panel + kRing * blk + ys + kLeafMax;
};

// The blocks of L' a CTA consumes, in order: for each row block I (ascending
// for TRSM, descending for TRMM) its off-diagonal blocks J = 0 .. I-1, then
// its diagonal block (J == I).
struct SeqCursor {
  int I, J, nblk;
  bool asc;
  __device__ void start(int nblk_, bool asc_) {
    nblk = nblk_;
    asc = asc_;
    I = asc ? 0 : nblk - 1;
    J = 0;
  }
  __device__ void next() {
    if (J < I) {
      ++J;
    } else {
      I += asc ? 1 : -1;
      J = 0;
    }
  }
};

template <typename T>
__global__ void __launch_bounds__(kThreads) leaf_kernel(const LeafParams<T> p) {
  using L = Layout<T>;
  extern __shared__ __align__(128) unsigned char leaf_smem[];
  T* panel = reinterpret_cast<T*>(leaf_smem);
  T* ring = panel + LeafSmem<T>::panel;          // kRing staged 32x32 blocks of L'
  T* ys = ring + kRing * LeafSmem<T>::blk;       // TRMM off-diagonal partial sums
  T* dg = ys + LeafSmem<T>::ys;                  // TRSM: 1 / d_r; TRMM: d_r (1 for Unit)

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n = p.n;
  const int nblk = (n + kRB - 1) / kRB;
  const int rows_p = nblk * kRB;
  const i64 c0 = static_cast<i64>(blockIdx.x) * kNC;
  const int ncols = static_cast<int>(min(static_cast<i64>(kNC), p.nrhs - c0));
  const bool asc = p.trsm != 0;  // TRMM runs bottom-up (in place)

  // Visits every panel element (r < rows_p, c < kNC) once per thread set,
  // with its global pointer (valid only when r < n && c < ncols):
  //   Left  -> each warp covers 4 rows x 8 right-hand sides (32-byte global
  //            sectors); the thread's 4 column pointers are fixed.
  //   Right -> each warp covers the 32 right-hand sides of one row.
  // No divisions, no 64-bit multiplies per element.
  const i64 rstep = p.reflected ? -1 : 1;  // global row step for r -> r + 1 (Left)
  auto for_panel = [&](auto&& f) {
    if (!p.right) {
      const int rl = lane & 3, cl = lane >> 2;
#pragma unroll
      for (int cg = 0; cg < kNC / 8; ++cg) {
        const int c = 8 * cg + cl;
        const T* colp = p.B + (c0 + c) * p.ldb + (p.reflected ? n - 1 : 0);
        for (int rt = warp; rt < rows_p / 4; rt += kThreads / 32) {
          const int r = 4 * rt + rl;
          f(r, c, colp + r * rstep);
        }
      }
    } else {
      const int c = lane;
      for (int r = warp; r < rows_p; r += kThreads / 32) {
        const i64 sr = p.reflected ? n - 1 - r : r;
        f(r, c, p.B + sr * p.ldb + c0 + c);
      }
    }
  };

  // TRMM with alpha == 0 writes zeros without reading B (base_kernels.cpp:143-150).
  if (!p.trsm && p.alpha == T(0)) {
    for_panel([&](int r, int c, const T* g) {
      if (r < n && c < ncols) *const_cast<T*>(g) = T(0);
    });
    return;
  }

  // Staging of a block of L' into a ring slot.  L'(r, j) is affine in the
  // thread's local (r, j): address = base(I, J) + sgn * (r_l * sr + j_l * sj)
  // with strides +-1 / +-lda, so each thread's 4 element offsets are
  // computed once.  Off-diagonal blocks are stored k-major for the GEMM part
  // (each warp copies 4 k x 8 rows); the diagonal block as [p][r] = L'(r, p)
  // for p < r, zero elsewhere.  Masked entries are zero-filled (never read).
  constexpr int kPer = kRB * kRB / kThreads;  // elements per thread per block
  const i64 sr = p.swapped ? p.lda : 1, sj = p.swapped ? 1 : p.lda;
  const i64 sgn = p.reflected ? -1 : 1;
  i64 off_o[kPer], off_d[kPer];
  int so_o[kPer], so_d[kPer];  // shared element offsets within a slot
  int rl_o[kPer], rl_d[kPer];
  bool lower_d[kPer];
#pragma unroll
  for (int it = 0; it < kPer; ++it) {
    const int q = tid + it * kThreads;
    const int w = q >> 5, l = q & 31;
    int r = 8 * (w & 3) + (l >> 2), j = 4 * (w >> 2) + (l & 3);
    off_o[it] = sgn * (r * sr + j * sj);
    so_o[it] = L::lblk(r, j);
    rl_o[it] = r;
    r = l;
    j = w;
    off_d[it] = sgn * (r * sr + j * sj);
    so_d[it] = j * kRB + r;
    rl_d[it] = r;
    lower_d[it] = j < r;
  }
  auto stage = [&](int I, int J, int slot) {
    T* dst = ring + slot * LeafSmem<T>::blk;
    const int r0 = I * kRB, j0 = J * kRB;
    const i64 rr = p.reflected ? n - 1 - r0 : r0;
    const i64 jj = p.reflected ? n - 1 - j0 : j0;
    const T* base = p.A + rr * sr + jj * sj;
    if (I != J) {
#pragma unroll
      for (int it = 0; it < kPer; ++it) {
        const bool ok = r0 + rl_o[it] < n;
        cp_async_elem(dst + so_o[it], ok ? base + off_o[it] : p.A, ok);
      }
    } else {
#pragma unroll
      for (int it = 0; it < kPer; ++it) {
        const bool ok = lower_d[it] && r0 + rl_d[it] < n;
        cp_async_elem(dst + so_d[it], ok ? base + off_d[it] : p.A, ok);
      }
    }
  };

  // 1. Panel load + the first ring elements (one commit group each).
  for_panel([&](int r, int c, const T* g) {
    const bool ok = r < n && c < ncols;
    cp_async_elem(panel + L::panel(r, c), ok ? g : p.B, ok);
  });
  cp_async_commit();
  const int nseq = nblk * (nblk + 1) / 2;
  SeqCursor prod, cons;  // producer runs kRing - 1 elements ahead
  prod.start(nblk, asc);
  cons.start(nblk, asc);
#pragma unroll
  for (int s = 0; s < kRing - 1; ++s) {
    if (s < nseq) {
      stage(prod.I, prod.J, s % kRing);
      prod.next();
    }
    cp_async_commit();
  }
  for (int r = tid; r < rows_p; r += kThreads) {
    T d = T(1);
    if (r < n && !p.unit) {
      const i64 sr = p.reflected ? n - 1 - r : r;
      d = p.A[sr + sr * p.lda];
    }
    dg[r] = p.trsm ? T(1) / d : d;
  }
  cp_async_wait<kRing - 1>();  // the panel group
  __syncthreads();
  if (p.trsm && p.alpha != T(1)) {  // x = alpha * b (base_kernels.cpp:76-77)
    for_panel([&](int r, int c, const T*) { panel[L::panel(r, c)] *= p.alpha; });
  }

  typename GemmPartOf<T>::type gp;
  gp.init(lane, warp);
  const uint32_t panel_u32 = smem_u32(panel);
  const uint32_t ring_u32 = smem_u32(ring);
  // Diagonal-part thread roles: column cc, row group gq (rows gq + 8q).
  const int cc = warp * 4 + (lane >> 3);
  const int gq = lane & 7;
  const bool neg = p.trsm != 0;

  for (int s = 0; s < nseq; ++s, cons.next()) {
    cp_async_wait<kRing - 2>();  // element s has landed (this thread's copies)
    __syncthreads();              // ... everyone's; slot (s-1) % kRing is free
    if (s + kRing - 1 < nseq) {
      stage(prod.I, prod.J, (s + kRing - 1) % kRing);
      prod.next();
    }
    cp_async_commit();

    const int I = cons.I, J = cons.J;
    const int r0 = I * kRB;
    const uint32_t slot = ring_u32 + static_cast<uint32_t>((s % kRing) * LeafSmem<T>::blk * sizeof(T));
    if (J == 0) {  // first element of row block I: fresh accumulators
      if (p.trsm) gp.load(panel, r0, neg);
      else gp.zero();
    }
    if (J < I) {  // 2. off-diagonal block-row GEMM
      if (p.debug_skip != 2) gp.mma(slot, panel_u32, J * kRB);
      continue;
    }
    // 3. diagonal block (slot holds ld[p * 32 + r] = L'(r, p), p < r).
    const T* ld = ring + (s % kRing) * LeafSmem<T>::blk;
    if (p.trsm) gp.store(panel, r0, neg);
    else gp.store(ys, 0, false);
    // debug_skip == 3 plants a race (missing barrier) for the racecheck
    // negative test (tests/test_gpu_sanitizer.py), cf. the reference's
    // build_trsm_program_missing_barrier (workgroup.cpp:333-349).
    if (p.debug_skip != 3) __syncthreads();
    if (p.debug_skip == 1) continue;
    T v[4];
    if (p.trsm) {
      T rv[4];  // reciprocal diagonal of this thread's rows, off the chain
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        v[q] = panel[L::panel(r0 + gq + 8 * q, cc)];
        rv[q] = dg[r0 + gq + 8 * q];
      }
#pragma unroll
      for (int pp = 0; pp < kRB; ++pp) {
        const int qo = pp >> 3, go = pp & 7;
        T x = T(0);
        if (gq == go) {
          v[qo] = v[qo] * rv[qo];
          x = v[qo];
        }
        x = __shfl_sync(0xffffffffu, x, (lane & ~7) | go);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          // Branch-free: the shared load is unconditional (always in range;
          // zero for r <= pp) so it pipelines; the update is selected, so a
          // masked entry never reaches v even when x is not finite.
          const int r = gq + 8 * q;
          const T nv = fma(-ld[pp * kRB + r], x, v[q]);
          v[q] = r > pp ? nv : v[q];
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) panel[L::panel(r0 + gq + 8 * q, cc)] = v[q];
    } else {
      T dr[4];  // diagonal of this thread's rows (1 for Unit)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        v[q] = ys[L::panel(gq + 8 * q, cc)];
        dr[q] = dg[r0 + gq + 8 * q];
      }
#pragma unroll
      for (int pp = 0; pp < kRB; ++pp) {
        const T b = panel[L::panel(r0 + pp, cc)];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          // Branch-free masked product (see the TRSM loop): p < r uses L',
          // p == r the diagonal, p > r is skipped by selection.
          const int r = gq + 8 * q;
          const T coef = pp == r ? dr[q] : ld[pp * kRB + r];
          const T nv = fma(coef, b, v[q]);
          v[q] = pp <= r ? nv : v[q];
        }
      }
      __syncwarp();  // all readers of column cc live in this warp
#pragma unroll
      for (int q = 0; q < 4; ++q) panel[L::panel(r0 + gq + 8 * q, cc)] = p.alpha * v[q];
    }
  }
  cp_async_wait<0>();
  __syncthreads();

  // 4. Write back.
  for_panel([&](int r, int c, const T* g) {
    if (r < n && c < ncols) *const_cast<T*>(g) = panel[L::panel(r, c)];
  });
}

int leaf_debug() {
  static int v = [] {
    const char* e = getenv("RECTRI_CU_LEAF_DEBUG");
    return e ? atoi(e) : 0;
  }();
  return v;
}

template <typename T>
void launch_leaf(const LeafParams<T>& p_in, cudaStream_t s) {
  if (p_in.n <= 0 || p_in.nrhs <= 0) return;
  LeafParams<T> p = p_in;
  p.debug_skip = leaf_debug();
  const int smem = static_cast<int>(LeafSmem<T>::total * sizeof(T));
  set_smem(leaf_kernel<T>, smem);
  const unsigned grid = static_cast<unsigned>(ceil_div(p.nrhs, kNC));
  leaf_kernel<T><<<grid, kThreads, smem, s>>>(p);
  ++launch_counter();
}

}  // namespace

void launch_leaf_f64_v1(const LeafParams<double>& p, cudaStream_t s) { launch_leaf<double>(p, s); }
void launch_leaf_f32_v1(const LeafParams<float>& p, cudaStream_t s) { launch_leaf<float>(p, s); }

}  // namespace rectri_cu
