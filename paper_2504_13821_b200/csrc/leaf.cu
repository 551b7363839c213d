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

// Off-diagonal block-row GEMM: acc(block I) += sign * Ls(32 x 32) * panel(block J).
// fp64: warp w owns the m8n8 tiles (w & 3, 2*(w >> 2) + e), e = 0, 1.
struct GemmPart64 {
  double c[2][2];
  int mt, nt0, g, t;
  __device__ void init(int lane, int warp) {
    g = lane >> 2;
    t = lane & 3;
    mt = warp & 3;
    nt0 = 2 * (warp >> 2);
  }
  __device__ void load(const double* panel, int r0) {
#pragma unroll
    for (int e = 0; e < 2; ++e)
#pragma unroll
      for (int h = 0; h < 2; ++h)
        c[e][h] = panel[Layout<double>::panel(r0 + 8 * mt + g, 8 * (nt0 + e) + 2 * t + h)];
  }
  __device__ void zero() {
#pragma unroll
    for (int e = 0; e < 2; ++e) c[e][0] = c[e][1] = 0.0;
  }
  __device__ void mma(const double* ls, const double* panel, int j0, double sign) {
#pragma unroll
    for (int kk = 0; kk < kRB / 4; ++kk) {
      const int k = 4 * kk + t;
      const double a = ls[swz64(k, 8 * mt + g, kRB)];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const double b = sign * panel[Layout<double>::panel(j0 + k, 8 * (nt0 + e) + g)];
        dmma884(c[e][0], c[e][1], a, b);
      }
    }
  }
  __device__ void store(double* dst, int r0) const {
#pragma unroll
    for (int e = 0; e < 2; ++e)
#pragma unroll
      for (int h = 0; h < 2; ++h)
        dst[Layout<double>::panel(r0 + 8 * mt + g, 8 * (nt0 + e) + 2 * t + h)] = c[e][h];
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
  __device__ void load(const float* panel, int r0) {
#pragma unroll
    for (int i = 0; i < 4; ++i) c[i] = panel[Layout<float>::panel(r0 + 4 * w + i, lane)];
  }
  __device__ void zero() {
#pragma unroll
    for (int i = 0; i < 4; ++i) c[i] = 0.f;
  }
  __device__ void mma(const float* ls, const float* panel, int j0, float sign) {
#pragma unroll 8
    for (int k = 0; k < kRB; ++k) {
      const float b = sign * panel[Layout<float>::panel(j0 + k, lane)];
      const float4 a = *reinterpret_cast<const float4*>(ls + k * kRB + 4 * w);
      c[0] = fmaf(a.x, b, c[0]);
      c[1] = fmaf(a.y, b, c[1]);
      c[2] = fmaf(a.z, b, c[2]);
      c[3] = fmaf(a.w, b, c[3]);
    }
  }
  __device__ void store(float* dst, int r0) const {
#pragma unroll
    for (int i = 0; i < 4; ++i) dst[Layout<float>::panel(r0 + 4 * w + i, lane)] = c[i];
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

template <typename T>
struct LeafSmem {
  static constexpr int panel = kLeafMax * Layout<T>::kPanelStride;
  static constexpr int blk = kRB * kRB;
  static constexpr int ys = kRB * Layout<T>::kPanelStride;
  static constexpr int total = panel + 3 * blk + ys + kLeafMax;
};

template <typename T>
__global__ void __launch_bounds__(kThreads) leaf_kernel(const LeafParams<T> p) {
  using L = Layout<T>;
  extern __shared__ __align__(128) unsigned char leaf_smem[];
  T* panel = reinterpret_cast<T*>(leaf_smem);
  T* ls = panel + LeafSmem<T>::panel;  // two staged off-diagonal blocks of L'
  T* ld = ls + 2 * LeafSmem<T>::blk;   // diagonal block, ld[p * 32 + r] = L'(r, p), p < r
  T* ys = ld + LeafSmem<T>::blk;       // TRMM off-diagonal partial sums
  T* dg = ys + LeafSmem<T>::ys;        // TRSM: 1 / d_r; TRMM: d_r (1 for Unit)

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n = p.n;
  const int nblk = (n + kRB - 1) / kRB;
  const int rows_p = nblk * kRB;
  const i64 c0 = static_cast<i64>(blockIdx.x) * kNC;
  const int ncols = static_cast<int>(min(static_cast<i64>(kNC), p.nrhs - c0));

  auto gaddr = [&](int r, int c) -> i64 {  // global offset of B'(r, c0 + c)
    const i64 sr = p.reflected ? n - 1 - r : r;
    return p.right ? sr * p.ldb + c0 + c : (c0 + c) * p.ldb + sr;
  };
  // Panel element assignment: Left -> each warp covers 4 rows x 8 rhs
  // (32-byte global sectors); Right -> each warp covers 32 rhs of one row.
  auto panel_rc = [&](int q, int& r, int& c) {
    if (p.right) {
      r = q / kNC;
      c = q % kNC;
    } else {
      const int w = q >> 5, l = q & 31;
      const int row_tiles = rows_p / 4;
      r = 4 * (w % row_tiles) + (l & 3);
      c = 8 * (w / row_tiles) + (l >> 2);
    }
  };

  // TRMM with alpha == 0 writes zeros without reading B (base_kernels.cpp:143-150).
  if (!p.trsm && p.alpha == T(0)) {
    for (int q = tid; q < rows_p * kNC; q += kThreads) {
      int r, c;
      panel_rc(q, r, c);
      if (r < n && c < ncols) p.B[gaddr(r, c)] = T(0);
    }
    return;
  }

  // 1. Panel load.
  for (int q = tid; q < rows_p * kNC; q += kThreads) {
    int r, c;
    panel_rc(q, r, c);
    const bool ok = r < n && c < ncols;
    cp_async_elem(panel + L::panel(r, c), ok ? p.B + gaddr(r, c) : p.B, ok);
  }
  cp_async_commit();
  for (int r = tid; r < rows_p; r += kThreads) {
    T d = T(1);
    if (r < n && !p.unit) {
      const i64 sr = p.reflected ? n - 1 - r : r;
      d = p.A[sr + sr * p.lda];
    }
    dg[r] = p.trsm ? T(1) / d : d;
  }

  // Staging of a 32x32 block of L' (rows r0.., k-columns j0..) with
  // masking: entries with j >= r (diagonal block) or outside n are zero.
  // Each warp copies 4 k-columns x 8 rows per step.
  auto stage_block = [&](T* dst, int r0, int j0, bool diag) {
#pragma unroll
    for (int it = 0; it < kRB * kRB / kThreads; ++it) {
      const int q = tid + it * kThreads;
      const int w = q >> 5, l = q & 31;
      int r, j;
      if (diag) {  // row pattern (conflict-free for the [p][r] layout)
        r = l;
        j = w;
      } else {
        r = 8 * (w & 3) + (l >> 2);
        j = 4 * (w >> 2) + (l & 3);
      }
      const int gr = r0 + r, gj = j0 + j;
      const bool ok = gr < n && (diag ? j < r : true);
      T* s = diag ? dst + j * kRB + r : dst + L::lblk(r, j);
      cp_async_elem(s, ok ? lprime_ptr(p, gr, gj) : p.A, ok);
    }
  };

  cp_async_wait<0>();
  __syncthreads();
  if (p.trsm && p.alpha != T(1)) {  // x = alpha * b (base_kernels.cpp:76-77)
    for (int q = tid; q < rows_p * kNC; q += kThreads) {
      int r, c;
      panel_rc(q, r, c);
      panel[L::panel(r, c)] *= p.alpha;
    }
    __syncthreads();
  }

  typename GemmPartOf<T>::type gp;
  gp.init(lane, warp);
  const T sign = p.trsm ? T(-1) : T(1);
  // Diagonal-part thread roles: column cc, row group gq (rows gq + 8q).
  const int cc = warp * 4 + (lane >> 3);
  const int gq = lane & 7;

  for (int step = 0; step < nblk; ++step) {
    const int I = p.trsm ? step : nblk - 1 - step;  // TRMM runs bottom-up (in place)
    const int r0 = I * kRB;

    // Prefetch: the diagonal block, then the first off-diagonal block.
    stage_block(ld, r0, r0, true);
    cp_async_commit();
    if (I > 0) {
      stage_block(ls, r0, 0, false);
      cp_async_commit();
    }

    // 2. Off-diagonal block-row GEMM, block J+1 in flight while J multiplies.
    if (p.trsm) gp.load(panel, r0);
    else gp.zero();
    for (int J = 0; J < I; ++J) {
      if (J + 1 < I) {
        stage_block(ls + ((J + 1) & 1) * LeafSmem<T>::blk, r0, (J + 1) * kRB, false);
        cp_async_commit();
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncthreads();
      gp.mma(ls + (J & 1) * LeafSmem<T>::blk, panel, J * kRB, sign);
      __syncthreads();
    }
    if (p.trsm) gp.store(panel, r0);
    else gp.store(ys, 0);
    cp_async_wait<0>();
    __syncthreads();

    // 3. Diagonal block.
    T v[4];
    if (p.trsm) {
#pragma unroll
      for (int q = 0; q < 4; ++q) v[q] = panel[L::panel(r0 + gq + 8 * q, cc)];
#pragma unroll
      for (int pp = 0; pp < kRB; ++pp) {
        const int qo = pp >> 3, go = pp & 7;
        T x = T(0);
        if (gq == go) {
          v[qo] = v[qo] * dg[r0 + pp];
          x = v[qo];
        }
        x = __shfl_sync(0xffffffffu, x, (lane & ~7) | go);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int r = gq + 8 * q;
          if (r > pp) v[q] = fma(-ld[pp * kRB + r], x, v[q]);
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) panel[L::panel(r0 + gq + 8 * q, cc)] = v[q];
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) v[q] = ys[L::panel(gq + 8 * q, cc)];
#pragma unroll 8
      for (int pp = 0; pp < kRB; ++pp) {
        const T b = panel[L::panel(r0 + pp, cc)];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int r = gq + 8 * q;
          if (pp < r) v[q] = fma(ld[pp * kRB + r], b, v[q]);
          else if (pp == r) v[q] = fma(dg[r0 + r], b, v[q]);
        }
      }
      __syncwarp();  // all readers of column cc live in this warp
#pragma unroll
      for (int q = 0; q < 4; ++q) panel[L::panel(r0 + gq + 8 * q, cc)] = p.alpha * v[q];
    }
    __syncthreads();
  }

  // 4. Write back.
  for (int q = tid; q < rows_p * kNC; q += kThreads) {
    int r, c;
    panel_rc(q, r, c);
    if (r < n && c < ncols) p.B[gaddr(r, c)] = panel[L::panel(r, c)];
  }
}

template <typename T>
void launch_leaf(const LeafParams<T>& p, cudaStream_t s) {
  if (p.n <= 0 || p.nrhs <= 0) return;
  const int smem = static_cast<int>(LeafSmem<T>::total * sizeof(T));
  cudaFuncSetAttribute(leaf_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const unsigned grid = static_cast<unsigned>(ceil_div(p.nrhs, kNC));
  leaf_kernel<T><<<grid, kThreads, smem, s>>>(p);
  ++launch_counter();
}

}  // namespace

void launch_leaf_f64(const LeafParams<double>& p, cudaStream_t s) { launch_leaf<double>(p, s); }
void launch_leaf_f32(const LeafParams<float>& p, cudaStream_t s) { launch_leaf<float>(p, s); }

}  // namespace rectri_cu
