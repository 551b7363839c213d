// leaf.cu -- the base (leaf) kernels trsm_base / trmm_base on sm_100a.
//
// Replaces src/base_kernels.cpp:94-177 (trsm_left_lower, trmm_left, and the
// Right-as-transposed-Left reduction of :35-47, :152-155, :172-176).
//
// Every variant is reduced, as in the reference, to the Left form on a
// virtual lower-triangular factor L' with reflected row indices
// (SURVEY.md 3.6).  One CTA owns kNC right-hand sides for the whole tile:
//   1. the B panel (n x kNC) is loaded once into shared memory (coalesced:
//      rows fastest for Left, right-hand sides fastest for Right);
//   2. the tile is walked in 32-row blocks.  The off-diagonal part of each
//      block row is a small GEMM against already-final blocks (DMMA m8n8k4
//      for fp64, FFMA for fp32), staged 32x32 blocks of L' at a time;
//   3. the 32x32 diagonal block is applied by 8 lanes per right-hand side,
//      4 rows each, broadcasting each resolved value with a warp shuffle
//      (TRSM: forward substitution with the reciprocal diagonal; TRMM: the
//      masked lower-triangular product);
//   4. the panel is written back once.
// Entries outside the stored triangle are never loaded: masked positions are
// explicit zeros in shared memory and the diagonal block's strict upper half
// is skipped by predicate, so NaN there never reaches the output
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
struct Smem {
  static constexpr int panel = kLeafMax * kNC;  // B' panel
  static constexpr int blk = kRB * kRB;         // staged L' block / diag block / Y
};

// Panel element (r, c): fp64 uses the conflict-free swizzle for the DMMA
// fragment pattern; fp32 is plain row-major (c contiguous).
__device__ __forceinline__ int pidx(double*, int r, int c) { return swz64(r, c, kNC); }
__device__ __forceinline__ int pidx(float*, int r, int c) { return r * kNC + c; }
// Staged off-diagonal block element (row r of the block, k-index j), k-major.
__device__ __forceinline__ int lidx(double*, int r, int j) { return swz64(j, r, kRB); }
__device__ __forceinline__ int lidx(float*, int r, int j) { return j * kRB + r; }

template <typename T>
__device__ __forceinline__ T load_lprime(const LeafParams<T>& p, int r, int j) {
  const int rr = p.reflected ? p.n - 1 - r : r;
  const int jj = p.reflected ? p.n - 1 - j : j;
  const i64 row = p.swapped ? jj : rr;
  const i64 col = p.swapped ? rr : jj;
  return p.A[row + col * p.lda];
}

// Off-diagonal block-row GEMM: acc(block I) += Ls(32 x 32) * panel(block J).
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
        c[e][h] = panel[swz64(r0 + 8 * mt + g, 8 * (nt0 + e) + 2 * t + h, kNC)];
  }
  __device__ void zero() {
#pragma unroll
    for (int e = 0; e < 2; ++e) c[e][0] = c[e][1] = 0.0;
  }
  __device__ void mma(const double* ls, const double* panel, int j0) {
#pragma unroll
    for (int kk = 0; kk < kRB / 4; ++kk) {
      const int k = 4 * kk + t;
      const double a = ls[swz64(k, 8 * mt + g, kRB)];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const double b = panel[swz64(j0 + k, 8 * (nt0 + e) + g, kNC)];
        dmma884(c[e][0], c[e][1], a, b);
      }
    }
  }
  // Stores the block into a 32 x kNC destination laid out like the panel.
  __device__ void store(double* dst, int r0) const {
#pragma unroll
    for (int e = 0; e < 2; ++e)
#pragma unroll
      for (int h = 0; h < 2; ++h)
        dst[swz64(r0 + 8 * mt + g, 8 * (nt0 + e) + 2 * t + h, kNC)] = c[e][h];
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
    for (int i = 0; i < 4; ++i) c[i] = panel[(r0 + 4 * w + i) * kNC + lane];
  }
  __device__ void zero() {
#pragma unroll
    for (int i = 0; i < 4; ++i) c[i] = 0.f;
  }
  __device__ void mma(const float* ls, const float* panel, int j0) {
#pragma unroll 8
    for (int k = 0; k < kRB; ++k) {
      const float b = panel[(j0 + k) * kNC + lane];
      const float4 a = *reinterpret_cast<const float4*>(ls + k * kRB + 4 * w);
      c[0] = fmaf(a.x, b, c[0]);
      c[1] = fmaf(a.y, b, c[1]);
      c[2] = fmaf(a.z, b, c[2]);
      c[3] = fmaf(a.w, b, c[3]);
    }
  }
  __device__ void store(float* dst, int r0) const {
#pragma unroll
    for (int i = 0; i < 4; ++i) dst[(r0 + 4 * w + i) * kNC + lane] = c[i];
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
__global__ void __launch_bounds__(kThreads) leaf_kernel(const LeafParams<T> p) {
  extern __shared__ __align__(128) unsigned char leaf_smem[];
  T* panel = reinterpret_cast<T*>(leaf_smem);
  T* ls = panel + Smem<T>::panel;  // staged (signed) off-diagonal block of L'
  T* ld = ls + Smem<T>::blk;       // diagonal block, [p][r]
  T* ys = ld + Smem<T>::blk;       // TRMM off-diagonal partial sums
  T* rinv = ys + Smem<T>::blk;     // TRSM reciprocal diagonal

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

  // TRMM with alpha == 0 writes zeros without reading B (base_kernels.cpp:143-150).
  if (!p.trsm && p.alpha == T(0)) {
    for (int q = tid; q < n * kNC; q += kThreads) {
      const int r = p.right ? q / kNC : q % n;
      const int c = p.right ? q % kNC : q / n;
      if (c < ncols) p.B[gaddr(r, c)] = T(0);
    }
    return;
  }

  // 1. Panel load (TRSM folds alpha in here: x = alpha * b, base_kernels.cpp:76-77).
  for (int q = tid; q < rows_p * kNC; q += kThreads) {
    const int r = p.right ? q / kNC : q % rows_p;
    const int c = p.right ? q % kNC : q / rows_p;
    T v = T(0);
    if (r < n && c < ncols) {
      v = p.B[gaddr(r, c)];
      if (p.trsm) v = p.alpha * v;
    }
    panel[pidx(panel, r, c)] = v;
  }
  if (p.trsm) {
    for (int r = tid; r < rows_p; r += kThreads) {
      T d = T(1);
      if (r < n && !p.unit) {
        const i64 sr = p.reflected ? n - 1 - r : r;
        d = p.A[sr + sr * p.lda];
      }
      rinv[r] = T(1) / d;
    }
  }
  __syncthreads();

  typename GemmPartOf<T>::type gp;
  gp.init(lane, warp);
  // Diagonal-part thread roles: column cc, row group gq (rows gq + 8q).
  const int cc = warp * 4 + (lane >> 3);
  const int gq = lane & 7;

  for (int step = 0; step < nblk; ++step) {
    const int I = p.trsm ? step : nblk - 1 - step;  // TRMM runs bottom-up (in place)
    const int r0 = I * kRB;

    // 2. Off-diagonal block-row GEMM.
    if (p.trsm) gp.load(panel, r0);
    else gp.zero();
    for (int J = 0; J < I; ++J) {
      for (int q = tid; q < kRB * kRB; q += kThreads) {
        // Walk the contiguous direction of A with consecutive threads.
        const int fast = q & (kRB - 1), slow = q >> 5;
        const int r = p.swapped ? slow : fast, j = p.swapped ? fast : slow;
        const int gr = r0 + r, gj = J * kRB + j;
        T v = T(0);
        if (gr < n) v = load_lprime(p, gr, gj);
        ls[lidx(ls, r, j)] = p.trsm ? -v : v;
      }
      __syncthreads();
      gp.mma(ls, panel, J * kRB);
      __syncthreads();
    }
    if (p.trsm) gp.store(panel, r0);
    else gp.store(ys, 0);

    // 3. Diagonal block, masked: ld[p][r] = L'(r, p) for p < r, diag on p == r.
    for (int q = tid; q < kRB * kRB; q += kThreads) {
      const int fast = q & (kRB - 1), slow = q >> 5;
      const int r = p.swapped ? slow : fast, pc = p.swapped ? fast : slow;
      const int gr = r0 + r, gp_ = r0 + pc;
      T v = T(0);
      if (gr < n && gp_ < n) {
        if (pc < r) v = load_lprime(p, gr, gp_);
        else if (pc == r) {
          if (p.unit) v = T(1);
          else if (!p.trsm) v = load_lprime(p, gr, gr);
        }
      }
      ld[pc * kRB + r] = v;
    }
    __syncthreads();

    T v[4];
    if (p.trsm) {
#pragma unroll
      for (int q = 0; q < 4; ++q) v[q] = panel[pidx(panel, r0 + gq + 8 * q, cc)];
#pragma unroll
      for (int pp = 0; pp < kRB; ++pp) {
        const int qo = pp >> 3, go = pp & 7;
        T x = T(0);
        if (gq == go) {
          v[qo] = v[qo] * rinv[r0 + pp];
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
      for (int q = 0; q < 4; ++q) panel[pidx(panel, r0 + gq + 8 * q, cc)] = v[q];
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) v[q] = ys[pidx(ys, gq + 8 * q, cc)];
#pragma unroll 8
      for (int pp = 0; pp < kRB; ++pp) {
        const T b = panel[pidx(panel, r0 + pp, cc)];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int r = gq + 8 * q;
          if (pp <= r) v[q] = fma(ld[pp * kRB + r], b, v[q]);
        }
      }
      __syncwarp();  // all readers of column cc live in this warp
#pragma unroll
      for (int q = 0; q < 4; ++q) panel[pidx(panel, r0 + gq + 8 * q, cc)] = p.alpha * v[q];
    }
    __syncthreads();
  }

  // 4. Write back.
  for (int q = tid; q < n * kNC; q += kThreads) {
    const int r = p.right ? q / kNC : q % n;
    const int c = p.right ? q % kNC : q / n;
    if (c < ncols) p.B[gaddr(r, c)] = panel[pidx(panel, r, c)];
  }
}

template <typename T>
void launch_leaf(const LeafParams<T>& p, cudaStream_t s) {
  if (p.n <= 0 || p.nrhs <= 0) return;
  const int smem = static_cast<int>((Smem<T>::panel + 3 * Smem<T>::blk + kLeafMax) * sizeof(T));
  cudaFuncSetAttribute(leaf_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const unsigned grid = static_cast<unsigned>(ceil_div(p.nrhs, kNC));
  leaf_kernel<T><<<grid, kThreads, smem, s>>>(p);
  ++launch_counter();
}

}  // namespace

void launch_leaf_f64(const LeafParams<double>& p, cudaStream_t s) { launch_leaf<double>(p, s); }
void launch_leaf_f32(const LeafParams<float>& p, cudaStream_t s) { launch_leaf<float>(p, s); }

}  // namespace rectri_cu
