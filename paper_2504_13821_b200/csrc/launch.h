// launch.h -- host-side launchers of the sm_100a kernels (internal).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace rectri_cu {

using i64 = int64_t;

// C[M x N] <- alpha * op(A)[M x K] * op(B)[K x N] + beta * C, column-major.
// beta == 0 never reads C.  The per-element reduction order is k-ascending
// and independent of the tile configuration chosen (so results do not depend
// on N, which is what makes RHS sharding bitwise-stable).
template <typename T>
struct GemmParams {
  i64 M, N, K;
  T alpha, beta;
  const T* A;
  i64 lda;
  const T* B;
  i64 ldb;
  T* C;
  i64 ldc;
  // Scheduling hint (never changes a bit): 1 when other work runs beside this
  // update (TRMM's concurrent halves), so it keeps the large tiles.
  int busy_gpu = 0;
  // Ring checking (RECTRI_CU_RING_CHECK, the TMA kernels' checker
  // instantiation): mismatch counter and planted stage mix-up.
  unsigned long long* ring_check = nullptr;
  int ring_plant = 0;
};

// Leaf (base-kernel) problem in the reference's Left form on a virtual lower
// factor L' (base_kernels.cpp:35-89): element r of right-hand side c is
// B(pi(r), c) (Left) or B(c, pi(r)) (Right, `right` = 1), pi(r) = n-1-r when
// `reflected`; L'(r, j) = A(R(r), R(j)) or, when `swapped`, A(R(j), R(r)),
// with R the same reflection.  Unit diag never reads A(r, r).
template <typename T>
struct LeafParams {
  int n;  // tile order, <= kLeafMax
  i64 nrhs;
  const T* A;
  i64 lda;
  T* B;
  i64 ldb;
  int right;
  int reflected;
  int swapped;
  int unit;
  int trsm;  // 1: solve, 0: multiply
  T alpha;
  // Experiments only (RECTRI_CU_LEAF_DEBUG): 1 no diagonal part, 2 no GEMM
  // part (timing), 3 planted missing barrier (racecheck negative test).
  int debug_skip = 0;
  long long* trace = nullptr;  // RECTRI_CU_LEAF_TRACE: per-CTA clock64 stamps (leaf64.cu)
  double* packed = nullptr;    // v3: this leaf's triangle already packed here (pack3_all_kernel)
  int pack_asc = 0;            // packed TRMM blocks in ascending row order (the v5 leaf's; TRSM always is)
  int direct = 0;              // a direct trmm_base / trsm_base call (not inside a recursion)
  // Ring checking (RECTRI_CU_RING_CHECK, leaf64_v3.cu): every fragment a
  // consumer warp read from a ring slot is compared with the packed block in
  // global memory; mismatches are counted here.  ring_plant: the consumers
  // read the wrong slot (the checker's negative test).
  unsigned long long* ring_check = nullptr;
  int ring_plant = 0;
};

constexpr int kLeafMax = 256;

void launch_gemm_f64(const GemmParams<double>& p, bool ta, bool tb, cudaStream_t s);
// 64x64 tiles with the last, short wave's columns in 32x32 tiles (same bits).
bool launch_gemm_f64_split(const GemmParams<double>& p, bool ta, bool tb, cudaStream_t s);
void launch_gemm_f32(const GemmParams<float>& p, bool ta, bool tb, cudaStream_t s);
// fp32 3xTF32 variant on tcgen05 (sgemm_tf32x3.cu), opt-in: RECTRI_CU_FP32_TF32X3=1.
bool tf32x3_enabled();
void tf32x3_set_call(bool on);  // RECTRI_CU_TF32X3 for the calling thread's current call
bool launch_gemm_f32_tf32x3(const GemmParams<float>& p, bool ta, bool tb, cudaStream_t s);
void tf32x3_reserve(cudaStream_t s, size_t floats);  // per-stream operand-split scratch
void launch_leaf_f64(const LeafParams<double>& p, cudaStream_t s);     // leaf64.cu (v2)
void launch_leaf_f64_v1(const LeafParams<double>& p, cudaStream_t s);  // leaf.cu
void launch_leaf_f64_v3(const LeafParams<double>& p, double* scratch, cudaStream_t s,
                        bool prepacked = false);  // leaf64_v3.cu
// Packs the triangles of all leaves of one recursion (leaf k: order d_n[k]
// at A(d_r0[k], d_r0[k]); base carries A, lda and the variant flags) into
// scratch + k * leaf3_scratch_doubles().
void launch_leaf3_pack_all(const LeafParams<double>& base, const long long* d_r0, const int* d_n, int nleaves,
                           double* scratch, cudaStream_t s);
size_t leaf3_scratch_doubles();
// Packs one leaf's triangle (p.A, p.n, variant flags) into dst.
void launch_leaf3_pack(const LeafParams<double>& p, double* dst, cudaStream_t s);
int leaf_version();  // RECTRI_CU_LEAF (fp64: 1 = leaf.cu, 2 = leaf64.cu, 3 = leaf64_v3.cu, 4 = v3 + v5 TRMM)
int leaf3_width(long long nrhs, bool trsm);  // fp64 leaf v3 panel width (8 / 16 / 32)
// fp64 TRMM leaf v5 (leaf64_v5.cu): row-block-owning warps for few
// right-hand sides, bitwise the v3 arithmetic; width 0 = not used for nrhs.
// Direct trmm_base calls use it; inside the recursion it is opt-in
// (RECTRI_CU_LEAF=4), since beside the other stream's GEMMs v3 measured faster.
int leaf5_width(long long nrhs);
void launch_leaf_f64_v5_trmm(const LeafParams<double>& p, const double* packed, int width, cudaStream_t s);
// Recursion TRMM triangles are packed in v5's ascending row order rather than
// v3's descending one: RECTRI_CU_LEAF >= 4.
inline bool leaf_trmm_asc() { return leaf_version() >= 4; }
// Allocates the v2 fp64 leaf's per-stream scratch (call before capturing on s).
void leaf_scratch_reserve(cudaStream_t s);
void launch_leaf_f32(const LeafParams<float>& p, cudaStream_t s);     // leaf64.cu dispatch
void launch_leaf_f32_v1(const LeafParams<float>& p, cudaStream_t s);  // leaf.cu
void launch_leaf_f32_v3(const LeafParams<float>& p, float* scratch, cudaStream_t s,
                        bool prepacked = false);  // leaf32_v3.cu
void launch_leaf32_pack_all(const LeafParams<float>& base, const long long* d_r0, const int* d_n, int nleaves,
                            float* scratch, long long stride, cudaStream_t s);

// B[rows x cols] (ld) <- alpha * B.
void launch_scale_f64(double* B, i64 ld, i64 rows, i64 cols, double alpha, cudaStream_t s);
void launch_scale_f32(float* B, i64 ld, i64 rows, i64 cols, float alpha, cudaStream_t s);
void launch_accumulate_f64(double* D, i64 ldd, const double* S, i64 rows, i64 cols, double c, cudaStream_t s);
void launch_accumulate_f32(float* D, i64 ldd, const float* S, i64 rows, i64 cols, float c, cudaStream_t s);
// flags[r] = (A(r, r) == 0) for r < n.
void launch_diag_zero_scan_f64(const double* A, i64 lda, i64 n, uint8_t* flags, cudaStream_t s);
void launch_diag_zero_scan_f32(const float* A, i64 lda, i64 n, uint8_t* flags, cudaStream_t s);

// Synthetic inputs: uniform [-1, 1) keyed by the global element index
// (col0 + c) * global_rows + r; diagonal := off-diagonal |row sum| + 1.
void launch_fill_uniform_f64(double* B, i64 ld, i64 rows, i64 cols, i64 col0, i64 grows,
                             uint64_t seed, cudaStream_t s);
void launch_fill_uniform_f32(float* B, i64 ld, i64 rows, i64 cols, i64 col0, i64 grows,
                             uint64_t seed, cudaStream_t s);
void launch_make_dominant_f64(double* A, i64 lda, i64 n, int upper, cudaStream_t s);
void launch_make_dominant_f32(float* A, i64 lda, i64 n, int upper, cudaStream_t s);
double probe_peak_tflops(int kind);

// Number of kernel launches issued (incremented by each launcher).
i64& launch_counter();
// RECTRI_CU_RING_CHECK = 1 (check) / 2 (check + planted slot mix-up): the
// device mismatch counter the v3 leaves report to, else nullptr; plant is set
// for mode 2.  leaf_ring_check_read synchronises the device and returns the
// count (allocating the counter on the first call, which must precede the
// checked launches), optionally resetting it.
unsigned long long* leaf_ring_check_counter(int* plant);
long long leaf_ring_check_read(bool reset);

// Scratch a captured graph owns, by the stream its kernels are captured on:
// the unpacked-leaf scratch (leaf64.cu) and the 3xTF32 operand splits
// (sgemm_tf32x3.cu).  While a graph is being captured the builder installs
// its set for the capturing thread, and the launchers take their buffers from
// it instead of the per-stream pools -- so a cached graph never shares
// scratch with another graph (two replays on different streams may run at
// once) and never points at a pool buffer that is later reallocated.
struct CallScratch {
  static constexpr int kMax = 8;
  int n = 0;
  cudaStream_t stream[kMax] = {};
  double* leaf[kMax] = {};
  float* split[kMax] = {};
  size_t split_floats[kMax] = {};
  int find(cudaStream_t s) const {
    for (int k = 0; k < n; ++k)
      if (stream[k] == s) return k;
    return -1;
  }
};
void set_call_scratch(const CallScratch* cs);  // thread-local; nullptr to clear
const CallScratch* call_scratch();
size_t leaf_scratch_bytes();  // one stream's unpacked-leaf scratch

}  // namespace rectri_cu
