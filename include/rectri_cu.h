/*
 * rectri_cu.h -- C-ABI of the B200 (sm_100a) recursive TRMM/TRSM library.
 *
 * This is the drop-in boundary for the reference's hot path
 * (arxiv/paper_2504_13821, "rectri", paths relative to /root/reference/proj).
 * Each entry point replaces one reference C++ entry point with the same
 * argument meaning, validation order and error behaviour:
 *
 *   rectri_cu_rec_trmm_{f32,f64}  <- rectri::rec_trmm<T>   include/rectri/recursion.hpp:66-75
 *                                                         src/recursion.cpp:165-176
 *   rectri_cu_rec_trsm_{f32,f64}  <- rectri::rec_trsm<T>   include/rectri/recursion.hpp:77-86
 *                                                         src/recursion.cpp:178-192
 *   rectri_cu_trmm_base_{f32,f64} <- rectri::trmm_base<T>  include/rectri/base_kernels.hpp:15-19
 *   rectri_cu_trsm_base_{f32,f64} <- rectri::trsm_base<T>  include/rectri/base_kernels.hpp:21-30
 *   rectri_cu_gemm_{f32,f64}      <- rectri::gemm<T>       include/rectri/gemm.hpp:18-21
 *   rectri_cu_scale_{f32,f64}     <- rectri::scale<T>      include/rectri/gemm.hpp:30-33
 *   rectri_cu_schema_for          <- rectri::schema_for    include/rectri/recursion.hpp:58
 *
 * Argument types mirror the reference's boundary types as plain C structs:
 *   rectri_cu_spec    <- rectri::TriangularSpec  include/rectri/flags.hpp:29-35
 *   rectri_cu_view    <- rectri::MatrixView<T>   include/rectri/matrix.hpp:75-160
 *   rectri_cu_backend <- rectri::Backend         include/rectri/backend.hpp:20-29
 *   rectri_cu_event_fn<- rectri::EventSink       include/rectri/recursion.hpp:60-64
 * and every reference exception type maps to one status code
 * (include/rectri/error.hpp:10-84).
 *
 * Matrices are column-major: element (r, c) of a view lives at
 *   origin[(col_offset + c) * origin_rows + row_offset + r].
 * Views may wrap DEVICE memory (computed in place on the device) or HOST
 * memory (staged to the device, computed, copied back); pinned host memory
 * takes the asynchronous copy path.  Calls are synchronous (the reference's
 * contract) unless backend->flags has RECTRI_CU_ASYNC, in which
 * case device-resident calls return once the work is enqueued on
 * backend->stream and singularity is reported by rectri_cu_sync().
 */
#ifndef RECTRI_CU_H_
#define RECTRI_CU_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RECTRI_CU_ABI_VERSION 1

/* Status codes, one per reference exception type. */
enum rectri_cu_status {
  RECTRI_CU_OK = 0,
  RECTRI_CU_CONFIG = 1,     /* ConfigError      */
  RECTRI_CU_SHAPE = 2,      /* ShapeError       */
  RECTRI_CU_ALIAS = 3,      /* AliasError       */
  RECTRI_CU_SINGULAR = 4,   /* SingularityError(index) -> *singular_row */
  RECTRI_CU_TILE_LIMIT = 5, /* TileLimitError   */
  RECTRI_CU_CUDA = 6,       /* CUDA runtime / launch failure (no reference twin) */
  RECTRI_CU_BOUNDS = 7,     /* BoundsError      */
  RECTRI_CU_SPLIT = 8       /* SplitError       */
};

/* Flag enumerations, same order as include/rectri/flags.hpp:14-27. */
enum rectri_cu_side { RECTRI_CU_LEFT = 0, RECTRI_CU_RIGHT = 1 };
enum rectri_cu_uplo { RECTRI_CU_LOWER = 0, RECTRI_CU_UPPER = 1 };
enum rectri_cu_trans { RECTRI_CU_NOTRANS = 0, RECTRI_CU_TRANS = 1, RECTRI_CU_CONJTRANS = 2 };
enum rectri_cu_diag { RECTRI_CU_NONUNIT = 0, RECTRI_CU_UNIT = 1 };

/* RecEvent (recursion.hpp:60): one per GEMM update and base-kernel call. */
enum rectri_cu_event { RECTRI_CU_EV_GEMM = 0, RECTRI_CU_EV_BASE_TRMM = 1, RECTRI_CU_EV_BASE_TRSM = 2 };

typedef struct rectri_cu_spec {
  int32_t side;  /* rectri_cu_side  */
  int32_t uplo;  /* rectri_cu_uplo  */
  int32_t trans; /* rectri_cu_trans */
  int32_t diag;  /* rectri_cu_diag  */
  double alpha;  /* must be finite (flags.hpp:47-49) */
} rectri_cu_spec;

typedef struct rectri_cu_view {
  void* origin;        /* base of the origin buffer (float* or double*) */
  int64_t origin_rows; /* leading dimension                              */
  int64_t origin_cols;
  int64_t row_offset;
  int64_t col_offset;
  int64_t rows;
  int64_t cols;
} rectri_cu_view;

/* backend->flags */
#define RECTRI_CU_ASYNC 1u    /* do not synchronize before returning        */
#define RECTRI_CU_NO_GRAPH 2u /* launch kernels directly, no graph capture  */
#define RECTRI_CU_TF32X3 4u   /* fp32 GEMM updates as 3xTF32 on tcgen05: an
                                 opt-in variant, reported separately under its
                                 own tolerance (default fp32 is exact FFMA)    */

typedef struct rectri_cu_backend {
  int32_t parallel_width; /* validated >= 1 (backend.hpp:31-37)            */
  int32_t device;         /* CUDA ordinal; -1 = the current device         */
  void* stream;           /* cudaStream_t; NULL = legacy default stream    */
  uint32_t flags;         /* RECTRI_CU_ASYNC | RECTRI_CU_NO_GRAPH | RECTRI_CU_TF32X3 */
  int64_t mc, kc, nc;     /* GemmBlocking, validated >= 1 (advisory on GPU) */
} rectri_cu_backend;

/* Event sink; called on the caller's thread, in recursion order, before the
 * corresponding work is enqueued.  NULL = no sink. */
typedef void (*rectri_cu_event_fn)(void* user, int32_t event, int64_t n, int64_t m);

/* Recursive drivers (rec_trmm / rec_trsm).  *singular_row receives the
 * global row of the first exact-zero pivot met in leaf order (TRSM only). */
int rectri_cu_rec_trmm_f64(const rectri_cu_spec* spec, rectri_cu_view A, rectri_cu_view B,
                           int64_t threshold, const rectri_cu_backend* backend,
                           rectri_cu_event_fn sink, void* sink_user);
int rectri_cu_rec_trmm_f32(const rectri_cu_spec* spec, rectri_cu_view A, rectri_cu_view B,
                           int64_t threshold, const rectri_cu_backend* backend,
                           rectri_cu_event_fn sink, void* sink_user);
int rectri_cu_rec_trsm_f64(const rectri_cu_spec* spec, rectri_cu_view A, rectri_cu_view B,
                           int64_t threshold, const rectri_cu_backend* backend,
                           rectri_cu_event_fn sink, void* sink_user, int64_t* singular_row);
int rectri_cu_rec_trsm_f32(const rectri_cu_spec* spec, rectri_cu_view A, rectri_cu_view B,
                           int64_t threshold, const rectri_cu_backend* backend,
                           rectri_cu_event_fn sink, void* sink_user, int64_t* singular_row);

/* Base (leaf) kernels.  tile_limit as base_kernels.hpp:10-19. */
int rectri_cu_trmm_base_f64(const rectri_cu_spec* spec, rectri_cu_view A, rectri_cu_view B,
                            int64_t tile_limit, const rectri_cu_backend* backend);
int rectri_cu_trmm_base_f32(const rectri_cu_spec* spec, rectri_cu_view A, rectri_cu_view B,
                            int64_t tile_limit, const rectri_cu_backend* backend);
int rectri_cu_trsm_base_f64(const rectri_cu_spec* spec, rectri_cu_view A, rectri_cu_view B,
                            int64_t tile_limit, const rectri_cu_backend* backend,
                            int64_t* singular_row);
int rectri_cu_trsm_base_f32(const rectri_cu_spec* spec, rectri_cu_view A, rectri_cu_view B,
                            int64_t tile_limit, const rectri_cu_backend* backend,
                            int64_t* singular_row);

/* C <- alpha * op(A) * op(B) + beta * C (gemm.hpp:18-21); trans codes as
 * rectri_cu_trans.  beta == 0 never reads C; alpha == 0 or k == 0 skips the
 * product. */
int rectri_cu_gemm_f64(double alpha, int32_t trans_a, rectri_cu_view A, int32_t trans_b,
                       rectri_cu_view B, double beta, rectri_cu_view C,
                       const rectri_cu_backend* backend);
int rectri_cu_gemm_f32(float alpha, int32_t trans_a, rectri_cu_view A, int32_t trans_b,
                       rectri_cu_view B, float beta, rectri_cu_view C,
                       const rectri_cu_backend* backend);

/* B <- alpha * B (gemm.hpp:30-33). */
int rectri_cu_scale_f64(double alpha, rectri_cu_view B, const rectri_cu_backend* backend);
int rectri_cu_scale_f32(float alpha, rectri_cu_view B, const rectri_cu_backend* backend);

/* schema_for (recursion.cpp:18-46); op 0 = trmm, 1 = trsm.  out[8] =
 * {first_is_a22, off_trans, off_on_left, read_half_is_b2, write_half_is_b2,
 *  sign, carries_alpha, second_is_a22}. */
int rectri_cu_schema_for(int32_t op, const rectri_cu_spec* spec, double out[8]);

/* Waits for all async work issued on `stream` by this library and reports
 * any deferred singularity (RECTRI_CU_ASYNC mode). */
int rectri_cu_sync(void* stream, int64_t* singular_row);

/* Message of the last non-OK status returned on this thread. */
const char* rectri_cu_last_error(void);

/* Number of kernel launches (graph nodes count individually) issued by this
 * library since load; used by the bench's gpu_launches accounting. */
int64_t rectri_cu_launch_count(void);

/* Drops every cached CUDA graph (e.g. before freeing buffers whose
 * addresses are baked into cached graphs).  The cache is bounded by entry
 * count (64) and by the device bytes its entries own
 * (RECTRI_CU_GRAPH_CACHE_MB, default 4096).  Deferred singularity checks of
 * RECTRI_CU_ASYNC calls survive and are reported by rectri_cu_sync. */
void rectri_cu_clear_graph_cache(void);

/* Frees the per-device staging buffers of the host-operand path (they grow
 * to the largest host-resident problem seen and are otherwise kept for
 * reuse).  Waits for a host-operand call in flight on that device. */
void rectri_cu_release_staging(void);

/* Device bytes the library currently holds across calls: cached graphs'
 * scratch plus staging buffers. */
int64_t rectri_cu_device_bytes_held(void);

int rectri_cu_abi_version(void);

/* ---- Utilities (not reference entry points) --------------------------------
 * Synthetic inputs on the device, the counterpart of the reference's bench
 * generators (src/bench.cpp:32-61): uniform [-1, 1) keyed by the GLOBAL
 * element index (col0 + c) * global_rows + r, so column shards generated on
 * different GPUs reproduce the unsharded matrix; and the diagonal-dominance
 * fixup diag := stored off-diagonal |row sum| + 1 (uplo selects the triangle).
 * dtype: 0 = f32, 1 = f64.  Device pointers only. */
int rectri_cu_fill_uniform(int32_t dtype, rectri_cu_view B, int64_t col0, int64_t global_rows,
                           uint64_t seed, const rectri_cu_backend* backend);
int rectri_cu_make_dominant(int32_t dtype, rectri_cu_view A, int32_t uplo,
                            const rectri_cu_backend* backend);

/* Measured issue-rate peak on the current device in TFLOP/s:
 * kind 0 = fp64 DMMA.8x8x4, 1 = fp32 FFMA.  Negative on failure. */
double rectri_cu_probe_peak(int32_t kind);

/* Ring checking of the mbarrier-guarded shared-memory rings (a diagnostic,
 * not a reference entry point; the role of the reference's workgroup race
 * detector, src/workgroup.cpp:138-177).  With RECTRI_CU_RING_CHECK=1 in the
 * environment when a kernel is launched (or a graph captured), the fp64 /
 * fp32 v3 leaves, the TMA DGEMM and the fp32 FFMA2 GEMM compare every
 * fragment a consumer warp reads from a stage with the element the stage
 * must hold (packed block / op(A), op(B) in global memory) -- a refill
 * overtaking a stage's readers shows up as a mismatch; =2 also plants a
 * stage mix-up (the negative test).  Synchronises the device and returns the mismatch count
 * (-1 if the counter cannot be allocated); reset != 0 zeroes it.  The first
 * call allocates the counter: make it before the checked launches (a graph
 * capture cannot allocate). */
int64_t rectri_cu_debug_ring_check(int32_t reset);

/* Host storage of the C++ drop-in's MatrixBuffer (include/rectri_b200.hpp;
 * the reference's std::vector storage, include/rectri/matrix.hpp:18-70):
 * page-locked when a CUDA device is present and RECTRI_CU_PINNED_BUFFERS is
 * not 0 (*pinned = 1), so host-resident operands in MatrixBuffers move at
 * full PCIe rate without a bounce copy; plain malloc otherwise.  NULL on
 * failure.  rectri_cu_host_free releases a pointer from rectri_cu_host_alloc
 * (and ignores anything else). */
void* rectri_cu_host_alloc(size_t bytes, int32_t* pinned);
void rectri_cu_host_free(void* p);

/* Per-kernel-class CUDA-event profiling.  While enabled, every call launches
 * directly (no graph) and brackets each launch with events on its stream.
 * rectri_cu_profile_read fills, for kinds 0 = GEMM, 1 = leaf, 2 = scale,
 * 3 = pivot scan: device milliseconds, launches and algorithmic flops
 * (GEMM 2MNK, leaf nb^2 * rhs), then clears the record. */
void rectri_cu_profile_enable(int32_t on);

/* Benchmark-harness helpers (bench CLI parity): the reference's input
 * generator (src/bench.cpp:32-61) and residual-gate column sample
 * (:109-117), evaluated with libstdc++ <random> -> bit-identical streams.
 * Host buffers, column-major (A n x n, B brows x bcols). */
void rectri_cu_bench_inputs_f64(double* a, double* b, int64_t n, int64_t brows, int64_t bcols,
                                int32_t is_trsm, int32_t uplo, int32_t diag, uint64_t seed);
void rectri_cu_bench_inputs_f32(float* a, float* b, int64_t n, int64_t brows, int64_t bcols,
                                int32_t is_trsm, int32_t uplo, int32_t diag, uint64_t seed);
int32_t rectri_cu_gate_columns(uint64_t seed, int64_t cols, int64_t out[8]);
int rectri_cu_profile_read(double ms[4], int64_t launches[4], double flops[4]);

#ifdef __cplusplus
}
#endif

#endif /* RECTRI_CU_H_ */
