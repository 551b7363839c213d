// driver.cu -- host side of the B200 TRMM/TRSM library and its C-ABI.
//
// Mirrors the reference's recursion driver (src/recursion.cpp:48-192) on
// the host: the same validation order (check_problem, :50-67), the same
// schema table (schema_for, :18-46), the same split at floor(n/2)
// (matrix.hpp:180-183) and the same event sequence (:94, :97, :139) -- but
// instead of computing, each node ENQUEUES one sm_100a kernel (leaf or GEMM)
// on a CUDA stream.  The launch sequence of a (problem, buffers) key is
// captured once into a CUDA graph and replayed on later calls, with the
// recorded event list replayed to the caller's sink.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <functional>
#include <list>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <type_traits>
#include <unordered_map>
#include <vector>

#include "../../include/rectri_cu.h"
#include "host_stage.h"
#include "launch.h"

namespace rectri_cu {
namespace {

// ---------------------------------------------------------------------------
// Errors: every reference exception type is one status code.
struct Fail {
  int code;
  std::string msg;
  i64 index = -1;
};

thread_local std::string g_last_error;

[[noreturn]] void fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  throw Fail{code, buf};
}

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(RECTRI_CU_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

template <typename F>
int guarded(F&& f, i64* index_out) {
  try {
    f();
    return RECTRI_CU_OK;
  } catch (const Fail& e) {
    g_last_error = e.msg;
    if (e.code == RECTRI_CU_SINGULAR && index_out) *index_out = e.index;
    return e.code;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return RECTRI_CU_CUDA;
  }
}

// NVTX ranges (tracing): one per library call and per recursion
// level of the host traversal (capture / descriptor runs / direct launches),
// so nsys / ncu timelines group the kernels by call and level.  Header-only
// NVTX v3: a no-op unless a tool injects itself.
struct Nvtx {
  explicit Nvtx(const char* name) { nvtxRangePushA(name); }
  Nvtx(const char* fmt, long long a, long long b) {
    char buf[96];
    std::snprintf(buf, sizeof buf, fmt, a, b);
    nvtxRangePushA(buf);
  }
  ~Nvtx() { nvtxRangePop(); }
};

// ---------------------------------------------------------------------------
// Boundary types.
enum OpK { kTrmm = 0, kTrsm = 1 };

const char* side_name(int s) { return s == RECTRI_CU_LEFT ? "left" : "right"; }

struct Spec {
  int side, uplo, trans, diag;  // trans already reduced: 0 = N, 1 = T
  double alpha;
};

Spec validate_spec(const rectri_cu_spec* s) {
  if (!s) fail(RECTRI_CU_CONFIG, "spec must not be null");
  if (s->side < 0 || s->side > 1 || s->uplo < 0 || s->uplo > 1 || s->trans < 0 || s->trans > 2 ||
      s->diag < 0 || s->diag > 1)
    fail(RECTRI_CU_CONFIG, "spec flag out of range");
  // flags.hpp:47-49
  if (!std::isfinite(s->alpha)) fail(RECTRI_CU_CONFIG, "alpha must be finite");
  // ConjTrans == Trans on real element kinds (flags.hpp:38-45).
  return Spec{s->side, s->uplo, s->trans == RECTRI_CU_NOTRANS ? 0 : 1, s->diag, s->alpha};
}

struct BackendInfo {
  int device = -1;
  cudaStream_t stream = nullptr;
  unsigned flags = 0;
};

// RECTRI_CU_TF32X3 for the duration of one fp32 call on this thread.
struct Tf32x3Scope {
  explicit Tf32x3Scope(bool on) { tf32x3_set_call(on); }
  ~Tf32x3Scope() { tf32x3_set_call(false); }
};

BackendInfo validate_backend(const rectri_cu_backend* b) {
  BackendInfo out;
  if (!b) return out;  // Backend{} defaults
  // backend.hpp:31-37
  if (b->parallel_width < 1) fail(RECTRI_CU_CONFIG, "backend parallel_width must be >= 1");
  if (b->mc < 1 || b->kc < 1 || b->nc < 1)
    fail(RECTRI_CU_CONFIG, "backend block sizes must be >= 1");
  out.device = b->device;
  out.stream = static_cast<cudaStream_t>(b->stream);
  out.flags = b->flags;
  return out;
}

void validate_view(const rectri_cu_view& v, const char* name) {
  if (v.rows < 0 || v.cols < 0 || v.row_offset < 0 || v.col_offset < 0 ||
      v.row_offset + v.rows > v.origin_rows || v.col_offset + v.cols > v.origin_cols)
    fail(RECTRI_CU_BOUNDS, "view %s escapes its origin", name);
}

bool view_empty(const rectri_cu_view& v) { return v.rows == 0 || v.cols == 0; }

// matrix.hpp:168-177
bool overlaps(const rectri_cu_view& a, const rectri_cu_view& b) {
  if (a.origin != b.origin) return false;
  if (view_empty(a) || view_empty(b)) return false;
  const bool rows_meet = a.row_offset < b.row_offset + b.rows && b.row_offset < a.row_offset + a.rows;
  const bool cols_meet = a.col_offset < b.col_offset + b.cols && b.col_offset < a.col_offset + a.cols;
  return rows_meet && cols_meet;
}

template <typename T>
struct DView {
  T* p;
  i64 ld, rows, cols;
  DView sub(i64 r0, i64 c0, i64 nr, i64 nc) const { return DView{p + c0 * ld + r0, ld, nr, nc}; }
  operator DView<const T>() const { return DView<const T>{p, ld, rows, cols}; }
};

template <typename T>
DView<T> dview_of(const rectri_cu_view& v) {
  T* base = static_cast<T*>(v.origin);
  return DView<T>{base + v.col_offset * v.origin_rows + v.row_offset, v.origin_rows, v.rows, v.cols};
}

bool is_device_memory(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// ---------------------------------------------------------------------------
// Recursion schema (recursion.cpp:18-46), verbatim rule.
struct Schema {
  bool first_a22;
  int off_trans;
  bool off_on_left;
  bool read_b2, write_b2;
  double sign;
  bool carries_alpha;
};

Schema schema_for(OpK op, int side, int uplo, int trans) {
  const bool straight = (uplo == RECTRI_CU_LOWER) == (trans == 0);
  const bool flip_for_op = op == kTrsm;
  const bool flip_for_side = side == RECTRI_CU_RIGHT;
  const bool first_is_a22 = (straight != flip_for_op) != flip_for_side;
  Schema s;
  s.first_a22 = first_is_a22;
  s.off_trans = trans;
  s.off_on_left = side == RECTRI_CU_LEFT;
  const bool first_b2 = first_is_a22;
  if (op == kTrmm) {
    s.write_b2 = first_b2;
    s.read_b2 = !first_b2;
    s.sign = 1.0;
    s.carries_alpha = true;
  } else {
    s.read_b2 = first_b2;
    s.write_b2 = !first_b2;
    s.sign = -1.0;
    s.carries_alpha = false;
  }
  return s;
}

// ---------------------------------------------------------------------------
// Kernel launch shims per element type.
template <typename T>
struct K;
template <>
struct K<double> {
  static void gemm(const GemmParams<double>& p, bool ta, bool tb, cudaStream_t s) {
    launch_gemm_f64(p, ta, tb, s);
  }
  static void leaf(const LeafParams<double>& p, cudaStream_t s) { launch_leaf_f64(p, s); }
  static void scale(double* B, i64 ld, i64 r, i64 c, double a, cudaStream_t s) {
    launch_scale_f64(B, ld, r, c, a, s);
  }
  static void accumulate(double* D, i64 ldd, const double* S, i64 r, i64 c, double k, cudaStream_t s) {
    launch_accumulate_f64(D, ldd, S, r, c, k, s);
  }
  static void scan(const double* A, i64 lda, i64 n, uint8_t* f, cudaStream_t s) {
    launch_diag_zero_scan_f64(A, lda, n, f, s);
  }
};
template <>
struct K<float> {
  static void gemm(const GemmParams<float>& p, bool ta, bool tb, cudaStream_t s) {
    launch_gemm_f32(p, ta, tb, s);
  }
  static void leaf(const LeafParams<float>& p, cudaStream_t s) { launch_leaf_f32(p, s); }
  static void scale(float* B, i64 ld, i64 r, i64 c, float a, cudaStream_t s) {
    launch_scale_f32(B, ld, r, c, a, s);
  }
  static void accumulate(float* D, i64 ldd, const float* S, i64 r, i64 c, float k, cudaStream_t s) {
    launch_accumulate_f32(D, ldd, S, r, c, k, s);
  }
  static void scan(const float* A, i64 lda, i64 n, uint8_t* f, cudaStream_t s) {
    launch_diag_zero_scan_f32(A, lda, n, f, s);
  }
};

struct Ev {
  int32_t e;
  i64 n, m;
};

// Per-kernel-class event profiling (rectri_cu_profile_*).
struct ProfRec {
  int kind;
  double flops;
  cudaEvent_t a, b;
};
struct Profiler {
  bool on = false;
  std::vector<ProfRec> recs;
};
Profiler g_prof;

struct ProfScope {
  ProfRec rec{};
  cudaStream_t s;
  bool active;
  ProfScope(int kind, double flops, cudaStream_t s_) : s(s_), active(g_prof.on) {
    if (!active) return;
    rec.kind = kind;
    rec.flops = flops;
    cudaEventCreate(&rec.a);
    cudaEventCreate(&rec.b);
    cudaEventRecord(rec.a, s);
  }
  ~ProfScope() {
    if (!active) return;
    cudaEventRecord(rec.b, s);
    g_prof.recs.push_back(rec);
  }
};

// Enqueues C <- alpha * op(A) * op(B) + beta * C (gemm.cpp:155-216 minus
// validation): alpha == 0 or K == 0 only applies beta.
template <typename T>
void enqueue_gemm(T alpha, bool ta, DView<const T> A, bool tb, DView<const T> B, T beta,
                  DView<T> C, cudaStream_t s, int busy_gpu = 0) {
  const i64 M = C.rows, N = C.cols, Kd = ta ? A.rows : A.cols;
  if (M == 0 || N == 0) return;
  if (alpha == T(0) || Kd == 0) {  // apply_beta (gemm.cpp:129-142)
    if (beta == T(0))
      cuda_check(cudaMemset2DAsync(C.p, sizeof(T) * C.ld, 0, sizeof(T) * M, N, s), "zero C");
    else if (beta != T(1))
      K<T>::scale(C.p, C.ld, M, N, beta, s);
    return;
  }
  GemmParams<T> p{M, N, Kd, alpha, beta, A.p, A.ld, B.p, B.ld, C.p, C.ld, busy_gpu};
  ProfScope prof(0, 2.0 * static_cast<double>(M) * N * Kd, s);
  K<T>::gemm(p, ta, tb, s);
}

// One base-kernel call on the device (base_kernels.cpp:137-177 minus
// validation and the zero-pivot scan).  Tiles above kLeafMax are solved by an
// internal recursion with the same schema (no events: semantically one call).
template <typename T>
void enqueue_base(OpK op, const Spec& spec, DView<const T> A, DView<T> B, cudaStream_t s,
                  double* packed = nullptr, int pack_asc = 0, int direct = 0);

// One kernel of the recursion, as emitted by a descriptor run (the streamed
// host path executes these itself).
template <typename T>
struct KDesc {
  bool leaf;
  Spec spec;             // leaf: the (alpha-adjusted) spec
  DView<const T> a;      // leaf: diagonal block; GEMM: off-diagonal block
  DView<T> src, dst;     // leaf: dst = its B block; GEMM: src (read), dst (updated)
  T coeff;               // GEMM: dst += coeff * op(off) * src  (Right: src * op(off))
  bool off_trans, off_on_left;
};

// Concurrent TRMM halves.  In a TRMM node the first half-problem writes the
// GEMM's destination and the second overwrites the GEMM's source, so the
// serial order is first -> GEMM -> second.  With a scratch S the GEMM can run
// beside the first half: S = op(off) * src (alpha 1, beta 0: S is the exact
// accumulator), then the second half on the GEMM's stream, and after the
// join dst = fma(coeff, S, dst) -- the GEMM epilogue's own single rounding,
// so the result is bitwise the serial one.  Used where the node's GEMM is
// too small to fill the GPU (latency-bound small calls), with streams,
// events and scratch from a per-call context; without one (or when it runs
// out) nodes run serially.
template <typename T>
struct ConcCtx {
  std::vector<cudaStream_t>* streams = nullptr;  // per device: one pool for captures, one for direct calls
  std::vector<cudaEvent_t> events;               // this call's fork/join events (never shared across calls)
  size_t next_stream = 0;
  T* scratch = nullptr;
  i64 cap = 0, used = 0;
  static constexpr i64 kMaxElems = i64(1) << 21;  // per node: mid x rhs (default)
  i64 max_elems = kMaxElems;
  cudaEvent_t event() {
    cudaEvent_t e;
    cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    events.push_back(e);
    return e;
  }
  ~ConcCtx() {
    for (cudaEvent_t e : events) cudaEventDestroy(e);
  }
};

template <typename T>
class Recursion {
 public:
  Recursion(OpK op, i64 threshold, cudaStream_t s, std::vector<Ev>* events,
            std::vector<std::pair<i64, i64>>* leaves, bool dry = false)
      : op_(op), threshold_(threshold), s_(s), events_(events), leaves_(leaves), dry_(dry) {}

  // Called before each kernel (also in dry runs): leaf (a = diagonal block,
  // b1 = its B block, b2 unused) or GEMM (a = off-diagonal block, b1 = src,
  // b2 = dst).
  std::function<void(bool leaf, DView<const T> a, DView<T> b1, DView<T> b2)> before;
  // Descriptor mode: every kernel is handed to `kernels` instead of launched.
  std::function<void(const KDesc<T>&)> kernels;
  // fp64 leaves whose triangles were packed once for the whole call
  // (launch_leaf3_pack_all): leaf k reads packed + k * packed_stride.
  double* packed = nullptr;
  size_t packed_stride = 0;
  int pack_asc = 0;  // TRMM triangles packed in ascending order (v5 leaf)
  int leaf_idx = 0;
  ConcCtx<T>* conc = nullptr;

  // Scratch elements the concurrent TRMM nodes of run(n, rhs) use.
  static i64 conc_need(OpK op, i64 threshold, i64 n, i64 rhs, i64 max_elems) {
    if (op != kTrmm || n <= threshold) return 0;
    const i64 mid = n / 2, big = n - mid;
    const i64 own = mid * rhs <= max_elems ? big * rhs : 0;
    return own + conc_need(op, threshold, mid, rhs, max_elems) + conc_need(op, threshold, big, rhs, max_elems);
  }

  // recursion.cpp:85-148
  void run(const Spec& spec, DView<const T> A, DView<T> B, i64 row0) {
    const i64 n = A.rows;
    const i64 rhs = spec.side == RECTRI_CU_LEFT ? B.cols : B.rows;
    if (n <= threshold_) {
      emit(op_ == kTrmm ? RECTRI_CU_EV_BASE_TRMM : RECTRI_CU_EV_BASE_TRSM, n, rhs);
      if (leaves_) leaves_->push_back({row0, n});
      if (before) before(true, A, B, B);
      if (kernels) kernels(KDesc<T>{true, spec, A, B, B, T(0), false, false});
      else if (!dry_)
        enqueue_base<T>(op_, spec, A, B, s_, packed ? packed + leaf_idx * packed_stride : nullptr, pack_asc);
      ++leaf_idx;
      return;
    }
    const i64 mid = n / 2;  // split_half
    // the upper levels only (each range formats a string on the host)
    std::unique_ptr<Nvtx> range;
    if (n >= 1024) range = std::make_unique<Nvtx>("rectri node n=%lld rhs=%lld", static_cast<long long>(n),
                                                  static_cast<long long>(rhs));
    const Schema sc = schema_for(op_, spec.side, spec.uplo, spec.trans);
    const DView<const T> a11 = A.sub(0, 0, mid, mid);
    const DView<const T> a22 = A.sub(mid, mid, n - mid, n - mid);
    const DView<const T> off =
        spec.uplo == RECTRI_CU_LOWER ? A.sub(mid, 0, n - mid, mid) : A.sub(0, mid, mid, n - mid);
    const bool left = spec.side == RECTRI_CU_LEFT;
    const DView<T> b1 = left ? B.sub(0, 0, mid, B.cols) : B.sub(0, 0, B.rows, mid);
    const DView<T> b2 = left ? B.sub(mid, 0, n - mid, B.cols) : B.sub(0, mid, B.rows, n - mid);

    const DView<T> dst = sc.write_b2 ? b2 : b1;
    const DView<const T> src = sc.read_b2 ? b2 : b1;
    const T coeff = static_cast<T>(sc.sign * (sc.carries_alpha ? spec.alpha : 1.0));
    if (conc_node(sc, mid, rhs, dst)) {
      run_concurrent(spec, sc, a11, a22, off, b1, b2, dst, src, coeff, mid, row0);
      return;
    }

    if (sc.first_a22) run(spec, a22, b2, row0 + mid);
    else run(spec, a11, b1, row0);

    emit(RECTRI_CU_EV_GEMM, dst.rows, dst.cols);
    if (before) before(false, off, sc.read_b2 ? b2 : b1, dst);
    if (kernels) {
      kernels(KDesc<T>{false, spec, off, sc.read_b2 ? b2 : b1, dst, coeff, sc.off_trans != 0, sc.off_on_left});
    } else if (dry_) {
    } else if (sc.off_on_left)
      enqueue_gemm<T>(coeff, sc.off_trans != 0, off, false, src, T(1), dst, s_, busy());
    else
      enqueue_gemm<T>(coeff, false, src, sc.off_trans != 0, off, T(1), dst, s_, busy());

    if (sc.first_a22) run(spec, a11, b1, row0);
    else run(spec, a22, b2, row0 + mid);
  }

 private:
  // TRMM calls with concurrent halves keep every GEMM on the large tiles (the
  // other half fills the GPU beside them); a TRSM is a serial chain.
  int busy() const { return conc != nullptr ? 1 : 0; }
  bool conc_node(const Schema& sc, i64 mid, i64 rhs, DView<T> dst) {
    if (!conc || dry_ || kernels || op_ != kTrmm || mid * rhs > conc->max_elems) return false;
    if (sc.first_a22 != sc.write_b2) return false;  // first half must be the GEMM's destination
    return conc->next_stream < conc->streams->size() && conc->used + dst.rows * dst.cols <= conc->cap;
  }

  void run_concurrent(const Spec& spec, const Schema& sc, DView<const T> a11, DView<const T> a22,
                      DView<const T> off, DView<T> b1, DView<T> b2, DView<T> dst, DView<const T> src,
                      T coeff, i64 mid, i64 row0) {
    cudaStream_t s2 = (*conc->streams)[conc->next_stream++];
    cudaEvent_t fork = conc->event();
    cudaEvent_t join = conc->event();
    const DView<T> S{conc->scratch + conc->used, dst.rows, dst.rows, dst.cols};
    conc->used += dst.rows * dst.cols;
    cuda_check(cudaEventRecord(fork, s_), "record fork");
    cuda_check(cudaStreamWaitEvent(s2, fork, 0), "wait fork");
    // host call order (events, leaf numbering) is the serial one
    if (sc.first_a22) run(spec, a22, b2, row0 + mid);
    else run(spec, a11, b1, row0);
    emit(RECTRI_CU_EV_GEMM, dst.rows, dst.cols);
    if (before) before(false, off, sc.read_b2 ? b2 : b1, dst);
    if (sc.off_on_left)
      enqueue_gemm<T>(T(1), sc.off_trans != 0, off, false, src, T(0), S, s2, 1);
    else
      enqueue_gemm<T>(T(1), false, src, sc.off_trans != 0, off, T(0), S, s2, 1);
    cudaStream_t s1 = s_;
    s_ = s2;
    if (sc.first_a22) run(spec, a11, b1, row0);
    else run(spec, a22, b2, row0 + mid);
    s_ = s1;
    cuda_check(cudaEventRecord(join, s2), "record join");
    cuda_check(cudaStreamWaitEvent(s_, join, 0), "wait join");
    K<T>::accumulate(dst.p, dst.ld, S.p, dst.rows, dst.cols, coeff, s_);
  }

  void emit(int32_t e, i64 n, i64 m) {
    if (events_) events_->push_back(Ev{e, n, m});
  }
  OpK op_;
  i64 threshold_;
  cudaStream_t s_;
  std::vector<Ev>* events_;
  std::vector<std::pair<i64, i64>>* leaves_;
  bool dry_;
};

// The leaf problem of a base call in the Left form on L' (base_kernels.cpp:35-47, 152-155).
template <typename T>
LeafParams<T> leaf_params(OpK op, const Spec& spec, DView<const T> A, DView<T> B) {
  const bool left = spec.side == RECTRI_CU_LEFT;
  const int eff = left ? spec.trans : 1 - spec.trans;
  LeafParams<T> p;
  p.n = static_cast<int>(A.rows);
  p.nrhs = left ? B.cols : B.rows;
  p.A = A.p;
  p.lda = A.ld;
  p.B = B.p;
  p.ldb = B.ld;
  p.right = left ? 0 : 1;
  p.reflected = (spec.uplo == RECTRI_CU_LOWER) == (eff == 1) ? 1 : 0;
  p.swapped = eff == 1 ? 1 : 0;
  p.unit = spec.diag == RECTRI_CU_UNIT ? 1 : 0;
  p.trsm = op == kTrsm ? 1 : 0;
  p.alpha = static_cast<T>(spec.alpha);
  return p;
}

template <typename T>
void enqueue_base(OpK op, const Spec& spec, DView<const T> A, DView<T> B, cudaStream_t s, double* packed,
                  int pack_asc, int direct) {
  const i64 n = A.rows;
  const bool left = spec.side == RECTRI_CU_LEFT;
  const i64 rhs = left ? B.cols : B.rows;
  if (n == 0 || rhs == 0) return;
  if (n > kLeafMax) {
    Recursion<T>(op, kLeafMax, s, nullptr, nullptr).run(spec, A, B, 0);
    return;
  }
  // Right is Left on the transposed problem with op flipped (base_kernels.cpp:152-155).
  const int eff = left ? spec.trans : 1 - spec.trans;
  LeafParams<T> p;
  p.n = static_cast<int>(n);
  p.nrhs = rhs;
  p.A = A.p;
  p.lda = A.ld;
  p.B = B.p;
  p.ldb = B.ld;
  p.right = left ? 0 : 1;
  p.reflected = (spec.uplo == RECTRI_CU_LOWER) == (eff == 1) ? 1 : 0;
  p.swapped = eff == 1 ? 1 : 0;
  p.unit = spec.diag == RECTRI_CU_UNIT ? 1 : 0;
  p.trsm = op == kTrsm ? 1 : 0;
  p.alpha = static_cast<T>(spec.alpha);
  p.packed = packed;
  p.pack_asc = pack_asc;
  p.direct = direct;
  ProfScope prof(1, static_cast<double>(n) * n * rhs, s);
  K<T>::leaf(p, s);
}

// ---------------------------------------------------------------------------
// Per-device resources: capture stream and a staging pool for host views.
struct DeviceRes {
  static constexpr int kAux = 3;  // extra streams of the right-hand-side panel split
  cudaStream_t capture = nullptr;
  cudaStream_t aux[kAux] = {nullptr, nullptr, nullptr};
  cudaStream_t h2d = nullptr, d2h = nullptr;  // copy streams of the staged path
  std::vector<cudaStream_t> conc_streams;      // concurrent TRMM nodes (ConcCtx), graph captures (under g_mu)
  std::vector<cudaStream_t> conc_streams_dir;  // the same for direct-launch calls
  cudaStream_t scan_cap = nullptr, scan_dir = nullptr;  // zero-pivot scan beside the recursion
  static constexpr int kSlots = 3;            // 0: A, 1..2: B panels
  void* stage[kSlots] = {nullptr, nullptr, nullptr};
  size_t stage_bytes[kSlots] = {0, 0, 0};
  // Held for a whole host-operand call: the staging buffers (and the copy
  // streams) serve one call at a time, and are never reallocated or released
  // under a call that is still using them.
  std::mutex stage_mu;
};

std::mutex g_mu;
std::map<int, DeviceRes> g_dev;

DeviceRes& device_res(int dev) {
  DeviceRes& r = g_dev[dev];
  if (!r.capture) {
    cuda_check(cudaStreamCreateWithFlags(&r.capture, cudaStreamNonBlocking), "stream");
    cuda_check(cudaStreamCreateWithFlags(&r.h2d, cudaStreamNonBlocking), "stream");
    cuda_check(cudaStreamCreateWithFlags(&r.d2h, cudaStreamNonBlocking), "stream");
    for (auto& a : r.aux) cuda_check(cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking), "stream");
    r.conc_streams.resize(16);
    for (auto& a : r.conc_streams) cuda_check(cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking), "stream");
    cuda_check(cudaStreamCreateWithFlags(&r.scan_cap, cudaStreamNonBlocking), "stream");
    cuda_check(cudaStreamCreateWithFlags(&r.scan_dir, cudaStreamNonBlocking), "stream");
    r.conc_streams_dir.resize(16);
    for (auto& a : r.conc_streams_dir) cuda_check(cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking), "stream");
  }
  return r;
}

// Concurrent TRMM nodes (ConcCtx), on unless RECTRI_CU_TRMM_CONC=0.
bool conc_enabled() {
  const char* e = getenv("RECTRI_CU_TRMM_CONC");
  return !(e && atoi(e) == 0);
}

// Streams the right-hand sides are split over (RECTRI_CU_STREAMS, default 2;
// panels narrower than 2048 right-hand sides are not split).
// Right-hand-side streams of a call: `pref` (RECTRI_CU_STREAMS overrides),
// fewer when the panels would drop below RECTRI_CU_PANEL_MIN columns.
int panel_streams(i64 rhs, int pref = 2) {
  const char* e = getenv("RECTRI_CU_STREAMS");
  int p = e ? atoi(e) : pref;
  if (p > DeviceRes::kAux + 1) p = DeviceRes::kAux + 1;
  const char* w = getenv("RECTRI_CU_PANEL_MIN");
  const i64 min_w = w && atoll(w) > 0 ? atoll(w) : 2048;
  while (p > 1 && rhs / p < min_w) --p;
  return p < 1 ? 1 : p;
}

// Device-resident graphs: three right-hand-side streams for fp64 calls with
// >= 8192 right-hand sides, two otherwise (fp64 small_probe, one B200:
// TRMM n = m = 8192 16036 -> 15972 us, 16384 124147 -> 123871 us; TRSM 8192
// 16110 -> 16075, 16384 124340 -> 124193; at 4096 a third stream costs TRMM
// 3 %; fp32 and the streamed host path keep two; profiles/r02_streams*.txt).
template <typename T>
int device_streams_pref(i64 rhs) {
  return sizeof(T) == 8 && rhs >= 8192 ? 3 : 2;
}

void* staging(DeviceRes& r, int slot, size_t bytes) {
  if (r.stage_bytes[slot] < bytes) {
    if (r.stage[slot]) cudaFree(r.stage[slot]);
    r.stage[slot] = nullptr;
    r.stage_bytes[slot] = 0;
    cuda_check(cudaMalloc(&r.stage[slot], bytes), "staging alloc");
    r.stage_bytes[slot] = bytes;
  }
  return r.stage[slot];
}

// ---------------------------------------------------------------------------
// Graph cache.
struct GraphEntry {
  cudaGraphExec_t exec = nullptr;
  std::vector<Ev> events;
  std::vector<std::pair<i64, i64>> leaves;
  uint8_t* d_flags = nullptr;
  uint8_t* h_flags = nullptr;
  double* packed = nullptr;  // fp64 leaf triangles, packed once per call
  void* leaf_meta = nullptr;  // their row offsets and orders
  void* conc_scratch = nullptr;  // concurrent TRMM nodes' GEMM products
  CallScratch scratch;           // unpacked-leaf and 3xTF32 split buffers of the captured kernels
  size_t bytes = 0;              // device bytes this entry owns (graph-cache byte cap)
  i64 nodes = 0;
  int device = 0;
  ~GraphEntry() {
    if (exec) cudaGraphExecDestroy(exec);
    for (int k = 0; k < scratch.n; ++k) {
      if (scratch.leaf[k]) cudaFree(scratch.leaf[k]);
      if (scratch.split[k]) cudaFree(scratch.split[k]);
    }
    if (packed) cudaFree(packed);
    if (leaf_meta) cudaFree(leaf_meta);
    if (conc_scratch) cudaFree(conc_scratch);
    if (d_flags) cudaFree(d_flags);
    if (h_flags) cudaFreeHost(h_flags);
  }
};

using Key = std::tuple<int, int, int, int, int, int, uint64_t, const void*, i64, i64, void*, i64,
                       i64, i64, i64, int>;

// LRU of captured calls, bounded by entry count AND by the device bytes the
// entries own (packed leaf triangles, TRMM scratch, graph-owned leaf/split
// scratch): RECTRI_CU_GRAPH_CACHE_MB (default 4096).  The newest entry is
// always kept.  Entries are shared_ptr: an evicted entry still referenced by
// a pending ASYNC call lives until that call is synced.
struct Cache {
  std::list<std::pair<Key, std::shared_ptr<GraphEntry>>> lru;
  std::map<Key, decltype(lru)::iterator> index;
  static constexpr size_t kCap = 64;
  size_t bytes = 0;
  static size_t byte_cap() {
    static const size_t cap = [] {
      const char* e = getenv("RECTRI_CU_GRAPH_CACHE_MB");
      return (e && atoll(e) > 0 ? static_cast<size_t>(atoll(e)) : size_t{4096}) << 20;
    }();
    return cap;
  }
  std::shared_ptr<GraphEntry> get(const Key& k) {
    auto it = index.find(k);
    if (it == index.end()) return nullptr;
    lru.splice(lru.begin(), lru, it->second);
    return it->second->second;
  }
  void put(const Key& k, std::shared_ptr<GraphEntry> e) {
    bytes += e->bytes;
    lru.emplace_front(k, std::move(e));
    index[k] = lru.begin();
    bool evicted = false;
    while (lru.size() > 1 && (lru.size() > kCap || bytes > byte_cap())) {
      bytes -= lru.back().second->bytes;
      index.erase(lru.back().first);
      // replays of an evicted graph may still be in flight on some stream:
      // finish them before its memory and executable are released
      if (!evicted) cudaDeviceSynchronize();
      evicted = true;
      lru.pop_back();
    }
  }
  void clear() {
    if (!lru.empty()) cudaDeviceSynchronize();
    index.clear();
    lru.clear();
    bytes = 0;
  }
};
Cache g_cache;

// Pending singularity checks for RECTRI_CU_ASYNC calls, per stream.  At most
// kMaxPending per stream: beyond that the stream is synchronized and the
// checks settled early, the first singular row kept in g_deferred until the
// caller's rectri_cu_sync reports it.
std::multimap<cudaStream_t, std::shared_ptr<GraphEntry>> g_pending;
std::map<cudaStream_t, i64> g_deferred;
constexpr size_t kMaxPending = 256;

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (dev >= 0 && dev != prev) cuda_check(cudaSetDevice(dev), "cudaSetDevice");
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

i64 first_singular(const GraphEntry& g) {
  for (const auto& leaf : g.leaves)
    for (i64 r = leaf.first; r < leaf.first + leaf.second; ++r)
      if (g.h_flags[r]) return r;
  return -1;
}

// Builds (captures) the whole device-side call: alpha pre-scale (TRSM,
// recursion.cpp:185-189), the zero-pivot pre-scan (TRSM NonUnit), and the
// recursion.  Runs on `s` directly when `capture` is false.
template <typename T>
std::shared_ptr<GraphEntry> build(OpK op, const Spec& spec, DView<const T> A, DView<T> B,
                                  i64 threshold, cudaStream_t s, bool capture, int dev) {
  auto g = std::make_shared<GraphEntry>();
  g->device = dev;
  const bool scan = op == kTrsm && spec.diag == RECTRI_CU_NONUNIT;
  if (scan) {
    cuda_check(cudaMalloc(&g->d_flags, static_cast<size_t>(A.rows)), "flags alloc");
    cuda_check(cudaMallocHost(&g->h_flags, static_cast<size_t>(A.rows)), "flags alloc");
  }
  Spec eff = spec;
  if (op == kTrsm) eff.alpha = 1.0;
  // fp64 v3 leaves: pack every leaf's triangle once, up front, for all
  // right-hand-side streams (allocations before any capture).
  LeafParams<T> pbase{};
  int nleaves = 0;
  {
    if (leaf_version() >= 3 && threshold <= kLeafMax && !(op == kTrmm && spec.alpha == 0.0)) {
      std::vector<std::pair<i64, i64>> lv;
      Recursion<T>(op, threshold, nullptr, nullptr, &lv, true).run(eff, A, B, 0);
      nleaves = static_cast<int>(lv.size());
      std::vector<long long> r0s(nleaves);
      std::vector<int> ns(nleaves);
      for (int k = 0; k < nleaves; ++k) {
        r0s[k] = lv[k].first;
        ns[k] = static_cast<int>(lv[k].second);
      }
      cuda_check(cudaMalloc(&g->packed, static_cast<size_t>(nleaves) * leaf3_scratch_doubles() * sizeof(double)),
                 "leaf pack alloc");
      g->bytes += static_cast<size_t>(nleaves) * leaf3_scratch_doubles() * sizeof(double);
      cuda_check(cudaMalloc(&g->leaf_meta, static_cast<size_t>(nleaves) * (sizeof(long long) + sizeof(int))),
                 "leaf meta alloc");
      long long* d_r0 = static_cast<long long*>(g->leaf_meta);
      int* d_n = reinterpret_cast<int*>(d_r0 + nleaves);
      cuda_check(cudaMemcpy(d_r0, r0s.data(), nleaves * sizeof(long long), cudaMemcpyHostToDevice), "leaf meta");
      cuda_check(cudaMemcpy(d_n, ns.data(), nleaves * sizeof(int), cudaMemcpyHostToDevice), "leaf meta");
      const bool left = spec.side == RECTRI_CU_LEFT;
      const int effop = left ? spec.trans : 1 - spec.trans;
      pbase.A = A.p;
      pbase.lda = A.ld;
      pbase.right = left ? 0 : 1;
      pbase.reflected = (spec.uplo == RECTRI_CU_LOWER) == (effop == 1) ? 1 : 0;
      pbase.swapped = effop == 1 ? 1 : 0;
      pbase.unit = spec.diag == RECTRI_CU_UNIT ? 1 : 0;
      pbase.trsm = op == kTrsm ? 1 : 0;
      pbase.alpha = static_cast<T>(eff.alpha);
      // fp64 TRMM leaves v4 / v5 read their triangles in ascending row order
      pbase.pack_asc = std::is_same<T, double>::value && op == kTrmm && leaf_trmm_asc() ? 1 : 0;
    }
  }
  // Concurrent TRMM nodes (ConcCtx): packed leaves only (no per-stream leaf
  // scratch), exact-FFMA fp32 only (3xTF32 keeps per-stream scratch).
  ConcCtx<T> conc;
  const bool left_ = spec.side == RECTRI_CU_LEFT;
  const i64 rhs_ = left_ ? B.cols : B.rows;
  const int P_ = g_prof.on ? 1 : panel_streams(rhs_, device_streams_pref<T>(rhs_));
  // Only where the GPU is not already full: n <= 4096 (fp64) / 8192 (fp32).
  i64 conc_max_n = sizeof(T) == 8 ? 4096 : 8192;
  if (const char* e = getenv("RECTRI_CU_TRMM_CONC_MAXN")) conc_max_n = atoll(e);
  if (op == kTrmm && nleaves > 0 && !g_prof.on && conc_enabled() && A.rows <= conc_max_n &&
      !(std::is_same<T, float>::value && tf32x3_enabled())) {
    const i64 w = P_ <= 1 ? rhs_ : ((rhs_ + P_ - 1) / P_ + 63) / 64 * 64;
    i64 need = 0;
    // At the largest concurrent sizes (fp64 4096, fp32 8192) only the deepest
    // nodes (their full-size halves already fill the GPU): fp64 TRMM n = 4096
    // 2239 -> 2203 us, fp32 n = 8192 11.71 -> 11.57 ms; smaller calls: every
    // node (fp32 n = 4096 with the cut: 1859 -> 1992 us).
    if (A.rows >= conc_max_n) conc.max_elems = i64(1) << 19;
    if (const char* e = getenv("RECTRI_CU_TRMM_CONC_ELEMS")) conc.max_elems = atoll(e);
    for (i64 r0 = 0; r0 < rhs_; r0 += w)
      need += Recursion<T>::conc_need(op, threshold, A.rows, std::min(w, rhs_ - r0), conc.max_elems);
    if (need > 0 && need * static_cast<i64>(sizeof(T)) <= (i64(512) << 20)) {
      DeviceRes* resp;
      if (capture) {  // the capture path already holds g_mu
        resp = &device_res(dev);
      } else {
        std::lock_guard<std::mutex> lock(g_mu);
        resp = &device_res(dev);
      }
      cuda_check(cudaMalloc(&g->conc_scratch, static_cast<size_t>(need) * sizeof(T)), "trmm scratch alloc");
      g->bytes += static_cast<size_t>(need) * sizeof(T);
      conc.streams = capture ? &resp->conc_streams : &resp->conc_streams_dir;
      conc.scratch = static_cast<T*>(g->conc_scratch);
      conc.cap = need;
    }
  }
  i64& counter = launch_counter();
  const i64 before = counter;
  struct ScratchScope {  // the graph's own scratch for the launchers, during the capture only
    explicit ScratchScope(const CallScratch* cs) { set_call_scratch(cs); }
    ~ScratchScope() { set_call_scratch(nullptr); }
  };
  std::unique_ptr<ScratchScope> scratch_scope;
  if (capture) {
    // Scratch of the kernels captured on each stream (s and the panel
    // streams), owned by this graph and allocated before the capture.
    DeviceRes& res = device_res(dev);  // the capture path holds g_mu
    const bool leaf_scratch = nleaves == 0 && leaf_version() >= 2;
    const bool split = std::is_same<T, float>::value && tf32x3_enabled();
    // 3xTF32 operand splits: hi + lo of the largest off-diagonal block and source half
    const i64 h = A.rows - A.rows / 2;
    const i64 pw = P_ <= 1 ? rhs_ : ((rhs_ + P_ - 1) / P_ + 63) / 64 * 64;  // a stream's panel
    const size_t split_need = 2 * static_cast<size_t>(h * h + h * std::min(pw, rhs_));
    CallScratch& cs = g->scratch;
    for (int k = 0; k < P_ && (leaf_scratch || split); ++k) {
      cs.stream[k] = k == 0 ? s : res.aux[k - 1];
      cs.n = k + 1;
      if (leaf_scratch) {
        cuda_check(cudaMalloc(&cs.leaf[k], leaf_scratch_bytes()), "leaf scratch alloc");
        g->bytes += leaf_scratch_bytes();
      }
      if (split) {
        cuda_check(cudaMalloc(&cs.split[k], split_need * sizeof(float)), "3xTF32 scratch alloc");
        cs.split_floats[k] = split_need;
        g->bytes += split_need * sizeof(float);
      }
    }
    scratch_scope = std::make_unique<ScratchScope>(&g->scratch);
    cuda_check(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal), "capture");
  }
  if (op == kTrsm && spec.alpha != 1.0) {
    ProfScope prof(2, 0.0, s);
    K<T>::scale(B.p, B.ld, B.rows, B.cols, static_cast<T>(spec.alpha), s);
  }
  if (nleaves > 0) {
    long long* d_r0 = static_cast<long long*>(g->leaf_meta);
    int* d_n = reinterpret_cast<int*>(d_r0 + nleaves);
    if constexpr (std::is_same<T, double>::value)
      launch_leaf3_pack_all(pbase, d_r0, d_n, nleaves, g->packed, s);
    else
      // slices at the same byte stride as the recursion's double* arithmetic
      launch_leaf32_pack_all(pbase, d_r0, d_n, nleaves, reinterpret_cast<float*>(g->packed),
                             2 * static_cast<long long>(leaf3_scratch_doubles()), s);
  }
  auto with_packs = [&](Recursion<T>& r) -> Recursion<T>& {
    if (nleaves > 0) {
      r.packed = g->packed;
      r.packed_stride = leaf3_scratch_doubles();
      r.pack_asc = pbase.pack_asc;
    }
    if (conc.scratch) r.conc = &conc;
    return r;
  };
  // The zero-pivot scan only reads A and its flags are read on the host after
  // the call: it runs on a side stream beside the recursion (joined at the
  // end) instead of ahead of it -- one kernel plus one D2H off every TRSM
  // NonUnit call's critical path.
  cudaEvent_t scan_ev[2] = {nullptr, nullptr};
  if (scan && g_prof.on) {
    ProfScope prof(3, 0.0, s);
    K<T>::scan(A.p, A.ld, A.rows, g->d_flags, s);
    cudaMemcpyAsync(g->h_flags, g->d_flags, static_cast<size_t>(A.rows), cudaMemcpyDeviceToHost, s);
  } else if (scan) {
    DeviceRes* rp;
    if (capture) {  // the capture path already holds g_mu
      rp = &device_res(dev);
    } else {
      std::lock_guard<std::mutex> lock(g_mu);
      rp = &device_res(dev);
    }
    cudaStream_t ss = capture ? rp->scan_cap : rp->scan_dir;
    for (auto& e : scan_ev) cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    cuda_check(cudaEventRecord(scan_ev[0], s), "record");
    cuda_check(cudaStreamWaitEvent(ss, scan_ev[0], 0), "wait");
    K<T>::scan(A.p, A.ld, A.rows, g->d_flags, ss);
    cudaMemcpyAsync(g->h_flags, g->d_flags, static_cast<size_t>(A.rows), cudaMemcpyDeviceToHost, ss);
    cuda_check(cudaEventRecord(scan_ev[1], ss), "record");
  }
  const bool left = spec.side == RECTRI_CU_LEFT;
  const i64 rhs = left ? B.cols : B.rows;
  const int P = g_prof.on ? 1 : panel_streams(rhs, device_streams_pref<T>(rhs));
  if (P <= 1) {
    Recursion<T> rec(op, threshold, s, &g->events, &g->leaves);
    with_packs(rec).run(eff, A, B, 0);
  } else {
    // Right-hand-side panels on P streams (fork/join inside the capture):
    // one panel's small kernels (leaves, short-K GEMMs) fill the SMs another
    // panel's kernel tails leave idle.  Kernels are independent of the
    // number of right-hand sides, so the result is bitwise the unsplit one;
    // events and leaf order are those of the single logical call.
    Recursion<T>(op, threshold, nullptr, &g->events, &g->leaves, true).run(eff, A, B, 0);
    DeviceRes* resp;
    if (capture) {  // the capture path already holds g_mu
      resp = &device_res(dev);
    } else {
      std::lock_guard<std::mutex> lock(g_mu);
      resp = &device_res(dev);
    }
    DeviceRes& res = *resp;
    std::vector<cudaEvent_t> evs;
    auto ev = [&]() {
      cudaEvent_t e;
      cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
      evs.push_back(e);
      return e;
    };
    cudaEvent_t fork = ev();
    cuda_check(cudaEventRecord(fork, s), "record fork");
    const i64 w = ((rhs + P - 1) / P + 63) / 64 * 64;
    for (int k = 0; k < P; ++k) {
      const i64 r0 = k * w;
      if (r0 >= rhs) break;
      const i64 wi = r0 + w <= rhs ? w : rhs - r0;
      const DView<T> panel = left ? B.sub(0, r0, B.rows, wi) : B.sub(r0, 0, wi, B.cols);
      cudaStream_t sk = k == 0 ? s : res.aux[k - 1];
      if (k > 0) cuda_check(cudaStreamWaitEvent(sk, fork, 0), "wait fork");
      Recursion<T> rec(op, threshold, sk, nullptr, nullptr);
      with_packs(rec).run(eff, A, panel, 0);
      if (k > 0) {
        cudaEvent_t join = ev();
        cuda_check(cudaEventRecord(join, sk), "record join");
        cuda_check(cudaStreamWaitEvent(s, join, 0), "wait join");
      }
    }
    for (cudaEvent_t e : evs) cudaEventDestroy(e);
  }
  if (scan_ev[1]) cuda_check(cudaStreamWaitEvent(s, scan_ev[1], 0), "wait scan");
  cudaError_t le = cudaGetLastError();
  for (cudaEvent_t e : scan_ev)
    if (e) cudaEventDestroy(e);
  if (capture) {
    cudaGraph_t graph = nullptr;
    cudaError_t ee = cudaStreamEndCapture(s, &graph);
    if (le != cudaSuccess) cuda_check(le, "launch during capture");
    cuda_check(ee, "end capture");
    cudaError_t ie = cudaGraphInstantiate(&g->exec, graph, 0);
    cudaGraphDestroy(graph);
    cuda_check(ie, "graph instantiate");
    g->nodes = counter - before;
    counter = before;  // counted when replayed
  } else {
    cuda_check(le, "kernel launch");
  }
  return g;
}

template <typename T>
int dtype_code();
template <>
int dtype_code<double>() { return 1; }
template <>
int dtype_code<float>() { return 0; }

uint64_t bits_of(double a) {
  uint64_t b;
  std::memcpy(&b, &a, sizeof b);
  return b;
}

// Enqueues one device-resident recursive call (both views on the device of
// `dev`) on `stream`: from the graph cache (captured on first use) or by
// direct launches.  Replays the call's events to `sink` when given.
template <typename T>
std::shared_ptr<GraphEntry> enqueue_device(OpK op, const Spec& spec, DView<const T> A, DView<T> B,
                                           i64 threshold, cudaStream_t stream, unsigned flags,
                                           rectri_cu_event_fn sink, void* user, int dev) {
  std::shared_ptr<GraphEntry> g;
  if ((flags & RECTRI_CU_NO_GRAPH) || g_prof.on) {
    g = build<T>(op, spec, A, B, threshold, stream, false, dev);
    for (const Ev& e : g->events)
      if (sink) sink(user, e.e, e.n, e.m);
    return g;
  }
  const int mode = dtype_code<T>() + (std::is_same<T, float>::value && tf32x3_enabled() ? 10 : 0);
  const Key key{static_cast<int>(op), mode, spec.side, spec.uplo, spec.trans,
                spec.diag, bits_of(spec.alpha), static_cast<const void*>(A.p), A.ld, A.rows,
                static_cast<void*>(B.p), B.ld, B.rows, B.cols, threshold, dev};
  {
    std::lock_guard<std::mutex> lock(g_mu);
    g = g_cache.get(key);
    if (!g) {
      DeviceRes& res = device_res(dev);
      g = build<T>(op, spec, A, B, threshold, res.capture, true, dev);
      g_cache.put(key, g);
    }
  }
  for (const Ev& e : g->events)
    if (sink) sink(user, e.e, e.n, e.m);
  cuda_check(cudaGraphLaunch(g->exec, stream), "graph launch");
  launch_counter() += g->nodes;
  return g;
}

void raise_if_singular(const GraphEntry& g) {
  if (!g.h_flags) return;
  const i64 r = first_singular(g);
  if (r >= 0) {
    Fail f{RECTRI_CU_SINGULAR, "singular triangular matrix: zero diagonal at row " + std::to_string(r)};
    f.index = r;
    throw f;
  }
}

// Device-resident recursive call: enqueue, then synchronize and report
// singularity (or defer both under RECTRI_CU_ASYNC).
template <typename T>
void run_device(OpK op, const Spec& spec, DView<const T> A, DView<T> B, i64 threshold,
                const BackendInfo& be, rectri_cu_event_fn sink, void* user, int dev,
                bool force_sync) {
  const bool async = (be.flags & RECTRI_CU_ASYNC) && !force_sync;
  std::shared_ptr<GraphEntry> g =
      enqueue_device<T>(op, spec, A, B, threshold, be.stream, be.flags, sink, user, dev);
  if (async) {
    if (g->h_flags) {
      std::vector<std::shared_ptr<GraphEntry>> settle;
      {
        std::lock_guard<std::mutex> lock(g_mu);
        g_pending.emplace(be.stream, g);
        if (g_pending.count(be.stream) > kMaxPending) {
          auto range = g_pending.equal_range(be.stream);
          for (auto it = range.first; it != range.second; ++it) settle.push_back(it->second);
          g_pending.erase(be.stream);
        }
      }
      if (!settle.empty()) {
        cuda_check(cudaStreamSynchronize(be.stream), "synchronize");
        i64 r = -1;
        for (const auto& e : settle)
          if (r < 0) r = first_singular(*e);
        if (r >= 0) {
          std::lock_guard<std::mutex> lock(g_mu);
          g_deferred.emplace(be.stream, r);  // keeps the earliest
        }
      }
    }
    return;
  }
  cuda_check(cudaStreamSynchronize(be.stream), "synchronize");
  raise_if_singular(*g);
}

// Copies the stored triangle of a host n x n A (the only part the kernels
// ever read: uplo triangle incl. diagonal) into a dense device n x n buffer,
// as column-block trapezoids.
template <typename T>
void copy_triangle_h2d(T* dA, const DView<const T>& A, int uplo, cudaStream_t s) {
  const i64 n = A.rows;
  constexpr i64 kW = 512;
  for (i64 c0 = 0; c0 < n; c0 += kW) {
    const i64 w = c0 + kW < n ? kW : n - c0;
    const i64 r0 = uplo == RECTRI_CU_LOWER ? c0 : 0;
    const i64 r1 = uplo == RECTRI_CU_LOWER ? n : c0 + w;
    cuda_check(cudaMemcpy2DAsync(dA + c0 * n + r0, sizeof(T) * n, A.p + c0 * A.ld + r0, sizeof(T) * A.ld,
                                 sizeof(T) * (r1 - r0), w, cudaMemcpyHostToDevice, s),
               "H2D A");
  }
}

// Host-resident B: the right-hand sides are cut into panels; H2D of panel
// i+1, the recursion on panel i and D2H of panel i-1 run concurrently on
// three streams (two device panel slots).  Kernels are independent of the
// number of right-hand sides, so the result is bitwise the unpanelled one;
// the event sink sees the single logical call.
template <typename T>
void run_host_panels(OpK op, const Spec& spec, DView<const T> dA, DView<T> hB, i64 threshold,
                     const BackendInfo& be, rectri_cu_event_fn sink, void* user, int dev,
                     cudaEvent_t a_ready) {
  const bool left = spec.side == RECTRI_CU_LEFT;
  const i64 n = dA.rows;
  const i64 rhs = left ? hB.cols : hB.rows;
  // Panel width: a few panels for overlap, none narrower than 2048
  // (RECTRI_CU_HOST_PANEL overrides, for tuning).
  i64 w = (rhs + 3) / 4;
  if (w < 2048) w = 2048;
  if (const char* e = getenv("RECTRI_CU_HOST_PANEL")) w = atoll(e) > 0 ? atoll(e) : w;
  if (w > rhs) w = rhs;
  const i64 np = (rhs + w - 1) / w;

  // Events of the single logical call (recursion.cpp:94, 97, 139).
  if (sink) {
    std::vector<Ev> evs;
    Spec eff = spec;
    Recursion<T>(op, threshold, nullptr, &evs, nullptr, true)
        .run(eff, dA, DView<T>{nullptr, hB.ld, hB.rows, hB.cols}, 0);
    for (const Ev& e : evs) sink(user, e.e, e.n, e.m);
  }

  DeviceRes* res;
  T* slot[2];
  {
    std::lock_guard<std::mutex> lock(g_mu);
    res = &device_res(dev);
    for (int k = 0; k < 2; ++k)
      slot[k] = static_cast<T*>(staging(*res, 1 + k, static_cast<size_t>(n * w) * sizeof(T)));
  }
  cudaStream_t cs = be.stream, hs = res->h2d, ds = res->d2h;
  std::vector<cudaEvent_t> evs;
  auto ev = [&]() {
    cudaEvent_t e;
    cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    evs.push_back(e);
    return e;
  };
  cudaEvent_t slot_free[2] = {nullptr, nullptr};
  std::shared_ptr<GraphEntry> first;
  try {
    if (a_ready) cuda_check(cudaStreamWaitEvent(hs, a_ready, 0), "wait A");
    for (i64 i = 0; i < np; ++i) {
      const i64 r0 = i * w, wi = r0 + w <= rhs ? w : rhs - r0;
      const int k = static_cast<int>(i & 1);
      // panel i in the slot's own packed layout (Left: n x wi, Right: wi x n)
      const DView<T> d = left ? DView<T>{slot[k], n, n, wi} : DView<T>{slot[k], wi, wi, n};
      const T* hsrc = left ? hB.p + r0 * hB.ld : hB.p + r0;
      if (slot_free[k]) cuda_check(cudaStreamWaitEvent(hs, slot_free[k], 0), "wait slot");
      cuda_check(cudaMemcpy2DAsync(d.p, sizeof(T) * d.ld, hsrc, sizeof(T) * hB.ld, sizeof(T) * d.rows,
                                   d.cols, cudaMemcpyHostToDevice, hs),
                 "H2D B panel");
      cudaEvent_t in = ev();
      cuda_check(cudaEventRecord(in, hs), "record");
      cuda_check(cudaStreamWaitEvent(cs, in, 0), "wait panel");
      auto g = enqueue_device<T>(op, spec, dA, d, threshold, cs, be.flags, nullptr, nullptr, dev);
      if (!first) first = g;
      cudaEvent_t done = ev();
      cuda_check(cudaEventRecord(done, cs), "record");
      cuda_check(cudaStreamWaitEvent(ds, done, 0), "wait compute");
      cuda_check(cudaMemcpy2DAsync(const_cast<T*>(hsrc), sizeof(T) * hB.ld, d.p, sizeof(T) * d.ld,
                                   sizeof(T) * d.rows, d.cols, cudaMemcpyDeviceToHost, ds),
                 "D2H B panel");
      slot_free[k] = ev();
      cuda_check(cudaEventRecord(slot_free[k], ds), "record");
    }
    cuda_check(cudaStreamSynchronize(ds), "synchronize");
    cuda_check(cudaStreamSynchronize(cs), "synchronize");
  } catch (...) {
    cudaStreamSynchronize(ds);
    cudaStreamSynchronize(cs);
    for (cudaEvent_t e : evs) cudaEventDestroy(e);
    throw;
  }
  for (cudaEvent_t e : evs) cudaEventDestroy(e);
  if (first) raise_if_singular(*first);
}

// Host-resident B (and optionally A), whole problem resident on the device:
// A's blocks and B's row chunks (Right side: column chunks) are copied H2D in
// the order the recursion first touches them, each kernel waits only for its
// own inputs, and each B chunk is copied back as soon as its last writer has
// run -- so the transfers hide under the compute except the first chunk's
// copy-in and the last chunk's copy-back.  GEMM updates whose destination
// spans several chunks are split at chunk boundaries (a split of the M
// dimension -- Right side: N -- never changes an element's arithmetic), so
// e.g. the level-1 update starts on the first chunk that has arrived.  Same
// kernels, same per-element order as the device path (bitwise the same
// result); the event sink sees the single logical call.  Returns false
// (nothing done) when the device cannot hold the problem; the caller then
// uses run_host_panels.
template <typename T>
bool run_host_streamed(OpK op, const Spec& spec, DView<const T> A, bool a_dev, DView<T> hB, i64 threshold,
                       const BackendInfo& be, rectri_cu_event_fn sink, void* user, int dev,
                       PageableStager* pg = nullptr) {
  const auto entry_t0 = std::chrono::steady_clock::now();
  std::chrono::steady_clock::time_point tmark[3];  // RECTRI_CU_E2E_TRACE: setup phases
  const bool left = spec.side == RECTRI_CU_LEFT;
  const i64 n = A.rows, brows = hB.rows, bcols = hB.cols;
  const size_t bbytes = static_cast<size_t>(brows * bcols) * sizeof(T);
  const size_t abytes = a_dev ? 0 : static_cast<size_t>(n * n) * sizeof(T);
  DeviceRes* res;
  T* dAp = nullptr;
  T* dBp = nullptr;
  {
    std::lock_guard<std::mutex> lock(g_mu);
    res = &device_res(dev);
    // Query free memory only when the staging buffers must grow: on a busy
    // box cudaMemGetInfo took 0.1-72 ms per call (e2e trace), the largest
    // source of the end-to-end step variance.
    const size_t have = (a_dev ? 0 : res->stage_bytes[0]) + res->stage_bytes[1];
    if (abytes > (a_dev ? 0 : res->stage_bytes[0]) || bbytes > res->stage_bytes[1]) {
      size_t free_b = 0, total_b = 0;
      cudaMemGetInfo(&free_b, &total_b);
      const size_t room = free_b + have > (size_t{1} << 30) ? free_b + have - (size_t{1} << 30) : 0;
      if (abytes + bbytes > room) return false;
    }
    tmark[0] = std::chrono::steady_clock::now();
    if (!a_dev) dAp = static_cast<T*>(staging(*res, 0, abytes));
    dBp = static_cast<T*>(staging(*res, 1, bbytes));
  }
  tmark[1] = std::chrono::steady_clock::now();
  const DView<const T> dA = a_dev ? A : DView<const T>{dAp, n, n, n};
  const DView<T> dB{dBp, brows, brows, bcols};
  Spec eff = spec;
  if (op == kTrsm) eff.alpha = 1.0;

  // Descriptor run: the recursion's kernels in order (and its events, leaves).
  std::vector<Ev> evs_logical;
  std::vector<std::pair<i64, i64>> leaves;
  std::vector<KDesc<T>> ks;
  {
    Recursion<T> dry(op, threshold, nullptr, &evs_logical, &leaves, true);
    dry.kernels = [&](const KDesc<T>& k) { ks.push_back(k); };
    dry.run(eff, dA, dB, 0);
  }
  tmark[2] = std::chrono::steady_clock::now();
  if (sink)
    for (const Ev& e : evs_logical) sink(user, e.e, e.n, e.m);

  // B chunks along the triangle dimension: consecutive leaves merged to
  // >= 1024 rows (columns, Right).
  std::vector<std::pair<i64, i64>> lv = leaves;
  std::sort(lv.begin(), lv.end());
  std::vector<i64> cb{0};
  const char* ce = getenv("RECTRI_CU_E2E_CHUNK");  // tuning knob (rows per chunk)
  const i64 chunk_min = ce && atoll(ce) > 0 ? atoll(ce) : 1024;
  for (const auto& l : lv) {
    // small chunks at both ends of the triangle dimension: the first copy-in
    // and the last copy-back are the transfers no compute hides
    const i64 end = l.first + l.second;
    const i64 want = (end <= chunk_min || end > n - chunk_min) ? chunk_min / 4 : chunk_min;
    if (end - cb.back() >= want || end == n) cb.push_back(end);
  }
  const int nch = static_cast<int>(cb.size()) - 1;
  auto off_of = [&](const T* p) { return left ? static_cast<i64>(p - dB.p) : static_cast<i64>(p - dB.p) / dB.ld; };
  auto len_of = [&](const DView<T>& v) { return left ? v.rows : v.cols; };
  auto chunk_of = [&](i64 r) {
    return static_cast<int>(std::upper_bound(cb.begin(), cb.end(), r) - cb.begin()) - 1;
  };
  auto b_chunk = [&](DView<T> base, int c) {
    return left ? base.sub(cb[c], 0, cb[c + 1] - cb[c], bcols) : base.sub(0, cb[c], brows, cb[c + 1] - cb[c]);
  };

  // Unit kernels: leaves as they are, GEMMs split at dst chunk boundaries.
  struct Unit {
    const KDesc<T>* k;
    DView<const T> a;  // the A block this unit reads (GEMM: its slice of off)
    DView<T> dst;      // the B range it writes
    i64 s0, s1;        // B range it reads besides dst (GEMM src), triangle coords
  };
  std::vector<Unit> units;
  for (const KDesc<T>& k : ks) {
    if (k.leaf) {
      units.push_back(Unit{&k, k.a, k.dst, 0, 0});
      continue;
    }
    const i64 d0 = off_of(k.dst.p), dl = len_of(k.dst);
    const i64 s0 = off_of(k.src.p), s1 = s0 + len_of(k.src);
    for (int c = chunk_of(d0); c < nch && cb[c] < d0 + dl; ++c) {
      const i64 lo = std::max(cb[c], d0) - d0, hi = std::min(cb[c + 1], d0 + dl) - d0;
      const i64 h = hi - lo;
      DView<T> dsub = left ? k.dst.sub(lo, 0, h, k.dst.cols) : k.dst.sub(0, lo, k.dst.rows, h);
      // slice of op(off) feeding those dst rows (Left) / columns (Right)
      DView<const T> asub = left ? (k.off_trans ? k.a.sub(0, lo, k.a.rows, h) : k.a.sub(lo, 0, h, k.a.cols))
                                 : (k.off_trans ? k.a.sub(lo, 0, h, k.a.cols) : k.a.sub(0, lo, k.a.rows, h));
      units.push_back(Unit{&k, asub, dsub, s0, s1});
    }
  }
  std::vector<int> last_writer(nch, -1);
  for (int i = 0; i < static_cast<int>(units.size()); ++i) {
    const i64 w0 = off_of(units[i].dst.p), w1 = w0 + len_of(units[i].dst);
    for (int c = chunk_of(w0); c < nch && cb[c] < w1; ++c) last_writer[c] = i;
  }

  const bool scan = op == kTrsm && spec.diag == RECTRI_CU_NONUNIT;
  uint8_t* d_flags = nullptr;
  uint8_t* h_flags = nullptr;
  std::vector<uint8_t> flags;
  cudaStream_t cs = be.stream, hs = res->h2d, ds = res->d2h;
  std::vector<cudaEvent_t> evs;
  auto ev = [&]() {
    cudaEvent_t e;
    cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    evs.push_back(e);
    return e;
  };
  // RECTRI_CU_E2E_NOCOPY=1 (timing experiments only; the result is garbage):
  // skip every transfer, leaving the streamed path's compute schedule alone.
  static const bool nocopy = getenv("RECTRI_CU_E2E_NOCOPY") != nullptr;
  auto copy2d = [&](T* dst, i64 dld, const T* src, i64 sld, i64 rows, i64 cols, cudaMemcpyKind kind,
                    cudaStream_t st) {
    if (nocopy) return;
    if (pg && kind == cudaMemcpyHostToDevice && pg->covers(src)) {  // pageable source: pinned bounce
      pg->h2d(dst, sizeof(T) * dld, src, sizeof(T) * sld, sizeof(T) * rows, cols, st);
      return;
    }
    if (pg && kind == cudaMemcpyDeviceToHost && pg->covers(dst)) {
      pg->d2h(dst, sizeof(T) * dld, src, sizeof(T) * sld, sizeof(T) * rows, cols, st);
      return;
    }
    cuda_check(cudaMemcpy2DAsync(dst, sizeof(T) * dld, src, sizeof(T) * sld, sizeof(T) * rows, cols, kind, st),
               "staged copy");
  };
  const bool trace = getenv("RECTRI_CU_E2E_TRACE") != nullptr;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> d2h_marks;
  try {
    cudaEvent_t start;
    cuda_check(cudaEventCreate(&start), "event");  // timed (RECTRI_CU_E2E_TRACE)
    evs.push_back(start);
    cuda_check(cudaEventRecord(start, cs), "record");  // staging buffers free (stream order)
    const auto host_t0 = std::chrono::steady_clock::now();
    cuda_check(cudaStreamWaitEvent(hs, start, 0), "wait");
    if (scan && a_dev) {
      cuda_check(cudaMalloc(&d_flags, static_cast<size_t>(n)), "flags alloc");
      cuda_check(cudaMallocHost(&h_flags, static_cast<size_t>(n)), "flags alloc");
      K<T>::scan(A.p, A.ld, n, d_flags, cs);
      cuda_check(cudaMemcpyAsync(h_flags, d_flags, static_cast<size_t>(n), cudaMemcpyDeviceToHost, cs), "flags");
    }
    // Right-hand sides in TP consecutive time panels (RECTRI_CU_E2E_PANELS;
    // default: ~8192-wide panels): panel t's chunks are copied back
    // while panel t+1 computes, so only the last panel's last rows are left
    // for the tail (C3: compute done 132.3 -> 130.2 ms, tail 6.6 -> 3.3 ms,
    // e2e 139.3 -> 134.3 ms; 4 panels: tail 1.4 ms but the narrower GEMMs
    // finish at 137 ms.  C5 slice n = 8192, 65536 columns: 1 / 2 / 4 / 8
    // panels 178 / 155 / 144 / 143 ms).  Within a panel the right-hand sides are split over P
    // streams as in the device path.  Arithmetic is per right-hand side, so
    // the result is bitwise the single-panel one.
    const i64 rhs = left ? bcols : brows;
    int TP = static_cast<int>(std::max<i64>(1, std::min<i64>(16, rhs / 8192)));
    if (const char* te = getenv("RECTRI_CU_E2E_PANELS")) TP = std::max(1, atoi(te));
    // Panel boundaries: TP equal panels, or (RECTRI_CU_E2E_FIRST, tuning)
    // a first panel of that width and TP - 1 equal ones after it.
    std::vector<i64> tb{0};
    {
      const char* fe = getenv("RECTRI_CU_E2E_FIRST");
      const i64 first = fe && TP > 1 ? std::min<i64>(rhs, (atoll(fe) + 63) / 64 * 64) : 0;
      if (first > 0) tb.push_back(first);
      const int rest = first > 0 ? TP - 1 : TP;
      const i64 w = (rhs - tb.back() + rest - 1) / rest;
      while (tb.back() < rhs) tb.push_back(std::min(rhs, tb.back() + w));
    }
    auto window = [&](DView<T> v, i64 r0, i64 r1) {
      return left ? v.sub(0, r0, v.rows, r1 - r0) : v.sub(r0, 0, r1 - r0, v.cols);
    };
    // fp64 v3 leaves: each leaf's triangle packed once (stream 0, after its
    // A block has arrived), shared by every stream's and panel's leaf launch.
    double* packs = nullptr;
    const bool pack_once = std::is_same<T, double>::value && leaf_version() >= 3 && threshold <= kLeafMax &&
                           !(op == kTrmm && spec.alpha == 0.0);
    if (pack_once) {
      std::lock_guard<std::mutex> lock(g_mu);
      packs = static_cast<double*>(staging(*res, 2, leaves.size() * leaf3_scratch_doubles() * sizeof(double)));
    }
    std::vector<cudaEvent_t> packed_evs(units.size(), nullptr);
    // TRMM triangles in the v4 / v5 leaves' ascending order
    const int pack_asc = pack_once && op == kTrmm && leaf_trmm_asc() ? 1 : 0;
    for (int tp = 0; tp + 1 < static_cast<int>(tb.size()); ++tp) {
      const i64 t0 = tb[tp], t1 = tb[tp + 1];
      // H2D in first-use order (A blocks in the first panel); ready[i] gates unit i.
      std::vector<cudaEvent_t> ready(units.size(), nullptr);
      std::vector<std::vector<int>> fresh(units.size());  // chunks first loaded for unit i
      std::vector<char> loaded(nch, 0);
      for (size_t i = 0; i < units.size(); ++i) {
        const Unit& u = units[i];
        bool issued = false;
        if (!a_dev && tp == 0) {  // device sub-view; the host block sits at the same offsets
          const i64 off = static_cast<i64>(u.a.p - dA.p);
          copy2d(const_cast<T*>(u.a.p), n, A.p + off % n + (off / n) * A.ld, A.ld, u.a.rows, u.a.cols,
                 cudaMemcpyHostToDevice, hs);
          issued = true;
        }
        const i64 w0 = off_of(u.dst.p), w1 = w0 + len_of(u.dst);
        for (int pass = 0; pass < 2; ++pass) {
          const i64 r0 = pass ? u.s0 : w0, r1 = pass ? u.s1 : w1;
          for (int c = chunk_of(r0); r1 > r0 && c < nch && cb[c] < r1; ++c) {
            if (loaded[c]) continue;
            loaded[c] = 1;
            const DView<T> d = window(b_chunk(dB, c), t0, t1), h = window(b_chunk(hB, c), t0, t1);
            copy2d(d.p, d.ld, h.p, h.ld, d.rows, d.cols, cudaMemcpyHostToDevice, hs);
            fresh[i].push_back(c);
            issued = true;
          }
        }
        if (issued) {
          ready[i] = ev();
          cuda_check(cudaEventRecord(ready[i], hs), "record");
        }
      }
      if (scan && !a_dev && tp == 0) {  // host-side zero-pivot scan (trsm_base scans before writing)
        flags.resize(static_cast<size_t>(n));
        for (i64 r = 0; r < n; ++r) flags[r] = A.p[r + r * A.ld] == T(0) ? 1 : 0;
      }
      // Compute: each unit after its inputs, the panel's right-hand sides split
      // over P streams; chunk copy-back after its last writer on every stream.
      const i64 prhs = t1 - t0;
      const int P = panel_streams(prhs);
      const i64 pw = ((prhs + P - 1) / P + 63) / 64 * 64;
      std::vector<cudaStream_t> ps(P);
      for (int q = 0; q < P; ++q) ps[q] = q == 0 ? cs : res->aux[q - 1];
      if (P > 1) {
        cudaEvent_t fork = ev();
        cuda_check(cudaEventRecord(fork, cs), "record");
        for (int q = 1; q < P; ++q) cuda_check(cudaStreamWaitEvent(ps[q], fork, 0), "wait");
      }
      auto rhs_part = [&](DView<T> v, int q) {  // right-hand sides [t0 + q*pw, ...) of a B view
        const i64 r0 = t0 + q * pw, r1 = std::min(t1, r0 + pw);
        return window(v, r0, r1);
      };
      int leaf_k = 0;
      for (size_t i = 0; i < units.size(); ++i) {
        const Unit& u = units[i];
        const KDesc<T>& k = *u.k;
        double* packed = nullptr;
        if (pack_once && k.leaf) {
          packed = packs + static_cast<size_t>(leaf_k++) * leaf3_scratch_doubles();
          if (tp == 0) {
            if (ready[i]) cuda_check(cudaStreamWaitEvent(ps[0], ready[i], 0), "wait input");
            if constexpr (std::is_same<T, double>::value)
            {
              LeafParams<double> lp = leaf_params<double>(op, k.spec, k.a, k.dst);
              lp.pack_asc = pack_asc;
              launch_leaf3_pack(lp, packed, ps[0]);
            }
            packed_evs[i] = ev();
            cuda_check(cudaEventRecord(packed_evs[i], ps[0]), "record");
          }
        }
        for (int q = 0; q < P && q * pw < prhs; ++q) {
          cudaStream_t sq = ps[q];
          if (ready[i]) cuda_check(cudaStreamWaitEvent(sq, ready[i], 0), "wait input");
          if (packed_evs[i] && (q > 0 || tp > 0)) cuda_check(cudaStreamWaitEvent(sq, packed_evs[i], 0), "wait pack");
          if (op == kTrsm && spec.alpha != 1.0)  // alpha once per element, at first arrival
            for (int c : fresh[i]) {
              const DView<T> d = rhs_part(b_chunk(dB, c), q);
              K<T>::scale(d.p, d.ld, d.rows, d.cols, static_cast<T>(spec.alpha), sq);
            }
          const DView<T> dst = rhs_part(u.dst, q);
          if (k.leaf) {
            enqueue_base<T>(op, k.spec, k.a, dst, sq, packed, pack_asc);
          } else if (k.off_on_left) {
            enqueue_gemm<T>(k.coeff, k.off_trans, u.a, false, rhs_part(k.src, q), T(1), dst, sq);
          } else {
            enqueue_gemm<T>(k.coeff, false, rhs_part(k.src, q), k.off_trans, u.a, T(1), dst, sq);
          }
        }
        for (int c = 0; c < nch; ++c) {
          if (last_writer[c] != static_cast<int>(i)) continue;
          for (int q = 0; q < P && q * pw < prhs; ++q) {
            cudaEvent_t done = ev();
            cuda_check(cudaEventRecord(done, ps[q]), "record");
            cuda_check(cudaStreamWaitEvent(ds, done, 0), "wait");
          }
          const DView<T> d = window(b_chunk(dB, c), t0, t1), h = window(b_chunk(hB, c), t0, t1);
          if (trace) {
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            evs.push_back(e0);
            evs.push_back(e1);
            cudaEventRecord(e0, ds);
            copy2d(h.p, h.ld, d.p, d.ld, d.rows, d.cols, cudaMemcpyDeviceToHost, ds);
            cudaEventRecord(e1, ds);
            d2h_marks.push_back({c, {e0, e1}});
          } else {
            copy2d(h.p, h.ld, d.p, d.ld, d.rows, d.cols, cudaMemcpyDeviceToHost, ds);
          }
        }
      }
      for (int q = 1; q < P; ++q) {  // join
        cudaEvent_t join = ev();
        cuda_check(cudaEventRecord(join, ps[q]), "record");
        cuda_check(cudaStreamWaitEvent(cs, join, 0), "wait");
      }
    }
    cuda_check(cudaGetLastError(), "kernel launch");
    cudaEvent_t t_end[3] = {nullptr, nullptr, nullptr};
    if (trace) {
      for (int q = 0; q < 3; ++q) {
        cudaEventCreate(&t_end[q]);
        evs.push_back(t_end[q]);
      }
      cudaEventRecord(t_end[0], hs);
      cudaEventRecord(t_end[1], cs);
      cudaEventRecord(t_end[2], ds);
    }
    const double host_ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - host_t0).count();
    cuda_check(cudaStreamSynchronize(ds), "synchronize");
    cuda_check(cudaStreamSynchronize(cs), "synchronize");
    cuda_check(cudaStreamSynchronize(hs), "synchronize");
    if (pg) pg->finish();  // pageable B: the copy-backs into user memory
    if (trace) {
      auto ms_since = [](std::chrono::steady_clock::time_point a) {
        return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - a).count();
      };
      auto ms_between = [](std::chrono::steady_clock::time_point a, std::chrono::steady_clock::time_point b) {
        return std::chrono::duration<double, std::milli>(b - a).count();
      };
      fprintf(stderr, "e2e trace: entry -> start %.2f ms (meminfo %.2f, staging %.2f, descriptor run %.2f), "
              "host enqueue %.2f ms, entry -> synced %.2f ms\n",
              ms_since(entry_t0) - ms_since(host_t0), ms_between(entry_t0, tmark[0]), ms_between(tmark[0], tmark[1]),
              ms_between(tmark[1], tmark[2]), host_ms, ms_since(entry_t0));
      float t[3] = {0, 0, 0};
      for (int q = 0; q < 3; ++q) cudaEventElapsedTime(&t[q], start, t_end[q]);
      fprintf(stderr, "e2e trace: h2d done %.2f ms, compute done %.2f ms, d2h done %.2f ms, %zu units, %d chunks\n",
              t[0], t[1], t[2], units.size(), nch);
      for (const auto& mk : d2h_marks) {
        float a = 0, b = 0;
        cudaEventElapsedTime(&a, start, mk.second.first);
        cudaEventElapsedTime(&b, start, mk.second.second);
        fprintf(stderr, "  d2h chunk %d rows [%lld, %lld): %.2f -> %.2f ms\n", mk.first, (long long)cb[mk.first],
                (long long)cb[mk.first + 1], a, b);
      }
    }
  } catch (...) {
    cudaStreamSynchronize(hs);
    cudaStreamSynchronize(ds);
    cudaStreamSynchronize(cs);
    for (cudaEvent_t e : evs) cudaEventDestroy(e);
    if (d_flags) cudaFree(d_flags);
    if (h_flags) cudaFreeHost(h_flags);
    throw;
  }
  for (cudaEvent_t e : evs) cudaEventDestroy(e);
  if (h_flags) {
    flags.assign(h_flags, h_flags + n);
    cudaFree(d_flags);
    cudaFreeHost(h_flags);
  }
  if (!flags.empty())
    for (const auto& leaf : leaves)
      for (i64 r = leaf.first; r < leaf.first + leaf.second; ++r)
        if (flags[static_cast<size_t>(r)]) {
          Fail f{RECTRI_CU_SINGULAR, "singular triangular matrix: zero diagonal at row " + std::to_string(r)};
          f.index = r;
          throw f;
        }
  if (trace)
    fprintf(stderr, "e2e trace: entry -> return %.2f ms\n",
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - entry_t0).count());
  return true;
}

// rec_trmm / rec_trsm entry (recursion.cpp:165-192).
template <typename T>
void rec_entry(OpK op, const rectri_cu_spec* cspec, const rectri_cu_view& Av,
               const rectri_cu_view& Bv, i64 threshold, const rectri_cu_backend* cbe,
               rectri_cu_event_fn sink, void* user) {
  validate_view(Av, "A");
  validate_view(Bv, "B");
  // check_problem (recursion.cpp:50-67): spec, backend, threshold, square,
  // conformal, alias -- in that order.
  const Spec spec = validate_spec(cspec);
  const BackendInfo be = validate_backend(cbe);
  const Tf32x3Scope tf32x3_scope(std::is_same<T, float>::value && (be.flags & RECTRI_CU_TF32X3));
  if (threshold < 1) fail(RECTRI_CU_CONFIG, "threshold must be >= 1");
  if (Av.rows != Av.cols)
    fail(RECTRI_CU_SHAPE, "triangular A must be square, got %lldx%lld", (long long)Av.rows,
         (long long)Av.cols);
  const i64 want = spec.side == RECTRI_CU_LEFT ? Bv.rows : Bv.cols;
  if (want != Av.rows)
    fail(RECTRI_CU_SHAPE, "B is %lldx%lld, not conformal with %lldx%lld A on the %s",
         (long long)Bv.rows, (long long)Bv.cols, (long long)Av.rows, (long long)Av.cols,
         side_name(spec.side));
  if (overlaps(Av, Bv)) fail(RECTRI_CU_ALIAS, "A and B views overlap");
  if (Av.rows == 0 || Bv.rows == 0 || Bv.cols == 0) return;
  const Nvtx range(op == kTrsm ? "rectri rec_trsm n=%lld rhs=%lld" : "rectri rec_trmm n=%lld rhs=%lld",
                   static_cast<long long>(Av.rows),
                   static_cast<long long>(spec.side == RECTRI_CU_LEFT ? Bv.cols : Bv.rows));

  DeviceGuard guard(be.device);
  int dev = 0;
  cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
  const bool a_dev = is_device_memory(Av.origin);
  const bool b_dev = is_device_memory(Bv.origin);
  if (a_dev && b_dev) {
    run_device<T>(op, spec, dview_of<const T>(Av), dview_of<T>(Bv), threshold, be, sink, user,
                  dev, false);
    return;
  }
  // Host-resident operands: A's stored triangle is staged once; a host B is
  // processed in pipelined panels (run_host_panels).
  const i64 n = Av.rows;
  cudaStream_t s = be.stream;
  DView<const T> A = dview_of<const T>(Av);
  DView<T> B = dview_of<T>(Bv);
  DView<const T> dA = A;
  DeviceRes* res;
  {
    std::lock_guard<std::mutex> lock(g_mu);
    res = &device_res(dev);
  }
  // one host-operand call per device at a time owns the staging buffers
  std::lock_guard<std::mutex> stage_lock(res->stage_mu);
  if (!a_dev) {
    std::lock_guard<std::mutex> lock(g_mu);
    dA = DView<const T>{static_cast<T*>(staging(*res, 0, static_cast<size_t>(n * n) * sizeof(T))), n, n, n};
  }
  BackendInfo be2 = be;
  be2.flags &= ~RECTRI_CU_ASYNC;
  if (b_dev) {
    if (!a_dev) copy_triangle_h2d<T>(const_cast<T*>(dA.p), A, spec.uplo, s);
    run_device<T>(op, spec, dA, B, threshold, be2, sink, user, dev, true);
    return;
  }
  // Pageable (e.g. std::vector-backed) host operands go through pinned
  // bounce buffers with host-thread copies overlapping the GPU (host_stage.h);
  // RECTRI_CU_PAGEABLE_DIRECT=1 copies straight from pageable memory instead.
  std::unique_ptr<PageableStager> pg;
  const bool a_pg = !a_dev && is_pageable_host(Av.origin), b_pg = is_pageable_host(Bv.origin);
  if ((a_pg || b_pg) && !getenv("RECTRI_CU_PAGEABLE_DIRECT")) {
    const size_t a_bytes = static_cast<size_t>((n - 1) * A.ld + n) * sizeof(T);
    const size_t b_bytes = static_cast<size_t>((B.cols - 1) * B.ld + B.rows) * sizeof(T);
    pg = std::make_unique<PageableStager>(dev, a_pg ? A.p : nullptr, a_pg ? a_bytes : 0, b_pg ? B.p : nullptr,
                                          b_pg ? b_bytes : 0);
  }
  if (!getenv("RECTRI_CU_HOST_PANEL") &&
      run_host_streamed<T>(op, spec, A, a_dev, B, threshold, be2, sink, user, dev, pg.get()))
    return;
  pg.reset();
  cudaEvent_t a_ready = nullptr;
  if (!a_dev) {
    copy_triangle_h2d<T>(const_cast<T*>(dA.p), A, spec.uplo, res->h2d);
  }
  run_host_panels<T>(op, spec, dA, B, threshold, be2, sink, user, dev, a_ready);
}

// Temporary device copies of host views for the non-recursive entry points.
template <typename T>
struct Staged {
  using U = std::remove_const_t<T>;
  DView<T> view{};
  U* dev = nullptr;
  const T* host = nullptr;
  i64 host_ld = 0;
  Staged(const rectri_cu_view& v, cudaStream_t s) {
    DView<T> h = dview_of<T>(v);
    if (view_empty(v) || is_device_memory(v.origin)) {
      view = h;
      return;
    }
    host = h.p;
    host_ld = h.ld;
    cuda_check(cudaMalloc(reinterpret_cast<void**>(&dev), static_cast<size_t>(h.rows * h.cols) * sizeof(T) + 16), "stage");
    view = DView<T>{dev, h.rows, h.rows, h.cols};
    cuda_check(cudaMemcpy2DAsync(dev, sizeof(T) * h.rows, h.p, sizeof(T) * h.ld,
                                 sizeof(T) * h.rows, h.cols, cudaMemcpyHostToDevice, s),
               "H2D");
  }
  void copy_back(cudaStream_t s) {
    if (!dev) return;
    cuda_check(cudaMemcpy2DAsync(const_cast<T*>(host), sizeof(T) * host_ld, dev,
                                 sizeof(T) * view.ld, sizeof(T) * view.rows, view.cols,
                                 cudaMemcpyDeviceToHost, s),
               "D2H");
  }
  ~Staged() {
    if (dev) cudaFree(dev);
  }
};

// trsm_base / trmm_base entry (base_kernels.cpp:16-33, 137-177).
template <typename T>
void base_entry(OpK op, const rectri_cu_spec* cspec, const rectri_cu_view& Av,
                const rectri_cu_view& Bv, i64 tile_limit, const rectri_cu_backend* cbe) {
  validate_view(Av, "A");
  validate_view(Bv, "B");
  // check_tile (base_kernels.cpp:16-33), then validate(backend).
  const Spec spec = validate_spec(cspec);
  if (Av.rows != Av.cols)
    fail(RECTRI_CU_SHAPE, "triangular A must be square, got %lldx%lld", (long long)Av.rows,
         (long long)Av.cols);
  const i64 want = spec.side == RECTRI_CU_LEFT ? Bv.rows : Bv.cols;
  if (want != Av.rows)
    fail(RECTRI_CU_SHAPE, "B is %lldx%lld, not conformal with %lldx%lld A on the %s",
         (long long)Bv.rows, (long long)Bv.cols, (long long)Av.rows, (long long)Av.cols,
         side_name(spec.side));
  if (Av.rows > tile_limit)
    fail(RECTRI_CU_TILE_LIMIT, "tile of size %lld exceeds limit %lld", (long long)Av.rows,
         (long long)tile_limit);
  if (overlaps(Av, Bv)) fail(RECTRI_CU_ALIAS, "A and B views overlap");
  const BackendInfo be = validate_backend(cbe);
  const Tf32x3Scope tf32x3_scope(std::is_same<T, float>::value && (be.flags & RECTRI_CU_TF32X3));
  const i64 n = Av.rows;
  const i64 rhs = spec.side == RECTRI_CU_LEFT ? Bv.cols : Bv.rows;

  DeviceGuard guard(be.device);
  cudaStream_t s = be.stream;
  if (op == kTrsm && spec.diag == RECTRI_CU_NONUNIT && n > 0) {
    // Zero pivots are found before B is touched (base_kernels.cpp:166-169).
    Staged<const T> A(Av, s);
    uint8_t* d = nullptr;
    cuda_check(cudaMalloc(&d, static_cast<size_t>(n)), "flags");
    std::vector<uint8_t> h(static_cast<size_t>(n));
    K<T>::scan(A.view.p, A.view.ld, n, d, s);
    cudaError_t e = cudaMemcpyAsync(h.data(), d, static_cast<size_t>(n), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    cudaFree(d);
    cuda_check(e, "pivot scan");
    for (i64 r = 0; r < n; ++r)
      if (h[static_cast<size_t>(r)]) {
        Fail f{RECTRI_CU_SINGULAR, "singular triangular matrix: zero diagonal at row " + std::to_string(r)};
        f.index = r;
        throw f;
      }
  }
  if (n == 0 || rhs == 0) return;
  Staged<const T> A(Av, s);
  Staged<T> B(Bv, s);
  enqueue_base<T>(op, spec, A.view, B.view, s, nullptr, 0, /*direct=*/1);
  cuda_check(cudaGetLastError(), "leaf launch");
  B.copy_back(s);
  cuda_check(cudaStreamSynchronize(s), "synchronize");
}

// gemm entry (gemm.cpp:155-216).
template <typename T>
void gemm_entry(T alpha, int32_t ta_c, const rectri_cu_view& Av, int32_t tb_c,
                const rectri_cu_view& Bv, T beta, const rectri_cu_view& Cv,
                const rectri_cu_backend* cbe) {
  validate_view(Av, "A");
  validate_view(Bv, "B");
  validate_view(Cv, "C");
  const BackendInfo be = validate_backend(cbe);
  const Tf32x3Scope tf32x3_scope(std::is_same<T, float>::value && (be.flags & RECTRI_CU_TF32X3));
  if (ta_c < 0 || ta_c > 2 || tb_c < 0 || tb_c > 2) fail(RECTRI_CU_CONFIG, "trans out of range");
  const bool ta = ta_c != RECTRI_CU_NOTRANS, tb = tb_c != RECTRI_CU_NOTRANS;
  const i64 M = Cv.rows, N = Cv.cols;
  const i64 Kd = ta ? Av.rows : Av.cols;
  const i64 a_rows = ta ? Av.cols : Av.rows;
  const i64 b_rows = tb ? Bv.cols : Bv.rows;
  const i64 b_cols = tb ? Bv.rows : Bv.cols;
  if (a_rows != M || b_rows != Kd || b_cols != N)
    fail(RECTRI_CU_SHAPE, "gemm: op(A) is %lldx%lld, op(B) is %lldx%lld, C is %lldx%lld",
         (long long)a_rows, (long long)Kd, (long long)b_rows, (long long)b_cols, (long long)M,
         (long long)N);
  if (overlaps(Cv, Av) || overlaps(Cv, Bv)) fail(RECTRI_CU_ALIAS, "gemm: C overlaps an input view");
  if (M == 0 || N == 0) return;
  DeviceGuard guard(be.device);
  cudaStream_t s = be.stream;
  Staged<const T> A(Av, s);
  Staged<const T> B(Bv, s);
  Staged<T> C(Cv, s);
  enqueue_gemm<T>(alpha, ta, A.view, tb, B.view, beta, C.view, s);
  cuda_check(cudaGetLastError(), "gemm launch");
  C.copy_back(s);
  cuda_check(cudaStreamSynchronize(s), "synchronize");
}

template <typename T>
void scale_entry(T alpha, const rectri_cu_view& Bv, const rectri_cu_backend* cbe) {
  validate_view(Bv, "B");
  const BackendInfo be = validate_backend(cbe);
  if (alpha == T(1) || view_empty(Bv)) return;  // gemm.cpp:219
  DeviceGuard guard(be.device);
  cudaStream_t s = be.stream;
  Staged<T> B(Bv, s);
  K<T>::scale(B.view.p, B.view.ld, B.view.rows, B.view.cols, alpha, s);
  cuda_check(cudaGetLastError(), "scale launch");
  B.copy_back(s);
  cuda_check(cudaStreamSynchronize(s), "synchronize");
}

}  // namespace
}  // namespace rectri_cu

using namespace rectri_cu;

extern "C" {

int rectri_cu_rec_trmm_f64(const rectri_cu_spec* spec, rectri_cu_view A, rectri_cu_view B,
                           int64_t threshold, const rectri_cu_backend* backend,
                           rectri_cu_event_fn sink, void* sink_user) {
  return guarded([&] { rec_entry<double>(kTrmm, spec, A, B, threshold, backend, sink, sink_user); },
                 nullptr);
}
int rectri_cu_rec_trmm_f32(const rectri_cu_spec* spec, rectri_cu_view A, rectri_cu_view B,
                           int64_t threshold, const rectri_cu_backend* backend,
                           rectri_cu_event_fn sink, void* sink_user) {
  return guarded([&] { rec_entry<float>(kTrmm, spec, A, B, threshold, backend, sink, sink_user); },
                 nullptr);
}
int rectri_cu_rec_trsm_f64(const rectri_cu_spec* spec, rectri_cu_view A, rectri_cu_view B,
                           int64_t threshold, const rectri_cu_backend* backend,
                           rectri_cu_event_fn sink, void* sink_user, int64_t* singular_row) {
  return guarded([&] { rec_entry<double>(kTrsm, spec, A, B, threshold, backend, sink, sink_user); },
                 singular_row);
}
int rectri_cu_rec_trsm_f32(const rectri_cu_spec* spec, rectri_cu_view A, rectri_cu_view B,
                           int64_t threshold, const rectri_cu_backend* backend,
                           rectri_cu_event_fn sink, void* sink_user, int64_t* singular_row) {
  return guarded([&] { rec_entry<float>(kTrsm, spec, A, B, threshold, backend, sink, sink_user); },
                 singular_row);
}

int rectri_cu_trmm_base_f64(const rectri_cu_spec* spec, rectri_cu_view A, rectri_cu_view B,
                            int64_t tile_limit, const rectri_cu_backend* backend) {
  return guarded([&] { base_entry<double>(kTrmm, spec, A, B, tile_limit, backend); }, nullptr);
}
int rectri_cu_trmm_base_f32(const rectri_cu_spec* spec, rectri_cu_view A, rectri_cu_view B,
                            int64_t tile_limit, const rectri_cu_backend* backend) {
  return guarded([&] { base_entry<float>(kTrmm, spec, A, B, tile_limit, backend); }, nullptr);
}
int rectri_cu_trsm_base_f64(const rectri_cu_spec* spec, rectri_cu_view A, rectri_cu_view B,
                            int64_t tile_limit, const rectri_cu_backend* backend,
                            int64_t* singular_row) {
  return guarded([&] { base_entry<double>(kTrsm, spec, A, B, tile_limit, backend); }, singular_row);
}
int rectri_cu_trsm_base_f32(const rectri_cu_spec* spec, rectri_cu_view A, rectri_cu_view B,
                            int64_t tile_limit, const rectri_cu_backend* backend,
                            int64_t* singular_row) {
  return guarded([&] { base_entry<float>(kTrsm, spec, A, B, tile_limit, backend); }, singular_row);
}

int rectri_cu_gemm_f64(double alpha, int32_t trans_a, rectri_cu_view A, int32_t trans_b,
                       rectri_cu_view B, double beta, rectri_cu_view C,
                       const rectri_cu_backend* backend) {
  return guarded([&] { gemm_entry<double>(alpha, trans_a, A, trans_b, B, beta, C, backend); },
                 nullptr);
}
int rectri_cu_gemm_f32(float alpha, int32_t trans_a, rectri_cu_view A, int32_t trans_b,
                       rectri_cu_view B, float beta, rectri_cu_view C,
                       const rectri_cu_backend* backend) {
  return guarded([&] { gemm_entry<float>(alpha, trans_a, A, trans_b, B, beta, C, backend); },
                 nullptr);
}

int rectri_cu_scale_f64(double alpha, rectri_cu_view B, const rectri_cu_backend* backend) {
  return guarded([&] { scale_entry<double>(alpha, B, backend); }, nullptr);
}
int rectri_cu_scale_f32(float alpha, rectri_cu_view B, const rectri_cu_backend* backend) {
  return guarded([&] { scale_entry<float>(alpha, B, backend); }, nullptr);
}

int rectri_cu_schema_for(int32_t op, const rectri_cu_spec* spec, double out[8]) {
  return guarded(
      [&] {
        const Spec s = validate_spec(spec);
        const Schema sc = schema_for(op == 1 ? kTrsm : kTrmm, s.side, s.uplo, s.trans);
        out[0] = sc.first_a22;
        out[1] = sc.off_trans;
        out[2] = sc.off_on_left;
        out[3] = sc.read_b2;
        out[4] = sc.write_b2;
        out[5] = sc.sign;
        out[6] = sc.carries_alpha;
        out[7] = !sc.first_a22;
      },
      nullptr);
}

int rectri_cu_sync(void* stream, int64_t* singular_row) {
  return guarded(
      [&] {
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        cuda_check(cudaStreamSynchronize(s), "synchronize");
        std::vector<std::shared_ptr<GraphEntry>> pend;
        i64 deferred = -1;
        {
          std::lock_guard<std::mutex> lock(g_mu);
          auto range = g_pending.equal_range(s);
          for (auto it = range.first; it != range.second; ++it) pend.push_back(it->second);
          g_pending.erase(s);
          auto d = g_deferred.find(s);
          if (d != g_deferred.end()) {
            deferred = d->second;
            g_deferred.erase(d);
          }
        }
        if (deferred >= 0) {
          Fail f{RECTRI_CU_SINGULAR, "singular triangular matrix: zero diagonal at row " + std::to_string(deferred)};
          f.index = deferred;
          throw f;
        }
        for (const auto& g : pend) {
          const i64 r = first_singular(*g);
          if (r >= 0) {
            Fail f{RECTRI_CU_SINGULAR,
                   "singular triangular matrix: zero diagonal at row " + std::to_string(r)};
            f.index = r;
            throw f;
          }
        }
      },
      singular_row);
}

const char* rectri_cu_last_error(void) { return g_last_error.c_str(); }

int64_t rectri_cu_launch_count(void) { return launch_counter(); }

void rectri_cu_clear_graph_cache(void) {
  // Pending ASYNC checks keep their entries alive (shared_ptr) and are still
  // reported by the next rectri_cu_sync on their stream.
  std::lock_guard<std::mutex> lock(g_mu);
  g_cache.clear();
}

void rectri_cu_release_staging(void) {
  std::vector<std::pair<int, DeviceRes*>> devs;  // map nodes are stable
  {
    std::lock_guard<std::mutex> lock(g_mu);
    for (auto& kv : g_dev) devs.push_back({kv.first, &kv.second});
  }
  int prev = 0;
  cudaGetDevice(&prev);
  for (auto& d : devs) {
    DeviceRes& r = *d.second;
    std::lock_guard<std::mutex> stage_lock(r.stage_mu);  // waits for a host-operand call in flight
    std::lock_guard<std::mutex> lock(g_mu);
    cudaSetDevice(d.first);
    for (int k = 0; k < DeviceRes::kSlots; ++k) {
      if (r.stage[k]) cudaFree(r.stage[k]);
      r.stage[k] = nullptr;
      r.stage_bytes[k] = 0;
    }
  }
  cudaSetDevice(prev);
  release_pageable_bounce();
}

int64_t rectri_cu_device_bytes_held(void) {
  std::lock_guard<std::mutex> lock(g_mu);
  size_t b = g_cache.bytes;
  for (auto& kv : g_dev)
    for (int k = 0; k < DeviceRes::kSlots; ++k) b += kv.second.stage_bytes[k];
  return static_cast<int64_t>(b);
}

int rectri_cu_abi_version(void) { return RECTRI_CU_ABI_VERSION; }

int rectri_cu_fill_uniform(int32_t dtype, rectri_cu_view B, int64_t col0, int64_t global_rows,
                           uint64_t seed, const rectri_cu_backend* backend) {
  return guarded(
      [&] {
        validate_view(B, "B");
        const BackendInfo be = validate_backend(backend);
        if (view_empty(B)) return;
        if (!is_device_memory(B.origin)) fail(RECTRI_CU_CONFIG, "fill_uniform needs device memory");
        DeviceGuard guard(be.device);
        if (dtype == 1) {
          DView<double> v = dview_of<double>(B);
          launch_fill_uniform_f64(v.p, v.ld, v.rows, v.cols, col0, global_rows, seed, be.stream);
        } else {
          DView<float> v = dview_of<float>(B);
          launch_fill_uniform_f32(v.p, v.ld, v.rows, v.cols, col0, global_rows, seed, be.stream);
        }
        cuda_check(cudaGetLastError(), "fill launch");
        if (!(be.flags & RECTRI_CU_ASYNC)) cuda_check(cudaStreamSynchronize(be.stream), "synchronize");
      },
      nullptr);
}

int rectri_cu_make_dominant(int32_t dtype, rectri_cu_view A, int32_t uplo,
                            const rectri_cu_backend* backend) {
  return guarded(
      [&] {
        validate_view(A, "A");
        const BackendInfo be = validate_backend(backend);
        if (A.rows != A.cols) fail(RECTRI_CU_SHAPE, "A must be square");
        if (view_empty(A)) return;
        if (!is_device_memory(A.origin)) fail(RECTRI_CU_CONFIG, "make_dominant needs device memory");
        DeviceGuard guard(be.device);
        if (dtype == 1) {
          DView<double> v = dview_of<double>(A);
          launch_make_dominant_f64(v.p, v.ld, v.rows, uplo, be.stream);
        } else {
          DView<float> v = dview_of<float>(A);
          launch_make_dominant_f32(v.p, v.ld, v.rows, uplo, be.stream);
        }
        cuda_check(cudaGetLastError(), "dominant launch");
        if (!(be.flags & RECTRI_CU_ASYNC)) cuda_check(cudaStreamSynchronize(be.stream), "synchronize");
      },
      nullptr);
}

double rectri_cu_probe_peak(int32_t kind) { return probe_peak_tflops(kind); }

int64_t rectri_cu_debug_ring_check(int32_t reset) { return leaf_ring_check_read(reset != 0); }

// Host storage for the C++ drop-in's MatrixBuffer: page-locked (portable)
// when a CUDA device is present and RECTRI_CU_PINNED_BUFFERS is not 0, so the
// host-operand path moves it at full PCIe rate with no bounce copy; plain
// malloc otherwise (or when pinning fails).  Allocations are remembered so
// rectri_cu_host_free releases each the way it was made.
namespace {
std::mutex g_host_mu;
std::map<void*, bool> g_host_allocs;  // pointer -> page-locked
}  // namespace

void* rectri_cu_host_alloc(size_t bytes, int32_t* pinned) {
  if (pinned) *pinned = 0;
  if (bytes == 0) bytes = 1;
  void* p = nullptr;
  bool pin = false;
  const char* e = getenv("RECTRI_CU_PINNED_BUFFERS");
  int ndev = 0;
  if (!(e && atoi(e) == 0) && cudaGetDeviceCount(&ndev) == cudaSuccess && ndev > 0) {
    pin = cudaHostAlloc(&p, bytes, cudaHostAllocPortable) == cudaSuccess;
    if (!pin) {
      p = nullptr;
      cudaGetLastError();  // clear the failed allocation's error
    }
  }
  if (!p) p = std::malloc(bytes);
  if (!p) return nullptr;
  {
    std::lock_guard<std::mutex> lock(g_host_mu);
    g_host_allocs[p] = pin;
  }
  if (pinned) *pinned = pin ? 1 : 0;
  return p;
}

void rectri_cu_host_free(void* p) {
  if (!p) return;
  bool pin = false;
  {
    std::lock_guard<std::mutex> lock(g_host_mu);
    auto it = g_host_allocs.find(p);
    if (it == g_host_allocs.end()) return;
    pin = it->second;
    g_host_allocs.erase(it);
  }
  if (pin) cudaFreeHost(p);
  else std::free(p);
}

void rectri_cu_profile_enable(int32_t on) {
  std::lock_guard<std::mutex> lock(g_mu);
  g_prof.on = on != 0;
}

int rectri_cu_profile_read(double ms[4], int64_t launches[4], double flops[4]) {
  return guarded(
      [&] {
        for (int k = 0; k < 4; ++k) {
          ms[k] = 0.0;
          launches[k] = 0;
          flops[k] = 0.0;
        }
        std::vector<ProfRec> recs;
        {
          std::lock_guard<std::mutex> lock(g_mu);
          recs.swap(g_prof.recs);
        }
        for (ProfRec& r : recs) {
          cuda_check(cudaEventSynchronize(r.b), "profile sync");
          float t = 0.f;
          cuda_check(cudaEventElapsedTime(&t, r.a, r.b), "profile elapsed");
          if (r.kind >= 0 && r.kind < 4) {
            ms[r.kind] += t;
            launches[r.kind] += 1;
            flops[r.kind] += r.flops;
          }
          cudaEventDestroy(r.a);
          cudaEventDestroy(r.b);
        }
      },
      nullptr);
}

}  // extern "C"
