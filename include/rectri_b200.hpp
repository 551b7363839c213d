// rectri_b200.hpp -- C++ drop-in for the reference's rectri TRMM/TRSM API,
// computing on the B200 through the C-ABI of rectri_cu.h (librectri_cu.so).
//
// Source compatibility target: code written against the reference headers
// (/root/reference/proj/include/rectri/{common,error,matrix,flags,backend,
// recursion,base_kernels,gemm}.hpp) compiles unchanged against this header
// -- the forwarding headers in include/rectri/ include it under the same
// paths -- and links against librectri_cu.so instead of the reference's
// static library.  Names, argument meaning, validation order and exception
// types follow the reference; compute always runs on the GPU:
//   * views over host memory (MatrixBuffer's std::vector) are staged to the
//     device and back inside each call;
//   * views over device memory (the public MatrixView constructor wrapping a
//     cudaMalloc'ed pointer) are computed in place;
//   * Backend gains device/stream/flags fields; Backend::seq()/par() keep
//     their signatures (parallel_width is validated, then advisory).
#pragma once

#include <cmath>
#include <cstdint>
#include <functional>
#include <new>
#include <stdexcept>
#include <string>
#include <string_view>
#include <thread>
#include <type_traits>
#include <vector>

#include "rectri_cu.h"

namespace rectri {

using index_t = std::int64_t;

enum class ElemKind { F32, F64 };
constexpr bool is_real(ElemKind) { return true; }
template <typename T> struct elem_kind_of;
template <> struct elem_kind_of<float> { static constexpr ElemKind value = ElemKind::F32; };
template <> struct elem_kind_of<double> { static constexpr ElemKind value = ElemKind::F64; };
constexpr const char* elem_kind_name(ElemKind k) { return k == ElemKind::F32 ? "f32" : "f64"; }

// ---- failures: one class per status code of the C-ABI ---------------------
struct Error : std::runtime_error { using std::runtime_error::runtime_error; };
struct ShapeError : Error { using Error::Error; };
struct BoundsError : Error { using Error::Error; };
struct AliasError : Error { using Error::Error; };
struct SplitError : Error { using Error::Error; };
struct TileLimitError : Error { using Error::Error; };
struct ConfigError : Error { using Error::Error; };
struct ValidationError : Error { using Error::Error; };
struct JoinError : Error { using Error::Error; };
struct IoError : Error { using Error::Error; };
struct CudaError : Error { using Error::Error; };
class SingularityError : public Error {
 public:
  explicit SingularityError(index_t row)
      : Error("singular triangular matrix: zero diagonal at row " + std::to_string(row)), row_(row) {}
  index_t index() const noexcept { return row_; }

 private:
  index_t row_;
};

namespace detail {
[[noreturn]] inline void throw_status(int st, index_t row) {
  const std::string msg = rectri_cu_last_error();
  switch (st) {
    case RECTRI_CU_CONFIG: throw ConfigError(msg);
    case RECTRI_CU_SHAPE: throw ShapeError(msg);
    case RECTRI_CU_ALIAS: throw AliasError(msg);
    case RECTRI_CU_SINGULAR: throw SingularityError(row);
    case RECTRI_CU_TILE_LIMIT: throw TileLimitError(msg);
    case RECTRI_CU_BOUNDS: throw BoundsError(msg);
    case RECTRI_CU_SPLIT: throw SplitError(msg);
    default: throw CudaError(msg);
  }
}
inline void check(int st, index_t row = -1) {
  if (st != RECTRI_CU_OK) throw_status(st, row);
}
}  // namespace detail

// ---- flags ------------------------------------------------------------------
enum class Side { Left, Right };
enum class Uplo { Lower, Upper };
enum class Trans { NoTrans, Trans, ConjTrans };
enum class Diag { NonUnit, Unit };

struct TriangularSpec {
  Side side = Side::Left;
  Uplo uplo = Uplo::Lower;
  Trans trans = Trans::NoTrans;
  Diag diag = Diag::NonUnit;
  double alpha = 1.0;
};

constexpr Trans effective_op(Trans t, ElemKind k) {
  return (t == Trans::ConjTrans && is_real(k)) ? Trans::Trans : t;
}
constexpr Trans effective_op(const TriangularSpec& s, ElemKind k) { return effective_op(s.trans, k); }
inline void validate(const TriangularSpec& s) {
  if (!std::isfinite(s.alpha)) throw ConfigError("alpha must be finite");
}

constexpr std::string_view to_string(Side s) { return s == Side::Left ? "left" : "right"; }
constexpr std::string_view to_string(Uplo u) { return u == Uplo::Lower ? "lower" : "upper"; }
constexpr std::string_view to_string(Trans t) {
  return t == Trans::NoTrans ? "n" : (t == Trans::Trans ? "t" : "c");
}
constexpr std::string_view to_string(Diag d) { return d == Diag::NonUnit ? "nonunit" : "unit"; }

inline Side parse_side(std::string_view s) {
  if (s == "left") return Side::Left;
  if (s == "right") return Side::Right;
  throw ConfigError("unknown side '" + std::string(s) + "' (left|right)");
}
inline Uplo parse_uplo(std::string_view s) {
  if (s == "lower") return Uplo::Lower;
  if (s == "upper") return Uplo::Upper;
  throw ConfigError("unknown uplo '" + std::string(s) + "' (lower|upper)");
}
inline Trans parse_trans(std::string_view s) {
  if (s == "n") return Trans::NoTrans;
  if (s == "t") return Trans::Trans;
  if (s == "c") return Trans::ConjTrans;
  throw ConfigError("unknown trans '" + std::string(s) + "' (n|t|c)");
}
inline Diag parse_diag(std::string_view s) {
  if (s == "unit") return Diag::Unit;
  if (s == "nonunit") return Diag::NonUnit;
  throw ConfigError("unknown diag '" + std::string(s) + "' (unit|nonunit)");
}
inline std::string variant_string(const TriangularSpec& s) {
  std::string v;
  for (std::string_view part : {to_string(s.side), to_string(s.uplo), to_string(s.trans), to_string(s.diag)}) {
    if (!v.empty()) v += '-';
    v += part;
  }
  return v;
}

// ---- storage and windows ----------------------------------------------------
template <typename T> class MatrixView;

// Storage allocator of MatrixBuffer: rectri_cu_host_alloc -- page-locked
// memory when a CUDA device is present (RECTRI_CU_PINNED_BUFFERS=0: plain
// malloc), so rec_trsm / rec_trmm on MatrixBuffers copy them at full PCIe
// rate with no bounce through a staging buffer.  The buffer's interface is
// the reference's (matrix.hpp:18-70); only where its bytes live changes.
template <typename T>
struct HostAllocator {
  using value_type = T;
  HostAllocator() noexcept = default;
  template <typename U>
  HostAllocator(const HostAllocator<U>&) noexcept {}
  T* allocate(std::size_t n) {
    void* p = rectri_cu_host_alloc(n * sizeof(T), nullptr);
    if (!p) throw std::bad_alloc();
    return static_cast<T*>(p);
  }
  void deallocate(T* p, std::size_t) noexcept { rectri_cu_host_free(p); }
  template <typename U>
  bool operator==(const HostAllocator<U>&) const noexcept { return true; }
  template <typename U>
  bool operator!=(const HostAllocator<U>&) const noexcept { return false; }
};

template <typename T>
class MatrixBuffer {
  static_assert(std::is_floating_point_v<T>);

 public:
  static constexpr ElemKind kind = elem_kind_of<T>::value;
  MatrixBuffer() = default;
  MatrixBuffer(index_t rows, index_t cols, T fill = T{}) : rows_(rows), cols_(cols) {
    if (rows < 0 || cols < 0) throw ShapeError("negative matrix dimension");
    store_.assign(static_cast<std::size_t>(rows) * static_cast<std::size_t>(cols), fill);
  }
  index_t rows() const noexcept { return rows_; }
  index_t cols() const noexcept { return cols_; }
  T* data() noexcept { return store_.data(); }
  const T* data() const noexcept { return store_.data(); }
  T& operator()(index_t r, index_t c) noexcept { return store_[static_cast<std::size_t>(c * rows_ + r)]; }
  const T& operator()(index_t r, index_t c) const noexcept {
    return store_[static_cast<std::size_t>(c * rows_ + r)];
  }
  T& at(index_t r, index_t c) {
    if (r < 0 || c < 0 || r >= rows_ || c >= cols_) throw BoundsError("matrix index out of range");
    return (*this)(r, c);
  }
  const T& at(index_t r, index_t c) const {
    if (r < 0 || c < 0 || r >= rows_ || c >= cols_) throw BoundsError("matrix index out of range");
    return (*this)(r, c);
  }
  MatrixView<T> view() noexcept { return MatrixView<T>(data(), rows_, cols_, 0, 0, rows_, cols_); }
  MatrixView<const T> view() const noexcept {
    return MatrixView<const T>(data(), rows_, cols_, 0, 0, rows_, cols_);
  }
  MatrixView<const T> cview() const noexcept { return view(); }

 private:
  index_t rows_ = 0, cols_ = 0;
  std::vector<T, HostAllocator<T>> store_;
};

// Window of an origin buffer (host or device), column-major, ld = origin rows.
template <typename T>
class MatrixView {
 public:
  using value_type = std::remove_const_t<T>;
  MatrixView() = default;
  MatrixView(T* origin, index_t origin_rows, index_t origin_cols, index_t row_offset, index_t col_offset,
             index_t rows, index_t cols)
      : o_(origin), orows_(origin_rows), ocols_(origin_cols), r0_(row_offset), c0_(col_offset), rows_(rows),
        cols_(cols) {}
  operator MatrixView<const T>() const noexcept {
    return MatrixView<const T>(o_, orows_, ocols_, r0_, c0_, rows_, cols_);
  }
  index_t rows() const noexcept { return rows_; }
  index_t cols() const noexcept { return cols_; }
  index_t row_offset() const noexcept { return r0_; }
  index_t col_offset() const noexcept { return c0_; }
  index_t leading_dim() const noexcept { return orows_; }
  bool empty() const noexcept { return rows_ == 0 || cols_ == 0; }
  T* data() const noexcept { return o_ + c0_ * orows_ + r0_; }
  T& operator()(index_t r, index_t c) const noexcept { return o_[(c0_ + c) * orows_ + r0_ + r]; }
  T& at(index_t r, index_t c) const {
    if (r < 0 || c < 0 || r >= rows_ || c >= cols_) throw BoundsError("view index out of range");
    return (*this)(r, c);
  }
  MatrixView subview(index_t r0, index_t c0, index_t nr, index_t nc) const {
    if (r0 < 0 || c0 < 0 || nr < 0 || nc < 0 || r0 + nr > rows_ || c0 + nc > cols_)
      throw BoundsError("subview escapes its parent view");
    return MatrixView(o_, orows_, ocols_, r0_ + r0, c0_ + c0, nr, nc);
  }
  const void* origin_id() const noexcept { return o_; }
  // The C-ABI descriptor of this window.
  rectri_cu_view c_view() const noexcept {
    return rectri_cu_view{const_cast<value_type*>(o_), orows_, ocols_, r0_, c0_, rows_, cols_};
  }

 private:
  T* o_ = nullptr;
  index_t orows_ = 0, ocols_ = 0, r0_ = 0, c0_ = 0, rows_ = 0, cols_ = 0;
};

template <typename A, typename B>
bool overlaps(const MatrixView<A>& a, const MatrixView<B>& b) noexcept {
  if (a.origin_id() != b.origin_id() || a.empty() || b.empty()) return false;
  return a.row_offset() < b.row_offset() + b.rows() && b.row_offset() < a.row_offset() + a.rows() &&
         a.col_offset() < b.col_offset() + b.cols() && b.col_offset() < a.col_offset() + a.cols();
}

inline index_t split_half(index_t n) {
  if (n < 2) throw SplitError("cannot split dimension " + std::to_string(n));
  return n / 2;
}

// ---- execution backend -------------------------------------------------------
struct GemmBlocking {
  index_t mc = 64, kc = 64, nc = 64;
};

struct Backend {
  std::string name = "seq";
  int parallel_width = 1;
  GemmBlocking blocking{};
  int device = -1;          // CUDA ordinal, -1 = current
  void* stream = nullptr;   // cudaStream_t, nullptr = legacy default stream
  std::uint32_t flags = 0;  // RECTRI_CU_ASYNC | RECTRI_CU_NO_GRAPH | RECTRI_CU_TF32X3

  static Backend seq() { return Backend{}; }
  static Backend par(int width = 0) {
    Backend b;
    b.name = "par";
    b.parallel_width = width > 0 ? width : static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
    return b;
  }
  static Backend cuda(int device = -1, void* stream = nullptr, std::uint32_t flags = 0) {
    Backend b;
    b.name = "cuda";
    b.device = device;
    b.stream = stream;
    b.flags = flags;
    return b;
  }
  rectri_cu_backend c_backend() const noexcept {
    return rectri_cu_backend{parallel_width, device, stream, flags, blocking.mc, blocking.kc, blocking.nc};
  }
};

inline void validate(const Backend& b) {
  if (b.parallel_width < 1) throw ConfigError("backend parallel_width must be >= 1");
  if (b.blocking.mc < 1 || b.blocking.kc < 1 || b.blocking.nc < 1)
    throw ConfigError("backend block sizes must be >= 1");
}

// ---- recursion ----------------------------------------------------------------
inline constexpr index_t kDefaultTileLimit = 256;
struct Threshold {
  index_t value = kDefaultTileLimit;
};
enum class DiagBlock { A11, A22 };
enum class BHalf { B1, B2 };
struct GemmUpdate {
  Trans off_trans = Trans::NoTrans;
  bool off_on_left = true;
  BHalf read_half = BHalf::B1;
  BHalf write_half = BHalf::B2;
  double sign = 1.0;
  bool carries_alpha = false;
};
struct RecursionSchema {
  DiagBlock first_block;
  GemmUpdate update;
  DiagBlock second_block;
};
enum class OpKind { Trmm, Trsm };
constexpr std::string_view to_string(OpKind op) { return op == OpKind::Trmm ? "trmm" : "trsm"; }
inline OpKind parse_op_kind(std::string_view s) {
  if (s == "trmm") return OpKind::Trmm;
  if (s == "trsm") return OpKind::Trsm;
  throw ConfigError("unknown op '" + std::string(s) + "' (trmm|trsm)");
}
enum class RecEvent { Gemm, BaseTrmm, BaseTrsm };
using EventSink = std::function<void(RecEvent, index_t n, index_t m)>;

namespace detail {
inline rectri_cu_spec c_spec(const TriangularSpec& s) {
  return rectri_cu_spec{static_cast<int32_t>(s.side), static_cast<int32_t>(s.uplo),
                        static_cast<int32_t>(s.trans), static_cast<int32_t>(s.diag), s.alpha};
}
inline void sink_tramp(void* user, int32_t ev, int64_t n, int64_t m) {
  const EventSink& sink = *static_cast<const EventSink*>(user);
  sink(static_cast<RecEvent>(ev), n, m);
}
template <typename T> struct abi;
template <> struct abi<double> {
  static constexpr auto trmm = rectri_cu_rec_trmm_f64;
  static constexpr auto trsm = rectri_cu_rec_trsm_f64;
  static constexpr auto trmm_base = rectri_cu_trmm_base_f64;
  static constexpr auto trsm_base = rectri_cu_trsm_base_f64;
  static constexpr auto gemm = rectri_cu_gemm_f64;
  static constexpr auto scale = rectri_cu_scale_f64;
};
template <> struct abi<float> {
  static constexpr auto trmm = rectri_cu_rec_trmm_f32;
  static constexpr auto trsm = rectri_cu_rec_trsm_f32;
  static constexpr auto trmm_base = rectri_cu_trmm_base_f32;
  static constexpr auto trsm_base = rectri_cu_trsm_base_f32;
  static constexpr auto gemm = rectri_cu_gemm_f32;
  static constexpr auto scale = rectri_cu_scale_f32;
};
}  // namespace detail

inline RecursionSchema schema_for(OpKind op, const TriangularSpec& spec) {
  const rectri_cu_spec cs = detail::c_spec(spec);
  double out[8];
  detail::check(rectri_cu_schema_for(op == OpKind::Trsm ? 1 : 0, &cs, out));
  RecursionSchema r{};
  r.first_block = out[0] != 0 ? DiagBlock::A22 : DiagBlock::A11;
  r.update.off_trans = out[1] != 0 ? Trans::Trans : Trans::NoTrans;
  r.update.off_on_left = out[2] != 0;
  r.update.read_half = out[3] != 0 ? BHalf::B2 : BHalf::B1;
  r.update.write_half = out[4] != 0 ? BHalf::B2 : BHalf::B1;
  r.update.sign = out[5];
  r.update.carries_alpha = out[6] != 0;
  r.second_block = out[7] != 0 ? DiagBlock::A22 : DiagBlock::A11;
  return r;
}

// B <- alpha op(A) B (Left) / alpha B op(A) (Right), in place.
template <typename T>
void rec_trmm(const TriangularSpec& spec, MatrixView<const T> A, MatrixView<T> B, Threshold threshold = {},
              const Backend& backend = Backend::seq(), const EventSink& sink = {}) {
  const rectri_cu_spec cs = detail::c_spec(spec);
  const rectri_cu_backend cb = backend.c_backend();
  detail::check(detail::abi<T>::trmm(&cs, A.c_view(), B.c_view(), threshold.value, &cb,
                                     sink ? detail::sink_tramp : nullptr, const_cast<EventSink*>(&sink)));
}

// Solves op(A) X = alpha B (Left) / X op(A) = alpha B (Right); X in B.
template <typename T>
void rec_trsm(const TriangularSpec& spec, MatrixView<const T> A, MatrixView<T> B, Threshold threshold = {},
              const Backend& backend = Backend::seq(), const EventSink& sink = {}) {
  const rectri_cu_spec cs = detail::c_spec(spec);
  const rectri_cu_backend cb = backend.c_backend();
  int64_t row = -1;
  const int st = detail::abi<T>::trsm(&cs, A.c_view(), B.c_view(), threshold.value, &cb,
                                      sink ? detail::sink_tramp : nullptr, const_cast<EventSink*>(&sink), &row);
  detail::check(st, row);
}

template <typename T>
void trmm_base(const TriangularSpec& spec, MatrixView<const T> A, MatrixView<T> B,
               index_t tile_limit = kDefaultTileLimit, const Backend& backend = Backend::seq()) {
  const rectri_cu_spec cs = detail::c_spec(spec);
  const rectri_cu_backend cb = backend.c_backend();
  detail::check(detail::abi<T>::trmm_base(&cs, A.c_view(), B.c_view(), tile_limit, &cb));
}

template <typename T>
void trsm_base(const TriangularSpec& spec, MatrixView<const T> A, MatrixView<T> B,
               index_t tile_limit = kDefaultTileLimit, const Backend& backend = Backend::seq()) {
  const rectri_cu_spec cs = detail::c_spec(spec);
  const rectri_cu_backend cb = backend.c_backend();
  int64_t row = -1;
  detail::check(detail::abi<T>::trsm_base(&cs, A.c_view(), B.c_view(), tile_limit, &cb, &row), row);
}

// C <- alpha op(A) op(B) + beta C.
template <typename T>
void gemm(T alpha, Trans trans_a, MatrixView<const T> A, Trans trans_b, MatrixView<const T> B, T beta,
          MatrixView<T> C, const Backend& backend = Backend::seq()) {
  const rectri_cu_backend cb = backend.c_backend();
  detail::check(detail::abi<T>::gemm(alpha, static_cast<int32_t>(trans_a), A.c_view(),
                                     static_cast<int32_t>(trans_b), B.c_view(), beta, C.c_view(), &cb));
}
template <typename T>
void gemm(T alpha, Trans trans_a, MatrixView<const T> A, MatrixView<const T> B, T beta, MatrixView<T> C,
          const Backend& backend = Backend::seq()) {
  gemm(alpha, trans_a, A, Trans::NoTrans, B, beta, C, backend);
}

// B <- alpha B.
template <typename T>
void scale(T alpha, MatrixView<T> B) {
  const rectri_cu_backend cb = Backend::seq().c_backend();
  detail::check(detail::abi<T>::scale(alpha, B.c_view(), &cb));
}

}  // namespace rectri
