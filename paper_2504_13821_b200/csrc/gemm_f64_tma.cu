// gemm_f64_tma.cu -- host side of the TMA-fed fp64 DMMA GEMM: tensor-map
// encoding (driver entry point, no -lcuda link) and configuration choice.
#include <cstdlib>
#include <mutex>

#include "gemm_f64_tma.cuh"
#include "gemm_f64_tma_cfgs.h"

namespace rectri_cu {
namespace {

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                              CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                              CUtensorMapFloatOOBfill);

EncodeFn encoder() {
  static EncodeFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<EncodeFn>(nullptr);
    return reinterpret_cast<EncodeFn>(f);
  }();
  return fn;
}

int env_int(const char* k, int d) {
  const char* e = getenv(k);
  return e ? atoi(e) : d;
}

}  // namespace

// A 2D column-major operand as a tensor map.  outer_contig: element (o, k)
// at X[o + k*ld] (dims {O, K}, box {BO + 4, 16}, no swizzle); else element (o, k)
// at X[k + o*ld] (dims {K, O}, box {16, BO}, 128-byte swizzle).
bool encode_operand(CUtensorMap* map, const double* X, i64 ld, i64 O, i64 K, int BO, bool outer_contig) {
  EncodeFn enc = encoder();
  if (!enc) return false;
  cuuint64_t dims[2], strides[1] = {static_cast<cuuint64_t>(ld) * 8};
  cuuint32_t box[2], estr[2] = {1, 1};
  if (outer_contig) {
    dims[0] = static_cast<cuuint64_t>(O);
    dims[1] = static_cast<cuuint64_t>(K);
    box[0] = static_cast<cuuint32_t>(BO + 4);  // padded k-rows (gemm_f64_tma.cuh)
    box[1] = dgemm_tma::kBK;
  } else {
    dims[0] = static_cast<cuuint64_t>(K);
    dims[1] = static_cast<cuuint64_t>(O);
    box[0] = dgemm_tma::kBK;
    box[1] = static_cast<cuuint32_t>(BO);
  }
  const CUresult r =
      enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(X), dims, strides, box, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, outer_contig ? CU_TENSOR_MAP_SWIZZLE_NONE : CU_TENSOR_MAP_SWIZZLE_128B,
          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

namespace {
const DgemmTmaRun kTmaRuns[] = {
#define RECTRI_ENTRY(ID, BM, BN, WM, WN, ST, PR) dgemm_tma_cfg##ID,
    RECTRI_DGEMM_TMA_CONFIGS(RECTRI_ENTRY)
#undef RECTRI_ENTRY
};
constexpr int kNumTma = sizeof(kTmaRuns) / sizeof(kTmaRuns[0]);
}  // namespace

bool tma_eligible(const GemmParams<double>& p) {
  const auto al16 = [](const void* x) { return (reinterpret_cast<uintptr_t>(x) & 15u) == 0; };
  const i64 lim = (i64{1} << 31) - 256;
  return encoder() != nullptr && al16(p.A) && al16(p.B) && p.lda % 2 == 0 && p.ldb % 2 == 0 &&
         p.M < lim && p.N < lim && p.K < lim;
}

// RECTRI_CU_GEMM64_TMA: -1 (default) automatic, 0 off, k+1 forces TMA config k.
bool launch_gemm_f64_tma(const GemmParams<double>& p, bool ta, bool tb, cudaStream_t s, int cfg) {
  const int forced = env_int("RECTRI_CU_GEMM64_TMA", -1);
  if (forced == 0 || !tma_eligible(p)) return false;
  if (forced > 0 && forced <= kNumTma) cfg = forced - 1;
  if (cfg < 0 || cfg >= kNumTma) return false;
  return kTmaRuns[cfg](p, ta, tb, s);
}

}  // namespace rectri_cu
