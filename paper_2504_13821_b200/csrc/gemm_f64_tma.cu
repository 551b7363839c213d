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

namespace {
template <bool MC_A, bool MC_B>
int split_smem() {
  constexpr int slot_a = ((MC_A ? 64 + 4 : 64) * dgemm_tma::kBK * 8 + 1023) / 1024 * 1024;
  constexpr int slot_b = ((MC_B ? 64 + 4 : 64) * dgemm_tma::kBK * 8 + 1023) / 1024 * 1024;
  return 4 * (slot_a + slot_b) + 16 * 4 + 1024;
}

// Resident CTAs of the 64x64 kernels on the current device (cached).
int slots64() {
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return 0;
  if (!cached[dev]) {
    auto kern = dgemm_tma::dgemm_tma_split_kernel<true, true>;
    const int smem = split_smem<true, true>();
    set_smem(kern, smem);
    int per_sm = 0, sms = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 5 * 32, smem);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cached[dev] = per_sm * sms;
  }
  return cached[dev];
}

template <bool MC_A, bool MC_B>
bool split_launch(const GemmParams<double>& p, int n_main, cudaStream_t s) {
  CUtensorMap a64, b64, a32, b32;
  if (!encode_operand(&a64, p.A, p.lda, p.M, p.K, 64, MC_A) || !encode_operand(&b64, p.B, p.ldb, p.N, p.K, 64, MC_B) ||
      !encode_operand(&a32, p.A, p.lda, p.M, p.K, 32, MC_A) || !encode_operand(&b32, p.B, p.ldb, p.N, p.K, 32, MC_B))
    return false;
  auto kern = p.ring_check ? dgemm_tma::dgemm_tma_split_kernel<MC_A, MC_B, true>
                           : dgemm_tma::dgemm_tma_split_kernel<MC_A, MC_B>;
  const int smem = split_smem<MC_A, MC_B>();
  set_smem(kern, smem);
  const long long grid = ceil_div(p.M, 64) * (n_main / 64) + ceil_div(p.M, 32) * ceil_div(p.N - n_main, 32);
  launch_kernel(kern, static_cast<unsigned>(grid), 5 * 32, smem, s, a64, b64, a32, b32, p, n_main);
  ++launch_counter();
  return true;
}
}  // namespace

// Wave-tail split (dgemm_tma_split_kernel): when the 64x64 tiles make a
// whole number of resident waves plus a short last one, the columns of that
// last wave go to 32x32 tiles (RECTRI_CU_GEMM64_SPLIT: 0 off; 2 forces a
// split at half of N, for the bitwise tests).  Same bits as config 1.
bool launch_gemm_f64_split(const GemmParams<double>& p, bool ta, bool tb, cudaStream_t s) {
  const int mode = env_int("RECTRI_CU_GEMM64_SPLIT", 1);
  if (!mode || env_int("RECTRI_CU_GEMM64_TMA", -1) >= 0 || !tma_eligible(p)) return false;
  const long long tm = ceil_div(p.M, 64), tn = ceil_div(p.N, 64), T = tm * tn;
  long long n_main = 0;
  if (mode == 2) {
    n_main = (p.N / 2) / 64 * 64;
  } else {
    const long long S = slots64();
    if (S <= 0 || T <= S || T >= 8 * S) return false;
    const long long waves = T / S;
    if (static_cast<double>(T - waves * S) / S > 0.5) return false;  // the last wave is full enough
    n_main = (waves * S / tm) * 64;
  }
  if (n_main <= 0 || n_main >= p.N) return false;
  const bool mc_a = !ta, mc_b = tb;
  if (mc_a && !mc_b) return split_launch<true, false>(p, static_cast<int>(n_main), s);
  if (!mc_a && !mc_b) return split_launch<false, false>(p, static_cast<int>(n_main), s);
  if (mc_a && mc_b) return split_launch<true, true>(p, static_cast<int>(n_main), s);
  return split_launch<false, true>(p, static_cast<int>(n_main), s);
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
