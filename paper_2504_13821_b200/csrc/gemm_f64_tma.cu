// gemm_f64_tma.cu -- host side of the TMA-fed fp64 DMMA GEMM: tensor-map
// encoding (driver entry point, no -lcuda link) and configuration choice.
#include <cstdlib>
#include <map>
#include <mutex>

#include "gemm_f64_tma.cuh"
#include "gemm_f64_tma_cfgs.h"
#include "gemm_f64_sk.cuh"

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

// ---------------------------------------------------------------------------
// Stream-K schedule (gemm_f64_sk.cuh): 64x64 tiles, 2x2 consumer warps +
// producer, 4 stages -- the data-parallel default's geometry, so identical bits.
namespace {
constexpr int kSkBM = 64, kSkBN = 64, kSkStages = 4;

template <bool MC_A, bool MC_B>
constexpr int sk_smem() {
  constexpr int slot_a = ((MC_A ? kSkBM + 4 : kSkBM) * dgemm_tma::kBK * 8 + 1023) / 1024 * 1024;
  constexpr int slot_b = ((MC_B ? kSkBN + 4 : kSkBN) * dgemm_tma::kBK * 8 + 1023) / 1024 * 1024;
  return kSkStages * (slot_a + slot_b) + 16 * kSkStages + 1024;
}

// Resident CTAs of the stream-K kernel on the current device (cached).
int sk_slots() {
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return 0;
  if (!cached[dev]) {
    auto kern = dgemm_tma::dgemm_sk_kernel<kSkBM, kSkBN, 2, 2, kSkStages, true, false>;
    const int smem = sk_smem<true, true>();
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int per_sm = 0, sms = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 5 * 32, smem);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cached[dev] = per_sm * sms;
  }
  return cached[dev];
}

// Per-(device, stream) workspace of direct launches: G partial tiles + flags.
struct SkWs {
  double* ws = nullptr;
  int* flags = nullptr;
  int ctas = 0;
};
std::mutex g_sk_mu;
std::map<std::pair<int, cudaStream_t>, SkWs> g_sk_ws;

template <bool MC_A, bool MC_B>
void sk_launch(const CUtensorMap& ma, const CUtensorMap& mb, const GemmParams<double>& p,
               const dgemm_tma::SkPlan& q, double* ws, int* flags, cudaStream_t s) {
  auto kern = dgemm_tma::dgemm_sk_kernel<kSkBM, kSkBN, 2, 2, kSkStages, MC_A, MC_B>;
  constexpr int smem = sk_smem<MC_A, MC_B>();
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  kern<<<q.G, 5 * 32, smem, s>>>(ma, mb, p, q, ws, flags);
  ++launch_counter();
}
}  // namespace

size_t gemm_sk_ws_bytes(int ctas) {
  return static_cast<size_t>(ctas) * (4 * 32 * 32) * sizeof(double) + static_cast<size_t>(ctas) * sizeof(int);
}
int gemm_sk_ctas() { return sk_slots(); }

// RECTRI_CU_GEMM_SK: 0 off; otherwise stream-K when the tile count lies in
// (G, RECTRI_CU_GEMM_SK_WAVES x G] (default 6 waves: beyond that the
// data-parallel tail is small).
bool launch_gemm_f64_sk(const GemmParams<double>& p, bool ta, bool tb, cudaStream_t s) {
  static const int mode = env_int("RECTRI_CU_GEMM_SK", 1);
  static const int waves = env_int("RECTRI_CU_GEMM_SK_WAVES", 6);
  if (!mode || env_int("RECTRI_CU_GEMM64_TMA", -1) >= 0 || !tma_eligible(p)) return false;
  const int G = sk_slots();
  const long long tm = ceil_div(p.M, kSkBM), tn = ceil_div(p.N, kSkBN), T = tm * tn;
  if (G <= 0 || T <= G || T > static_cast<long long>(waves) * G) return false;
  double* ws = nullptr;
  int* flags = nullptr;
  if (const CallScratch* cs = call_scratch()) {  // a graph capture: the graph's own workspace
    const int k = cs->find(s);
    if (k < 0 || !cs->gemm_ws[k] || cs->gemm_ctas[k] < G) return false;
    ws = cs->gemm_ws[k];
    flags = reinterpret_cast<int*>(ws + static_cast<size_t>(G) * 4 * 32 * 32);
  } else {
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &st);
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(g_sk_mu);
    SkWs& w = g_sk_ws[{dev, s}];
    if (w.ctas < G) {
      if (st != cudaStreamCaptureStatusNone) return false;  // no allocation inside a foreign capture
      if (w.ws) {
        cudaStreamSynchronize(s);
        cudaFree(w.ws);
      }
      w = SkWs{};
      if (cudaMalloc(&w.ws, gemm_sk_ws_bytes(G)) != cudaSuccess) {
        cudaGetLastError();
        return false;
      }
      w.flags = reinterpret_cast<int*>(w.ws + static_cast<size_t>(G) * 4 * 32 * 32);
      cudaMemsetAsync(w.flags, 0, static_cast<size_t>(G) * sizeof(int), s);
      cudaStreamSynchronize(s);
      w.ctas = G;
    }
    ws = w.ws;
    flags = w.flags;
  }
  const bool mc_a = !ta, mc_b = tb;
  CUtensorMap ma, mb;
  if (!encode_operand(&ma, p.A, p.lda, p.M, p.K, kSkBM, mc_a)) return false;
  if (!encode_operand(&mb, p.B, p.ldb, p.N, p.K, kSkBN, mc_b)) return false;
  dgemm_tma::SkPlan q;
  q.tiles_m = static_cast<int>(tm);
  q.tiles_n = static_cast<int>(tn);
  q.KT = static_cast<int>(ceil_div(p.K, dgemm_tma::kBK));
  q.W = T * q.KT;
  q.G = G;
  if (mc_a && !mc_b) sk_launch<true, false>(ma, mb, p, q, ws, flags, s);
  else if (!mc_a && !mc_b) sk_launch<false, false>(ma, mb, p, q, ws, flags, s);
  else if (mc_a && mc_b) sk_launch<true, true>(ma, mb, p, q, ws, flags, s);
  else sk_launch<false, true>(ma, mb, p, q, ws, flags, s);
  return true;
}

}  // namespace rectri_cu
