// gemm_tma.cu — host side of the TMA-fed DMMA GEMM (gemm4.cuh): tensor-map
// encoding (cuTensorMapEncodeTiled through the runtime's driver entry point,
// no link-time libcuda dependency), tile selection and launch.
#include <cuda.h>

#include <cstdlib>

#include "gemm4.cuh"
#include "kernels.h"

namespace lrgw_dev {

namespace {

using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled encoder() {
  static const EncodeTiled fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      return static_cast<EncodeTiled>(nullptr);
    }
    return reinterpret_cast<EncodeTiled>(p);
  }();
  return fn;
}

// Column-major rows x cols matrix (rows contiguous, ld >= rows) as a 2-D
// tensor of boxes {16 rows, bk columns}, 128-byte swizzle.
bool encode_mn(CUtensorMap* map, const double* ptr, long long rows, long long cols, long long ld, int bk) {
  EncodeTiled enc = encoder();
  if (!enc || rows < 1 || cols < 1) return false;
  if ((reinterpret_cast<uintptr_t>(ptr) & 15) != 0 || (ld * 8) % 16 != 0) return false;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(cols)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 8};
  const cuuint32_t box[2] = {16, static_cast<cuuint32_t>(bk)};
  const cuuint32_t estr[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(ptr), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// K-contiguous rows x k matrix (A(r, k) at r * ld + k) as a 2-D tensor of
// boxes {16 k, box_rows rows}, 128-byte swizzle.
bool encode_k(CUtensorMap* map, const double* ptr, long long rows, long long k, long long ld, int box_rows) {
  EncodeTiled enc = encoder();
  if (!enc || rows < 1 || k < 1) return false;
  if ((reinterpret_cast<uintptr_t>(ptr) & 15) != 0 || (ld * 8) % 16 != 0) return false;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(k), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 8};
  const cuuint32_t box[2] = {16, static_cast<cuuint32_t>(box_rows)};
  const cuuint32_t estr[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(ptr), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// K-contiguous SYRK configurations (LRGW_TMA_KCFG picks one; measured in profiles/r02/)
using K4 = Gemm4kCfg<128, 128, 64, 32, 5, 1>;         // 8 compute warps, thread 0 refills
using K4P = Gemm4kCfg<96, 96, 48, 48, 6, 1, true>;     // 4 compute warps + TMA warp
using K4S = Gemm4kCfg<64, 64, 32, 32, 6, 2, true>;     // 4 compute warps + TMA warp, 2 CTAs per SM
// Measured with the wave-aware split-K (tools/bench_syrk.py,
// profiles/r02/syrk_splits.txt): 128 x 128 tiles where 128 divides N_mu
// (1024: 0.804, 3456: 0.886, 8192: 0.912 of the DMMA peak against 0.782 /
// 0.862 / 0.897 for 64 x 64), the 64 x 64 two-CTA tiles for other widths
// (960: 0.805 vs 0.709 — a half-empty 128 edge tile row). LRGW_TMA_KCFG
// forces one.
int kcfg(int m) {
  static const int v = getenv("LRGW_TMA_KCFG") ? atoi(getenv("LRGW_TMA_KCFG")) : -1;
  if (v >= 0) return v;
  return m % 128 != 0 ? 2 : 0;
}

template <class Cfg>
cudaError_t launch4(cudaStream_t st, const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& a2,
                    const CUtensorMap& b2, const Dgemm4Params& p) {
  auto kern = dgemm4_kernel<Cfg>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES);
  if (e != cudaSuccess) return e;
  dim3 grid((p.N + Cfg::BN - 1) / Cfg::BN, (p.M + Cfg::BM - 1) / Cfg::BM);
  kern<<<grid, Cfg::THREADS, Cfg::SMEM_BYTES, st>>>(a, b, a2, b2, p);
  count_launches(1);
  return cudaGetLastError();
}

constexpr int kBK = 16;
// 64 x 32 warp tiles, 2 warp rows; BN = 32 x warp columns
template <int BN>
using T4 = Gemm4Cfg<128, BN, 64, 32, kBK, 4, false, 1>;         // + TMA warp
using T4S = Gemm4Cfg<128, 128, 64, 32, kBK, 4, false, 1, false>;  // thread 0 refills
int mncfg() {
  static const int v = getenv("LRGW_TMA_MNCFG") ? atoi(getenv("LRGW_TMA_MNCFG")) : 0;
  return v;
}
// Tall-skinny outputs (the selection's L-pass and W columns, N = 33..112):
// 64-row CTAs of 4 compute warps whose 16-row warp tiles span every column,
// 2 CTAs per SM (+ the TMA warp each). Measured against the cp.async family
// (tools/bench_tall.py, profiles/r02/tall_engines.txt): 884736 x 80 x 7000
// 87.0 -> 94.1 %, x 96 89.8 -> 92.9 %, x 112 -> 94.7 % of the DMMA peak; the
// Hadamard pair 884736 x 96 x (1024 + 1024) 84.9 -> 91.3 %.
// LRGW_TMA_TALL=0 keeps these shapes on the cp.async family.
using TT64 = Gemm4Cfg<128, 64, 32, 32, kBK, 5, false, 1>;   // 8 compute warps of 32 x 32
using TT80 = Gemm4Cfg<64, 80, 16, 80, kBK, 4, false, 2>;
using TT96 = Gemm4Cfg<64, 96, 16, 96, kBK, 4, false, 2>;
using TT112 = Gemm4Cfg<64, 112, 16, 112, kBK, 4, false, 2>;
using HT64 = Gemm4Cfg<64, 64, 16, 64, kBK, 4, true, 2>;
using HT80 = Gemm4Cfg<64, 80, 16, 80, kBK, 4, true, 2>;
using HT96 = Gemm4Cfg<64, 96, 16, 96, kBK, 4, true, 2>;
// Hadamard pair: two accumulator sets -> 32 x 32 warp tiles
template <int BN>
using H4 = Gemm4Cfg<64, BN, 32, 32, kBK, 4, true, 1>;

}  // namespace

bool tma_encode_mn(void* map, const double* ptr, long long rows, long long cols, long long ld, int bk) {
  return encode_mn(static_cast<CUtensorMap*>(map), ptr, rows, cols, ld, bk);
}

int dgemm_tma_k_tile(int m) { return kcfg(m) == 1 ? K4P::BM : kcfg(m) == 2 ? K4S::BM : K4::BM; }
int dgemm_tma_k_per_sm(int m) { return kcfg(m) == 2 ? K4S::MINB : 1; }

template <class Cfg>
cudaError_t launch4k(cudaStream_t st, int M, int N, int K, const double* A, long long lda, const double* B,
                     long long ldb, double* C, long long ldc, double alpha, double beta, const double* scale,
                     bool lower, int splits, int k_chunk, double* partial) {
  if (K <= 0 || (lower && M != N) || (splits > 1 && (!partial || k_chunk % 16 != 0))) return cudaErrorNotSupported;
  CUtensorMap ma, mb;
  if (!encode_k(&ma, A, M, K, lda, Cfg::BM) || !encode_k(&mb, B, N, K, ldb, Cfg::BN)) return cudaErrorNotSupported;
  Dgemm4kParams p{};
  p.M = M, p.N = N, p.K = K, p.C = C, p.ldc = ldc, p.alpha = alpha, p.beta = beta, p.scale = scale;
  p.lower = lower ? 1 : 0;
  if (splits > 1) {
    p.k_chunk = k_chunk;
    p.partial = partial;
    p.part_stride = (long long)M * N;
  }
  auto kern = dgemm4k_kernel<Cfg>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES);
  if (e != cudaSuccess) return e;
  const int tm = (M + Cfg::BM - 1) / Cfg::BM, tn = (N + Cfg::BN - 1) / Cfg::BN;
  dim3 grid(lower ? tm * (tm + 1) / 2 : tn, lower ? 1 : tm, splits > 1 ? splits : 1);
  kern<<<grid, Cfg::THREADS, Cfg::SMEM_BYTES, st>>>(ma, mb, p);
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t dgemm_tma_k(cudaStream_t st, int M, int N, int K, const double* A, long long lda, const double* B,
                        long long ldb, double* C, long long ldc, double alpha, double beta, const double* scale,
                        bool lower, int splits, int k_chunk, double* partial) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  switch (kcfg(M)) {
    case 1: return launch4k<K4P>(st, M, N, K, A, lda, B, ldb, C, ldc, alpha, beta, scale, lower, splits, k_chunk, partial);
    case 2: return launch4k<K4S>(st, M, N, K, A, lda, B, ldb, C, ldc, alpha, beta, scale, lower, splits, k_chunk, partial);
    default: {
      // ring depth of the 128 x 128 configuration (LRGW_TMA_KSTAGES = 5 / 6 / 7; 32 KB per stage)
      static const int stages = getenv("LRGW_TMA_KSTAGES") ? atoi(getenv("LRGW_TMA_KSTAGES")) : 5;
      if (stages == 7)
        return launch4k<Gemm4kCfg<128, 128, 64, 32, 7, 1>>(st, M, N, K, A, lda, B, ldb, C, ldc, alpha, beta, scale, lower, splits, k_chunk, partial);
      if (stages == 6)
        return launch4k<Gemm4kCfg<128, 128, 64, 32, 6, 1>>(st, M, N, K, A, lda, B, ldb, C, ldc, alpha, beta, scale, lower, splits, k_chunk, partial);
      return launch4k<K4>(st, M, N, K, A, lda, B, ldb, C, ldc, alpha, beta, scale, lower, splits, k_chunk, partial);
    }
  }
}

// Persistent MN engine (dgemm4p_kernel): LRGW_TMA_PERSIST=0 / 1.
bool persist_enabled() {
  static const bool on = !(getenv("LRGW_TMA_PERSIST") && atoi(getenv("LRGW_TMA_PERSIST")) == 0);
  return on;
}

bool tma_tall_enabled() {
  static const bool on = !(getenv("LRGW_TMA_TALL") && atoi(getenv("LRGW_TMA_TALL")) == 0);
  return on;
}

// On by default (LRGW_TMA=0 turns it off). Measured (tools/bench_gemm.py,
// profiles/r02/gemm_engines.txt): 110592 x 1024 x 1024 86.0 -> 93.9 % and
// 8192^3 89.0 -> 95.7 % of the DMMA peak against the cp.async engines.
bool tma_gemm_enabled() {
  static const bool on = !(getenv("LRGW_TMA") && atoi(getenv("LRGW_TMA")) == 0);
  return on && encoder() != nullptr;
}

cudaError_t dgemm_tma(cudaStream_t st, int M, int N, int K, const double* A, long long lda, const double* B,
                      long long ldb, double* C, long long ldc, double alpha, double beta, bool tri_b,
                      const int* colmap, const int* n_dev) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  if (K <= 0) return cudaErrorNotSupported;
  CUtensorMap ma, mb;
  if (!encode_mn(&ma, A, M, K, lda, kBK) || !encode_mn(&mb, B, N, K, ldb, kBK)) return cudaErrorNotSupported;
  Dgemm4Params p{};
  p.M = M, p.N = N, p.K = K, p.C = C, p.ldc = ldc, p.alpha = alpha, p.beta = beta;
  p.tri_b = tri_b ? 1 : 0, p.colmap = colmap, p.n_dev = n_dev;
  p.vec_store = (reinterpret_cast<uintptr_t>(C) & 15) == 0 && ldc % 2 == 0;
  if (N < 128) {
    // tall-skinny: one column tile of width 16 ceil(N / 16) (>= 2 waves of CTAs)
    if (n_dev || N <= 32 || !tma_tall_enabled() || (long long)((M + 63) / 64) < 2LL * 148)
      return cudaErrorNotSupported;
    if (N <= 64) return launch4<TT64>(st, ma, mb, ma, mb, p);
    if (N <= 80) return launch4<TT80>(st, ma, mb, ma, mb, p);
    if (N <= 96) return launch4<TT96>(st, ma, mb, ma, mb, p);
    if (N <= 112) return launch4<TT112>(st, ma, mb, ma, mb, p);
  }
  if (n_dev) return cudaErrorNotSupported;
  if (mncfg() == 1) return launch4<T4S>(st, ma, mb, ma, mb, p);
  if (persist_enabled()) {
    using C = T4<128>;
    using C6 = Gemm4Cfg<128, 128, 64, 32, kBK, 6, false, 1>;  // LRGW_TMA_MNSTAGES=6: a 6-deep ring (192 KB)
    static const int stages = getenv("LRGW_TMA_MNSTAGES") ? atoi(getenv("LRGW_TMA_MNSTAGES")) : 4;
    auto kern = stages == 6 ? dgemm4p_kernel<C6> : dgemm4p_kernel<C>;
    const int smem = stages == 6 ? C6::SMEM_BYTES : C::SMEM_BYTES;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    const int tm = (M + C::BM - 1) / C::BM, tn = (N + C::BN - 1) / C::BN;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int grid = std::min(tm * tn, sms * C::MINB);
    kern<<<grid, C::THREADS, smem, st>>>(ma, mb, p, tm, tn);
    count_launches(1);
    return cudaGetLastError();
  }
  return launch4<T4<128>>(st, ma, mb, ma, mb, p);
}

cudaError_t hadamard_tma(cudaStream_t st, int M, int N, const double* a1, long long lda1, const double* b1,
                         long long ldb1, int k1, const double* a2, long long lda2, const double* b2, long long ldb2,
                         int k2, double* C, long long ldc, double alpha, double beta) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  if (k1 <= 0 || k2 <= 0) return cudaErrorNotSupported;
  CUtensorMap ma, mb, ma2, mb2;
  if (!encode_mn(&ma, a1, M, k1, lda1, kBK) || !encode_mn(&mb, b1, N, k1, ldb1, kBK) ||
      !encode_mn(&ma2, a2, M, k2, lda2, kBK) || !encode_mn(&mb2, b2, N, k2, ldb2, kBK))
    return cudaErrorNotSupported;
  Dgemm4Params p{};
  p.M = M, p.N = N, p.K = k1, p.K2 = k2, p.C = C, p.ldc = ldc, p.alpha = alpha, p.beta = beta;
  p.vec_store = (reinterpret_cast<uintptr_t>(C) & 15) == 0 && ldc % 2 == 0;
  if (N > 32 && N <= 96 && tma_tall_enabled() && (long long)((M + 63) / 64) >= 2LL * 148) {
    if (N <= 64) return launch4<HT64>(st, ma, mb, ma2, mb2, p);
    if (N <= 80) return launch4<HT80>(st, ma, mb, ma2, mb2, p);
    return launch4<HT96>(st, ma, mb, ma2, mb2, p);
  }
  const int w = (N + 31) / 32;
  if (w >= 4) return launch4<H4<128>>(st, ma, mb, ma2, mb2, p);
  if (w == 3) return launch4<H4<96>>(st, ma, mb, ma2, mb2, p);
  return launch4<H4<64>>(st, ma, mb, ma2, mb2, p);
}

}  // namespace lrgw_dev
