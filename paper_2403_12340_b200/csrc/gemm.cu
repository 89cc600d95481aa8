// gemm.cu — dispatch for the FP64 DMMA GEMM engine (gemm.cuh) plus the small
// elementwise kernels the path needs (split-K reduction, symmetric mirror,
// row gather).
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "gemm.cuh"
#include "gemm2.cuh"
#include "gemm3.cuh"
#include "kernels.h"

namespace lrgw_dev {

namespace {

// Large tiles: 128x64 CTA, 8 warps of 32x32, 3 stages (~90 KB smem, 2 CTA/SM).
// Small tiles: 64x64 CTA, 4 warps of 32x32, 4 stages (~80 KB smem, 2 CTA/SM).
template <bool AK, bool BK, int VA, int VB>
using CfgL = GemmCfg<128, 64, 32, 32, 3, AK, BK, VA, VB, 16, 2>;
template <bool AK, bool BK, int VA, int VB>
using CfgS = GemmCfg<64, 64, 32, 32, 4, AK, BK, VA, VB, 16, 2>;
// Square 128x128 CTA, 16 warps of 32x32, 3 stages (~120 KB smem, 1 CTA/SM):
// the symmetric (lower-tile) split-K SYRK of Theta^T V Theta.
template <bool AK, bool BK, int VA, int VB>
using CfgX = GemmCfg<128, 128, 32, 32, 3, AK, BK, VA, VB, 32>;

// Hadamard pair (two live accumulator sets): 128x64 CTA, 16 warps of 32x16;
// 128x32 CTA, 8 warps of 32x16 when N would otherwise pad badly.
template <int V>
using CfgH = GemmCfg<128, 64, 32, 16, 3, false, false, V, V>;
template <int V>
using CfgH32 = GemmCfg<128, 32, 32, 16, 3, false, false, V, V>;
// Tall-skinny outputs (N not a multiple of 64): 128x32 CTA, 4 warps of 32x32.
template <bool AK, bool BK, int VA, int VB>
using CfgN = GemmCfg<128, 32, 32, 32, 4, AK, BK, VA, VB, 16, 2>;
// Single-column-tile widths 96 / 128 for the tall-skinny GEMMs of the
// selection (N = new candidates, K = pivots so far): 12 / 16 warps of 32x32.
template <bool AK, bool BK, int VA, int VB>
using Cfg96 = GemmCfg<128, 96, 32, 32, 3, AK, BK, VA, VB>;

// Tall-skinny family (M >> N, N <= 128, A MN-contiguous): one column tile of
// width 16 Q (Q = ceil(N / 16)) so at most 15 padded columns, 8 warps of
// 32 x 8Q. A is streamed from HBM exactly once.
template <int Q, bool BK>
using CfgT = GemmCfg<128, 16 * Q, 32, 8 * Q, 3, false, BK, 2, 2, (Q >= 5 ? 32 : 16)>;
// (Hadamard: two live accumulator sets, so 64-row tiles of 8 warps of
// 16 x 8Q beyond Q = 5.)
template <int Q>
using CfgHT = typename std::conditional<(Q <= 5), GemmCfg<128, 16 * Q, 32, 8 * Q, 3, false, false, 2, 2>,
                                        GemmCfg<64, 16 * Q, 16, 8 * Q, 3, false, false, 2, 2>>::type;

enum class Tile { S, L, X, N, W96, W128, T };

// Column padding of an N-wide output under 64- vs 32-wide tiles.
bool prefer_narrow(int N) {
  const int p64 = (N + 63) / 64 * 64, p32 = (N + 31) / 32 * 32;
  return p32 * 5 < p64 * 4;  // narrow tiles save > 20% padded work
}

template <class Cfg>
cudaError_t launch_cfg(cudaStream_t st, const DgemmParams& p, int splits) {
  dim3 grid;
  if (p.lower) {
    const int t = (p.M + Cfg::BM - 1) / Cfg::BM;
    grid = dim3(t * (t + 1) / 2, 1, splits);
  } else {
    grid = dim3((p.N + Cfg::BN - 1) / Cfg::BN, (p.M + Cfg::BM - 1) / Cfg::BM, splits);
  }
  if (grid.x == 0 || grid.y == 0) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(dgemm_kernel<Cfg>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES);
  if (e != cudaSuccess) return e;
  dgemm_kernel<Cfg><<<grid, Cfg::THREADS, Cfg::SMEM_BYTES, st>>>(p); count_launches(1);
  return cudaGetLastError();
}

template <bool AK, bool BK>
cudaError_t launch_layout(cudaStream_t st, const DgemmParams& p, Tile tile, bool va, bool vb,
                          int splits) {
  if (tile == Tile::L) {
    if (va && vb) return launch_cfg<CfgL<AK, BK, 2, 2>>(st, p, splits);
    return launch_cfg<CfgL<AK, BK, 1, 1>>(st, p, splits);
  }
  if (tile == Tile::X) {
    if (va && vb) return launch_cfg<CfgX<AK, BK, 2, 2>>(st, p, splits);
    return launch_cfg<CfgX<AK, BK, 1, 1>>(st, p, splits);
  }
  if (tile == Tile::N) {
    if (va && vb) return launch_cfg<CfgN<AK, BK, 2, 2>>(st, p, splits);
    return launch_cfg<CfgN<AK, BK, 1, 1>>(st, p, splits);
  }
  if (tile == Tile::W96) {
    if (va && vb) return launch_cfg<Cfg96<AK, BK, 2, 2>>(st, p, splits);
    return launch_cfg<Cfg96<AK, BK, 1, 1>>(st, p, splits);
  }
  if (tile == Tile::W128) {
    if (va && vb) return launch_cfg<CfgX<AK, BK, 2, 2>>(st, p, splits);
    return launch_cfg<CfgX<AK, BK, 1, 1>>(st, p, splits);
  }
  if (va && vb) return launch_cfg<CfgS<AK, BK, 2, 2>>(st, p, splits);
  return launch_cfg<CfgS<AK, BK, 1, 1>>(st, p, splits);
}

template <bool BK>
cudaError_t launch_tall(cudaStream_t st, const DgemmParams& p, int q) {
  switch (q) {
    case 1:
    case 2: return launch_cfg<CfgT<2, BK>>(st, p, 1);
    case 3: return launch_cfg<CfgT<3, BK>>(st, p, 1);
    case 4: return launch_cfg<CfgT<4, BK>>(st, p, 1);
    case 5: return launch_cfg<CfgT<5, BK>>(st, p, 1);
    case 6: return launch_cfg<CfgT<6, BK>>(st, p, 1);
    case 7: return launch_cfg<CfgT<7, BK>>(st, p, 1);
    default: return launch_cfg<CfgT<8, BK>>(st, p, 1);
  }
}

// The TMA Hadamard pair: the tall widths 33..96 (16-row warp tiles) by default,
// the 32 x 32-warp-tile configuration for the other widths opt-in (LRGW_TMA_HAD=1).
bool tma_k_enabled() {
  static const bool on = !(getenv("LRGW_TMA_K") && atoi(getenv("LRGW_TMA_K")) == 0);
  return on;
}

bool hadamard_tma_enabled() {
  static const bool on = getenv("LRGW_TMA_HAD") && atoi(getenv("LRGW_TMA_HAD")) == 1;
  return on;
}

bool tall_family_enabled() {
  static const bool on = !(getenv("LRGW_TALL") && atoi(getenv("LRGW_TALL")) == 0);
  return on;
}

// ---- v3 (paired fragments for either layout) configurations ---------------
// Symmetric (lower-tile) outputs: 64 x 64 tiles, 4 warps of 32 x 32, 3 per SM.
template <bool AK, bool BK, int V>
using G3S = Gemm3Cfg<64, 64, 32, 32, 3, AK, BK, V, 16, 3>;

template <class Cfg>
cudaError_t launch3(cudaStream_t st, const DgemmParams& p, int splits) {
  dim3 grid;
  if (p.lower) {
    const int t = (p.M + Cfg::BM - 1) / Cfg::BM;
    grid = dim3(t * (t + 1) / 2, 1, splits);
  } else {
    grid = dim3((p.N + Cfg::BN - 1) / Cfg::BN, (p.M + Cfg::BM - 1) / Cfg::BM, splits);
  }
  if (grid.x == 0 || grid.y == 0) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(dgemm3_kernel<Cfg>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       Cfg::SMEM_BYTES);
  if (e != cudaSuccess) return e;
  dgemm3_kernel<Cfg><<<grid, Cfg::THREADS, Cfg::SMEM_BYTES, st>>>(p); count_launches(1);
  return cudaGetLastError();
}

template <template <bool, bool, int> class C>
cudaError_t launch3_layout(cudaStream_t st, const DgemmParams& p, bool ak, bool bk, bool vec, int splits) {
  if (vec) {
    if (!ak && !bk) return launch3<C<false, false, 2>>(st, p, splits);
    if (!ak && bk) return launch3<C<false, true, 2>>(st, p, splits);
    if (ak && !bk) return launch3<C<true, false, 2>>(st, p, splits);
    return launch3<C<true, true, 2>>(st, p, splits);
  }
  if (!ak && !bk) return launch3<C<false, false, 1>>(st, p, splits);
  if (!ak && bk) return launch3<C<false, true, 1>>(st, p, splits);
  if (ak && !bk) return launch3<C<true, false, 1>>(st, p, splits);
  return launch3<C<true, true, 1>>(st, p, splits);
}

// Split count that fills whole waves of `slots` resident CTAs: the smallest
// s (each split >= 16 k-tiles) whose last wave is >= 90% full, else the best.
int choose_splits(long long tiles, int ktiles, long long slots) {
  // chunks of >= 16 k-tiles; >= 4 when the tile grid is a handful of CTAs
  const int min_chunk = tiles * 8 < slots ? 4 : 16;
  const int smax = std::max(1, std::min(ktiles / min_chunk, 64));
  int best = 1;
  double best_eff = 0.0;
  for (int s = 1; s <= smax; ++s) {
    const long long ctas = tiles * s;
    const long long waves = (ctas + slots - 1) / slots;
    const double eff = (double)ctas / (double)(waves * slots);
    if (ctas >= slots && eff >= 0.9) return s;
    if (eff > best_eff + 1e-9) {
      best_eff = eff;
      best = s;
    }
  }
  return best;
}

// Splits (<= 8) that keep the tile grid closest to whole waves of `slots`;
// a smaller split wins ties within 2 % (each split adds an M N partial to
// the reduction).
int choose_splits_waves(long long tiles, int ktiles, long long slots) {
  const int smax = std::max(1, std::min(ktiles / 16, 8));
  int best = 1;
  double best_eff = 0.0;
  for (int s = 1; s <= smax; ++s) {
    const long long ctas = tiles * s;
    const long long waves = (ctas + slots - 1) / slots;
    const double eff = (double)ctas / (double)(waves * slots);
    if (eff > best_eff + 0.02) {
      best_eff = eff;
      best = s;
    }
  }
  return best;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

__global__ void splitk_reduce_kernel(const double* partial, int splits, long long stride, int M,
                                     int N, double* C, long long ldc, double beta, int lower,
                                     int tile) {
  const long long total = (long long)M * N;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int m = static_cast<int>(idx % M), n = static_cast<int>(idx / M);
    if (lower && (n / tile) > (m / tile)) continue;
    double s = 0.0;
    for (int z = 0; z < splits; ++z) s += partial[z * stride + idx];
    double* c = C + m + (long long)n * ldc;
    *c = (beta == 0.0) ? s : s + beta * (*c);
  }
}

__global__ void mirror_lower_kernel(double* a, int n, long long lda, int average) {
  const long long total = (long long)n * n;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int i = static_cast<int>(idx % n), j = static_cast<int>(idx / n);
    if (i <= j) continue;  // (i, j) strictly lower
    double* lo = a + i + (long long)j * lda;
    double* up = a + j + (long long)i * lda;
    const double v = average ? 0.5 * (*lo + *up) : *lo;
    *lo = v;
    *up = v;
  }
}

__global__ void gather_rows_kernel(const double* src, long long lds, int cols, const int* rows,
                                   int n_rows, double* dst, long long ldd) {
  const long long total = (long long)n_rows * cols;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int r = static_cast<int>(idx % n_rows), c = static_cast<int>(idx / n_rows);
    dst[r + c * ldd] = src[rows[r] + c * lds];
  }
}

// The selection's row gathers in one launch: rows `rows` of three column-major
// sources (a: n1 cols, b: n2 cols, l: nl cols) into three destinations of leading dim ldd.
__global__ void gather_rows3_kernel(const double* a, long long lda, int n1, const double* b, long long ldb, int n2,
                                    const double* l, long long ldl, int nl, const int* rows, int n_rows, double* da,
                                    double* db, double* dl, long long ldd, const int* nl_dev, const int* nrows_dev,
                                    const int* row_off_dev) {
  if (nl_dev) nl = *nl_dev;
  if (nrows_dev) n_rows = *nrows_dev;
  if (row_off_dev) rows += *row_off_dev;
  const long long total = (long long)n_rows * (n1 + n2 + nl);
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int r = static_cast<int>(idx % n_rows);
    int c = static_cast<int>(idx / n_rows);
    const int g = rows[r];
    if (c < n1) {
      da[r + c * ldd] = a[g + c * lda];
    } else if ((c -= n1) < n2) {
      db[r + c * ldd] = b[g + c * ldb];
    } else {
      c -= n2;
      dl[r + c * ldd] = l[g + c * ldl];
    }
  }
}

__global__ void gather_cols_kernel(const double* src, long long lds, int rows, const int* cols, int n,
                                   double* dst, long long ldd) {
  const long long total = (long long)rows * n;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int r = static_cast<int>(idx % rows), c = static_cast<int>(idx / rows);
    dst[r + c * ldd] = src[r + cols[c] * lds];
  }
}

// ---- v2 (paired-fragment) configurations ---------------------------------
// BK = 32 (3-stage ring) for the 128-row-wide 12- and 8-warp configurations,
// BK = 16 for the narrow ones (measured, tools/bench_gemm.py).
template <int V>
using G2W64 = Gemm2Cfg<128, 64, 64, 32, 4, V, false>;
template <int V>
using G2W32 = Gemm2Cfg<128, 32, 32, 32, 4, V, false>;

template <int V>
using H2W64 = Gemm2Cfg<128, 64, 32, 32, 4, V, true>;
template <int V>
using H2W32 = Gemm2Cfg<128, 32, 32, 32, 4, V, true>;

// Tall Hadamard (selection: W columns of the accepted pivots, N = 48..128):
// 64 x 16Q CTAs of 4 warps (16 x 16Q each), 2 per SM.
// Shared memory decides the residency: the parked product (FM FN 2 doubles
// per thread) plus the operand ring must leave room for 8 warps per SM.
//   Q <= 4: 64-row CTAs, 3-stage ring (<= 84 KB: 2 CTAs per SM);
//   Q 5-7:  64-row CTAs, 2-stage ring (<= 105 KB: 2 CTAs per SM) or, with
//           LRGW_HAD_WIDE=1, 128-row CTAs of 8 warps with a 3-stage ring (1 per SM).
template <int Q>
using H2T = Gemm2Cfg<64, 16 * Q, 16, 16 * Q, (Q <= 4 ? 3 : 2), 2, true, 16, 2, false, true>;
template <int Q>
using H2TW = Gemm2Cfg<128, 16 * Q, 16, 16 * Q, 3, 2, true, 16, 1, false, true>;
// widths 113-128: BK = 8 keeps the 2-stage ring + parked product at 91 KB (2 CTAs per SM)
using H2T8 = Gemm2Cfg<64, 128, 16, 128, 2, 2, true, 8, 2, false, true>;

bool had128_park() {
  static const bool on = !(getenv("LRGW_HAD128") && atoi(getenv("LRGW_HAD128")) == 0);
  return on;
}

bool had_wide() {
  static const bool on = getenv("LRGW_HAD_WIDE") && atoi(getenv("LRGW_HAD_WIDE")) == 1;
  return on;
}

bool had_tall_v2_enabled() {
  static const bool on = !(getenv("LRGW_HAD_TALL") && atoi(getenv("LRGW_HAD_TALL")) == 0);
  return on;
}

template <class Cfg>
cudaError_t launch2(cudaStream_t st, const Dgemm2Params& p) {
  dim3 grid((p.N + Cfg::BN - 1) / Cfg::BN, (p.M + Cfg::BM - 1) / Cfg::BM);
  if (grid.x == 0 || grid.y == 0) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(dgemm2_kernel<Cfg>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       Cfg::SMEM_BYTES);
  if (e != cudaSuccess) return e;
  dgemm2_kernel<Cfg><<<grid, Cfg::THREADS, Cfg::SMEM_BYTES, st>>>(p); count_launches(1);
  return cudaGetLastError();
}

// Column tile width for an N-wide output: the narrowest padding, preferring wide.
int v2_width(int N) {
  if (N > 96) return 128;
  if (N > 64) return 96;
  if (N > 32) return 64;
  return 32;
}

// 4-warp CTAs of 64 x 96 (warp tiles 32 x 48), 3 resident per SM = 12 warps:
// the occupancy the library DGEMM runs at on this chip (its SASS: 4-warp
// CTAs, 3 per SM). Measured 86-89 % of the DMMA peak on the wide shapes vs
// 83-85 % for the 8-warp 128 x 128 tile (tools/bench_gemm.py).
template <int V>
using G2Q96 = Gemm2Cfg<64, 96, 32, 48, 3, V, false, 16, 3>;

// Tall-skinny widths 48 / 80 / 112: 4-warp 64-row CTAs (warp tiles 16 x 16q).
template <int V>
using G2Q48 = Gemm2Cfg<64, 48, 16, 48, 3, V, false, 16, 3>;
template <int V>
using G2Q80 = Gemm2Cfg<64, 80, 16, 80, 3, V, false, 16, 3>;
template <int V>
using G2Q112 = Gemm2Cfg<64, 112, 16, 112, 3, V, false, 16, 2>;
template <int V>
using G2Q128 = Gemm2Cfg<64, 128, 32, 64, 3, V, false, 16, 2>;
// Device-bounded N: 16 warps of 16 x 32, four per column slice so skipping
// the dead slices unloads every SM sub-partition equally.
template <int V>
using G2N128 = Gemm2Cfg<64, 128, 16, 32, 3, V, false, 16, 2, true>;

// Tall-skinny outputs of width 16q, q odd (the even widths use dispatch2).
template <int V>
cudaError_t dispatch2_odd(cudaStream_t st, const Dgemm2Params& p) {
  const int q = (p.N + 15) / 16;
  if (q >= 8) return launch2<G2Q128<V>>(st, p);
  if (q <= 3) return launch2<G2Q48<V>>(st, p);
  if (q <= 5) return launch2<G2Q80<V>>(st, p);
  if (q <= 6) return launch2<G2Q96<V>>(st, p);
  return launch2<G2Q112<V>>(st, p);
}

template <int V>
cudaError_t dispatch2(cudaStream_t st, const Dgemm2Params& p, bool had) {
  int w = v2_width(p.N);
  if (had) return w <= 32 ? launch2<H2W32<V>>(st, p) : launch2<H2W64<V>>(st, p);
  switch (w) {
    case 32: return launch2<G2W32<V>>(st, p);
    case 64: return launch2<G2W64<V>>(st, p);
    default: return launch2<G2Q96<V>>(st, p);
  }
}

}  // namespace

cudaError_t dgemm_batched(cudaStream_t st, int batch, int M, int N, int K, const double* A, long long lda,
                          long long bsa, Lay la, const double* B, long long ldb, long long bsb, Lay lb, double* C,
                          long long ldc, long long bsc, double alpha, double beta, bool tri_b) {
  if (M <= 0 || N <= 0 || batch <= 0) return cudaSuccess;
  DgemmParams p{};
  p.M = M, p.N = N, p.K = K, p.A = A, p.lda = lda, p.B = B, p.ldb = ldb, p.C = C, p.ldc = ldc;
  p.alpha = alpha, p.beta = beta, p.tri_b = tri_b ? 1 : 0;
  p.batch = batch, p.bsa = bsa, p.bsb = bsb, p.bsc = bsc;
  const bool ak = la == Lay::K, bk = lb == Lay::K;
  const bool va = aligned16(A) && lda % 2 == 0 && bsa % 2 == 0 && (ak ? K % 2 == 0 : (M % 2 == 0 || lda > M));
  const bool vb = aligned16(B) && ldb % 2 == 0 && bsb % 2 == 0 && (bk ? K % 2 == 0 : (N % 2 == 0 || ldb > N));
  if (!ak && !bk) return launch_layout<false, false>(st, p, Tile::S, va, vb, batch);
  if (!ak && bk) return launch_layout<false, true>(st, p, Tile::S, va, vb, batch);
  if (ak && !bk) return launch_layout<true, false>(st, p, Tile::S, va, vb, batch);
  return launch_layout<true, true>(st, p, Tile::S, va, vb, batch);
}

cudaError_t gather_rows3(cudaStream_t st, const double* a, long long lda, int n1, const double* b, long long ldb,
                        int n2, const double* l, long long ldl, int nl, const int* rows, int n_rows, double* da,
                        double* db, double* dl, long long ldd, const int* nl_dev, const int* nrows_dev,
                        const int* row_off_dev) {
  if ((n_rows <= 0 && !nrows_dev) || (n1 + n2 + nl <= 0 && !nl_dev)) return cudaSuccess;
  gather_rows3_kernel<<<592, 256, 0, st>>>(a, lda, n1, b, ldb, n2, l, ldl, nl, rows, n_rows, da, db, dl, ldd, nl_dev,
                                           nrows_dev, row_off_dev);
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t gather_cols(cudaStream_t st, const double* src, long long lds, int rows, const int* cols, int n,
                        double* dst, long long ldd) {
  if (rows <= 0 || n <= 0) return cudaSuccess;
  gather_cols_kernel<<<1184, 256, 0, st>>>(src, lds, rows, cols, n, dst, ldd); count_launches(1);
  return cudaGetLastError();
}

cudaError_t dgemm(cudaStream_t st, int M, int N, int K, const double* A, long long lda, Lay la,
                  const double* B, long long ldb, Lay lb, double* C, long long ldc, double alpha,
                  double beta, const double* scale, bool lower, int sm_count, double* work,
                  size_t work_elems, bool tri_b, const int* colmap, const int* n_dev, const double* cin,
                  long long ldcin, const int* cin_map) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  DgemmParams p{};
  p.M = M;
  p.N = N;
  p.K = K;
  p.A = A;
  p.lda = lda;
  p.B = B;
  p.ldb = ldb;
  p.C = C;
  p.ldc = ldc;
  p.alpha = alpha;
  p.beta = beta;
  p.scale = scale;
  p.lower = lower ? 1 : 0;
  p.tri_b = tri_b ? 1 : 0;
  p.colmap = colmap;
  p.n_dev = n_dev;
  p.Cin = cin;
  p.ldcin = ldcin;
  p.cin_map = cin_map;
  if (cin && (lower || work || !cin_map)) return cudaErrorInvalidValue;
  if ((tri_b || colmap || n_dev) && (lower || work)) return cudaErrorInvalidValue;
  const bool ak = la == Lay::K, bk = lb == Lay::K;
  // TMA-fed engine for K-contiguous operands (the G-space SYRK): 128 x 128
  // tiles (lower ones when symmetric), split-K when the tile grid is small
  if (ak && bk && !cin && !tri_b && !colmap && !n_dev && tma_gemm_enabled() && tma_k_enabled() &&
      (lower || (long long)((M + 127) / 128) * ((N + 127) / 128) >= sm_count)) {
    const int bt = dgemm_tma_k_tile(M);
    const long long tm = (M + bt - 1) / bt, tn = (N + bt - 1) / bt;
    const long long tiles = lower ? tm * (tm + 1) / 2 : tm * tn;
    const int ktiles = (K + 15) / 16;
    int splits = 1, kc = 0;
    // split-K against the wave quantisation of the resident tile slots (a
    // 1485-tile grid on 296 slots runs 5.02 waves: 84 % busy)
    const long long slots = (long long)sm_count * dgemm_tma_k_per_sm(M);
    static const int force = getenv("LRGW_TMA_KSPLITS") ? atoi(getenv("LRGW_TMA_KSPLITS")) : 0;
    if (ktiles >= 32 && work) {
      splits = force > 0 ? force : choose_splits_waves(tiles, ktiles, slots);
      while (splits > 1 && (size_t)splits * M * N > work_elems) --splits;
      if (splits > 1) {
        kc = ((ktiles + splits - 1) / splits) * 16;
        splits = (K + kc - 1) / kc;
      }
    }
    const cudaError_t e = dgemm_tma_k(st, M, N, K, A, lda, B, ldb, C, ldc, alpha, beta, scale, lower, splits, kc,
                                      splits > 1 ? work : nullptr);
    if (e != cudaErrorNotSupported) {
      if (e != cudaSuccess || splits <= 1) return e;
      splitk_reduce_kernel<<<1184, 256, 0, st>>>(work, splits, (long long)M * N, M, N, C, ldc, beta, lower ? 1 : 0,
                                                 bt);
      count_launches(1);
      return cudaGetLastError();
    }
    cudaGetLastError();
  }
  // TMA-fed engine for MN-contiguous operands when the tile grid fills the chip
  if (!ak && !bk && !lower && !scale && !cin && tma_gemm_enabled() &&
      (long long)((M + 127) / 128) * ((N + 127) / 128) >= sm_count) {
    const cudaError_t e = dgemm_tma(st, M, N, K, A, lda, B, ldb, C, ldc, alpha, beta, tri_b, colmap, n_dev);
    if (e != cudaErrorNotSupported) return e;
    cudaGetLastError();
  }
  // 16-byte cp.async needs aligned bases, even leading dims and even extents
  // along the contiguous axis.
  // (an odd M / N is fine with a padded even ld: the straddling pair only
  // feeds output rows / columns that are never stored; an odd K is not)
  const bool va = aligned16(A) && lda % 2 == 0 && (ak ? K % 2 == 0 : (M % 2 == 0 || lda > M));
  const bool vb = aligned16(B) && ldb % 2 == 0 && (bk ? K % 2 == 0 : (N % 2 == 0 || ldb > N));
  if (lower && M != N) return cudaErrorInvalidValue;
  Tile tile;
  long long tiles;
  int occ;
  if (lower) {
    // symmetric outputs: 64x64 lower tiles + split-K (measured faster than
    // 128x128 tiles for the long-K SYRK of Theta^T V Theta: 4.52 vs 4.66 ms)
    tile = Tile::S;
    const long long t = (M + 63) / 64;
    tiles = t * (t + 1) / 2;
    occ = 3;  // v3 engine, 3 CTAs per SM
  } else if (!ak && va && vb && !scale && !n_dev && N > 32 && N <= 128 && ((N + 15) / 16) % 2 == 1 &&
             (long long)((M + 127) / 128) >= 2LL * sm_count && tall_family_enabled()) {
    // tall-skinny with N in (32, 48], (64, 80], (96, 112]: one column tile of
    // width 16 ceil(N / 16) (the 32 / 64 / 96 / 128 tiles cover the rest)
    tile = Tile::T;
    tiles = (M + 127) / 128;
    occ = 1;
  } else if (n_dev && N > 64 && N <= 128 && (long long)((M + 127) / 128) >= 2LL * sm_count) {
    // device-side N bound (the selection's L block): one 128-wide column tile
    // (A streamed once); warps past the live columns skip their MMAs
    tile = Tile::W128;
    tiles = (M + 127) / 128;
    occ = 1;
  } else if (n_dev && (long long)((M + 127) / 128) >= 2LL * sm_count) {
    // device-side N bound: 32-wide column tiles (CTAs past the live columns exit)
    tile = Tile::N;
    tiles = (long long)((M + 127) / 128) * ((N + 31) / 32);
    occ = 2;
  } else if (N > 64 && N <= 128 && (long long)((M + 127) / 128) >= 2LL * sm_count) {
    // one column tile of width 96 or 128 (A streamed once)
    tile = N <= 96 ? Tile::W96 : Tile::W128;
    tiles = (M + 127) / 128;
    occ = 1;
  } else if ((long long)((M + 127) / 128) * ((N + 31) / 32) >= 2LL * sm_count && prefer_narrow(N)) {
    tile = Tile::N;
    tiles = (long long)((M + 127) / 128) * ((N + 31) / 32);
    occ = 2;
  } else if ((long long)((M + 127) / 128) * ((N + 63) / 64) >= 2LL * sm_count) {
    tile = Tile::L;
    tiles = (long long)((M + 127) / 128) * ((N + 63) / 64);
    occ = 2;
  } else {
    tile = Tile::S;
    tiles = (long long)((M + 63) / 64) * ((N + 63) / 64);
    occ = 2;
  }
  // split-K when the output tile grid cannot fill the chip and K is long
  int splits = 1;
  const int ktiles = (K + 15) / 16;
  if (tiles < 2LL * sm_count * occ && (ktiles >= 32 || (tiles * 8 < (long long)sm_count * occ && ktiles >= 8)) &&
      work) {
    splits = choose_splits(tiles, ktiles, (long long)sm_count * occ);
    while (splits > 1 && (size_t)splits * M * N > work_elems) --splits;
  }
  if (splits > 1) {
    const int kc = ((ktiles + splits - 1) / splits) * 16;
    splits = (K + kc - 1) / kc;
    p.k_chunk = kc;
    p.partial = work;
    p.part_stride = (long long)M * N;
  }
  if (lower) {
    // symmetric outputs on the v3 engine (either operand layout, scale, split-K)
    cudaError_t e = launch3_layout<G3S>(st, p, ak, bk, va && vb, splits);
    if (e != cudaSuccess || splits <= 1) return e;
    splitk_reduce_kernel<<<1184, 256, 0, st>>>(work, splits, (long long)M * N, M, N, C, ldc, beta, 1, 64);
    count_launches(1);
    return cudaGetLastError();
  }
  // v2 (paired fragments) wins for full-width tiles; narrow outputs stay on v1
  // (and for tall-skinny outputs whose width is a multiple of 32: 32 / 64 / 96)
  const bool narrow_v2 = !ak && !bk && !lower && !scale && !cin && splits <= 1 && N > 16 &&
                         N <= 128 && (n_dev || ((N + 15) / 16) % 2 == 0) &&
                         (long long)((M + 127) / 128) >= 2LL * sm_count &&
                         (tile == Tile::W96 || tile == Tile::W128 || tile == Tile::L || tile == Tile::N);
  if (narrow_v2 || (!ak && !bk && !lower && !scale && !cin && splits <= 1 && N >= 128 && tile == Tile::L)) {
    Dgemm2Params q{};
    q.M = M;
    q.N = N;
    q.K = K;
    q.A = A;
    q.lda = lda;
    q.B = B;
    q.ldb = ldb;
    q.C = C;
    q.ldc = ldc;
    q.alpha = alpha;
    q.beta = beta;
    q.tri_b = tri_b ? 1 : 0;
    q.colmap = colmap;
    q.n_dev = n_dev;
    // a device-bounded N (the selection's L block) takes 96-wide column tiles:
    // the CTAs past the live columns exit at once
    if (n_dev && narrow_v2 && va && vb) return launch2<G2N128<2>>(st, q);
    if (N > 96 && N <= 128 && narrow_v2 && va && vb) return dispatch2_odd<2>(st, q);
    return (va && vb) ? dispatch2<2>(st, q, false) : dispatch2<1>(st, q, false);
  }
  cudaError_t e;
  if (tile == Tile::T) {
    const int q = (N + 15) / 16;
    if (!bk && va && vb && !cin) {  // (the gathered beta term stays on v1)
      Dgemm2Params t{};
      t.M = M;
      t.N = N;
      t.K = K;
      t.A = A;
      t.lda = lda;
      t.B = B;
      t.ldb = ldb;
      t.C = C;
      t.ldc = ldc;
      t.alpha = alpha;
      t.beta = beta;
      t.tri_b = tri_b ? 1 : 0;
      t.colmap = colmap;
      t.n_dev = n_dev;
      return dispatch2_odd<2>(st, t);
    }
    return bk ? launch_tall<true>(st, p, q) : launch_tall<false>(st, p, q);
  }
  if (!ak && !bk) e = launch_layout<false, false>(st, p, tile, va, vb, splits);
  else if (!ak && bk) e = launch_layout<false, true>(st, p, tile, va, vb, splits);
  else if (ak && !bk) e = launch_layout<true, false>(st, p, tile, va, vb, splits);
  else e = launch_layout<true, true>(st, p, tile, va, vb, splits);
  if (e != cudaSuccess || splits <= 1) return e;
  splitk_reduce_kernel<<<1184, 256, 0, st>>>(work, splits, (long long)M * N, M, N, C, ldc, beta,
                                             lower ? 1 : 0, 64); count_launches(1);
  return cudaGetLastError();
}

// The selection's L block with the residual downdate fused in the epilogue:
// C = A B^T (M x N, N <= 128 in one column tile whose warps span all N
// columns) and d[m] -= sum_n C(m, n)^2 for rows with pos[m] >= kend.
// Returns cudaErrorNotSupported when the shape / alignment does not fit (the
// caller then runs the GEMM and the downdate kernel separately).
template <int Q, int V>
using G2D = Gemm2Cfg<64, 16 * Q, 16, 16 * Q, 3, V, false, 16, (Q <= 5 ? 3 : 2)>;

cudaError_t dgemm_tall_downdate(cudaStream_t st, int M, int N, int K, const double* A, long long lda,
                                const double* B, long long ldb, double* C, long long ldc, double* d,
                                const int* pos, int kend) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  const bool vec = aligned16(A) && aligned16(B) && aligned16(C) && lda % 2 == 0 && ldb % 2 == 0 && ldc % 2 == 0;
  if (N > 128 || N < 17 || !vec) return cudaErrorNotSupported;
  Dgemm2Params q{};
  q.M = M, q.N = N, q.K = K, q.A = A, q.lda = lda, q.B = B, q.ldb = ldb, q.C = C, q.ldc = ldc;
  q.alpha = 1.0, q.beta = 0.0, q.dd = d, q.dpos = pos, q.dkend = kend;
  switch ((N + 15) / 16) {
    case 2: return launch2<G2D<2, 2>>(st, q);
    case 3: return launch2<G2D<3, 2>>(st, q);
    case 4: return launch2<G2D<4, 2>>(st, q);
    case 5: return launch2<G2D<5, 2>>(st, q);
    case 6: return launch2<G2D<6, 2>>(st, q);
    case 7: return launch2<G2D<7, 2>>(st, q);
    default: return launch2<G2D<8, 2>>(st, q);
  }
}

cudaError_t hadamard_gemm(cudaStream_t st, int M, int N, const double* a1, long long lda1,
                          const double* b1, long long ldb1, int k1, const double* a2,
                          long long lda2, const double* b2, long long ldb2, int k2, double* C,
                          long long ldc, double alpha, double beta) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  if (tma_gemm_enabled() && (hadamard_tma_enabled() || (tma_tall_enabled() && N > 32 && N <= 96)) &&
      (long long)((M + 63) / 64) >= 2 * 148) {
    const cudaError_t e = hadamard_tma(st, M, N, a1, lda1, b1, ldb1, k1, a2, lda2, b2, ldb2, k2, C, ldc, alpha, beta);
    if (e != cudaErrorNotSupported) return e;
    cudaGetLastError();
  }
  HadamardParams p{M, N, k1, k2, a1, b1, a2, b2, lda1, ldb1, lda2, ldb2, C, ldc, alpha, beta};
  const bool vec = aligned16(a1) && aligned16(b1) && aligned16(a2) && aligned16(b2) &&
             lda1 % 2 == 0 && ldb1 % 2 == 0 && lda2 % 2 == 0 && ldb2 % 2 == 0 &&
             (M % 2 == 0 || (lda1 > M && lda2 > M)) && (N % 2 == 0 || (ldb1 > N && ldb2 > N));
  auto go = [&](auto cfg) -> cudaError_t {
    using Cfg = decltype(cfg);
    dim3 grid((N + Cfg::BN - 1) / Cfg::BN, (M + Cfg::BM - 1) / Cfg::BM);
    auto kern = hadamard_kernel<Cfg>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES);
    if (e != cudaSuccess) return e;
    kern<<<grid, Cfg::THREADS, Cfg::SMEM_BYTES, st>>>(p); count_launches(1);
    return cudaGetLastError();
  };
  if (N <= 128 && vec && N > 32 && tall_family_enabled() && had_tall_v2_enabled() && (N <= 112 || had128_park()) &&
      (long long)((M + 63) / 64) >= 2LL * 148) {
    // paired-fragment engine, one column tile of width 16 Q, 4 warps of 16 x 16 Q; the first
    // product parks in shared memory (one register accumulator set)
    Dgemm2Params q{};
    q.M = M, q.N = N, q.K = k1, q.K2 = k2;
    q.A = a1, q.lda = lda1, q.B = b1, q.ldb = ldb1, q.A2 = a2, q.lda2 = lda2, q.B2 = b2, q.ldb2 = ldb2;
    q.C = C, q.ldc = ldc, q.alpha = alpha, q.beta = beta;
    switch ((N + 15) / 16) {
      case 3: return launch2<H2T<3>>(st, q);
      case 4: return launch2<H2T<4>>(st, q);
      case 5: return had_wide() ? launch2<H2TW<5>>(st, q) : launch2<H2T<5>>(st, q);
      case 6: return had_wide() ? launch2<H2TW<6>>(st, q) : launch2<H2T<6>>(st, q);
      case 7: return had_wide() ? launch2<H2TW<7>>(st, q) : launch2<H2T<7>>(st, q);
      default: return launch2<H2T8>(st, q);
    }
  }
  // widths 113-127: the general paired-fragment Hadamard below (two 64-wide column tiles)
  const bool v2_wide = vec && N > 112 && had_tall_v2_enabled() && !had128_park();
  if (!v2_wide && N < 128 && vec && N > 32 && tall_family_enabled() && (long long)((M + 127) / 128) >= 2LL * 148) {
    switch ((N + 15) / 16) {
      case 3: return go(CfgHT<3>{});
      case 4: return go(CfgHT<4>{});
      case 5: return go(CfgHT<5>{});
      case 6: return go(CfgHT<6>{});
      case 7: return go(CfgHT<7>{});
      default: return go(CfgHT<8>{});
    }
  }
  if (M <= 256 && N <= 256) {
    // a candidate block's Schur block (s x s): 32 x 32 tiles for parallelism
    return vec ? go(GemmCfg<32, 32, 16, 16, 3, false, false, 2, 2>{}) : go(GemmCfg<32, 32, 16, 16, 3, false, false, 1, 1>{});
  }
  if (N < 128 && !v2_wide) {
    if (prefer_narrow(N)) return vec ? go(CfgH32<2>{}) : go(CfgH32<1>{});
    return vec ? go(CfgH<2>{}) : go(CfgH<1>{});
  }
  Dgemm2Params q{};
  q.M = M;
  q.N = N;
  q.K = k1;
  q.K2 = k2;
  q.A = a1;
  q.lda = lda1;
  q.B = b1;
  q.ldb = ldb1;
  q.A2 = a2;
  q.lda2 = lda2;
  q.B2 = b2;
  q.ldb2 = ldb2;
  q.C = C;
  q.ldc = ldc;
  q.alpha = alpha;
  q.beta = beta;
  return vec ? dispatch2<2>(st, q, true) : dispatch2<1>(st, q, true);
}

cudaError_t mirror_lower(cudaStream_t st, double* a, int n, long long lda, bool average) {
  if (n <= 1) return cudaSuccess;
  mirror_lower_kernel<<<592, 256, 0, st>>>(a, n, lda, average ? 1 : 0); count_launches(1);
  return cudaGetLastError();
}

cudaError_t gather_rows(cudaStream_t st, const double* src, long long lds, int cols, const int* rows,
                        int n_rows, double* dst, long long ldd) {
  if (n_rows <= 0 || cols <= 0) return cudaSuccess;
  gather_rows_kernel<<<592, 256, 0, st>>>(src, lds, cols, rows, n_rows, dst, ldd); count_launches(1);
  return cudaGetLastError();
}

}  // namespace lrgw_dev
