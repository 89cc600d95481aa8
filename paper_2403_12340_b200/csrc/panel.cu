// panel.cu — K1 step 4 in one launch: the selection's block panel.
//
// For a candidate block that accepted nb pivots (grid rows R, pivots before
// the block k), the block's columns of the pivoted-Cholesky factor are
//   W     = (Phi_a Phi_a[R]^T) o (Phi_b Phi_b[R]^T) - L[:, :k] L[R, :k]^T   (n_r x nb)
//   L_blk = W X^T,   X = L_sel^-1 (nb x nb, from the greedy)
//   d    -= rowsum(L_blk^2)   (rows not yet selected)
// (the reference's QRCP, linalg.hpp:26-111, restated as matrix-free pivoted
// Cholesky on the Hadamard Gram — select.cu). Three GEMM launches (Hadamard
// pair, L-pass, L block with the downdate epilogue) and the n_r x nb W
// round trip through HBM become one kernel with four K phases feeding one
// register accumulator:
//   phase 1  Phi_a . Phi_a[R]^T          -> parked in shared memory
//   phase 2  Phi_b . Phi_b[R]^T          -> acc = park o acc
//   phase 3  acc -= L[:, :k] L[R, :k]^T  (negated A fragments)
//   phase 4  W parked; acc = W X^T with W's fragments read straight from the
//            park slots: the DMMA accumulator layout is reused as the A
//            operand by permuting k — thread t of a 4-lane group holds
//            columns c0 + 4t + s of W (s = 2h + (jn & 1)), so X^T's 16-row
//            tiles are staged with row 4 (k % 4) + k / 4 and the ordinary
//            fragment reads pick up the matching k.
// CTAs are 64 x 16Q (4 warps of 16 rows x all columns), so every row's sum
// of squares is complete inside one warp and the downdate needs no atomics.
#include <algorithm>
#include <cstdlib>

#include "gemm2.cuh"
#include "kernels.h"

namespace lrgw_dev {

namespace {

struct PanelParams {
  int M, N;        // rows (n_r), accepted pivots nb
  int K1, K2, K3;  // n1, n2, k
  const double* A1;
  long long lda1;
  const double* B1;
  long long ldb1;
  const double* A2;
  long long lda2;
  const double* B2;
  long long ldb2;
  const double* A3;
  long long lda3;
  const double* B3;
  long long ldb3;
  const double* X;
  long long ldx;
  double* C;
  long long ldc;
  double* d;
  const int* pos;
  int kend;
  const int* kdev;  // device-driven loop: k, N from the device (see select_panel)
  const int* ndev;
};

template <int Q, int STAGES_, int MINB_>
struct PanelCfg {
  static constexpr int BM = 64, BN = 16 * Q, BK = 16, WM = 16, WN = BN, STAGES = STAGES_, MINB = MINB_;
  static constexpr int THREADS = 32 * (BM / WM);
  static constexpr int FM = WM / 8, FN = WN / 8;
  static constexpr int PA = BM + 4, PB = BN + 4;
  static constexpr int STAGE_ELEMS = BK * (PA + PB);
  static constexpr int PARK_ELEMS = FM * FN * 2 * THREADS;
  static constexpr int SMEM_BYTES = (STAGES * STAGE_ELEMS + PARK_ELEMS) * 8;
};

// X^T tile for phase 4: global k-row c (0..15) of the tile lands on smem row
// 4 (c % 4) + c / 4, the row the fragment read of sub-step s = c % 4 by lane
// group t = c / 4 addresses.
template <int ROWS, int PITCH, int THREADS>
__device__ __forceinline__ void load_x_tile(double* s, const double* g, long long ld, int rows, int k0, int kend,
                                            int tid) {
  constexpr int CHUNKS = ROWS * 16 / 2;
#pragma unroll
  for (int i = 0; i < (CHUNKS + THREADS - 1) / THREADS; ++i) {
    const int c = tid + i * THREADS;
    if (CHUNKS % THREADS != 0 && c >= CHUNKS) break;
    const int k = c / (ROWS / 2);
    const int r = (c % (ROWS / 2)) * 2;
    const int gk = k0 + k;
    const bool ok = r < rows && gk < kend;
    const double* src = ok ? g + r + (long long)gk * ld : g;
    cp_async16(s + (4 * (k & 3) + (k >> 2)) * PITCH + r, src, ok);
  }
}

template <class Cfg>
__device__ __forceinline__ void panel_body(const PanelParams& p, double* smem, const int N, const int K3,
                                           const int kend, double* cout) {
  constexpr int BM = Cfg::BM, BN = Cfg::BN, BK = Cfg::BK, STAGES = Cfg::STAGES;
  constexpr int FM = Cfg::FM, FN = Cfg::FN, PA = Cfg::PA, PB = Cfg::PB, T = Cfg::THREADS;
  const int m0 = blockIdx.x * BM;
  const int kt1 = (p.K1 + BK - 1) / BK, kt2 = (p.K2 + BK - 1) / BK, kt3 = (K3 + BK - 1) / BK;
  const int e1 = kt1, e2 = e1 + kt2, e3 = e2 + kt3, nkt = e3 + (N + BK - 1) / BK;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp * Cfg::WM;
  const int g = lane >> 2, t = lane & 3;
  double* park = smem + STAGES * Cfg::STAGE_ELEMS + tid;  // slot q of this thread: park[q * T]

  double acc[FM][FN][2];
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  auto issue = [&](int kt) {
    double* sa = smem + (kt % STAGES) * Cfg::STAGE_ELEMS;
    double* sb = sa + BK * PA;
    if (kt < e1) {
      load_mn_tile<BM, BK, PA, 2, T>(sa, p.A1, p.lda1, m0, p.M, kt * BK, p.K1, tid);
      load_mn_tile<BN, BK, PB, 2, T>(sb, p.B1, p.ldb1, 0, N, kt * BK, p.K1, tid);
    } else if (kt < e2) {
      load_mn_tile<BM, BK, PA, 2, T>(sa, p.A2, p.lda2, m0, p.M, (kt - e1) * BK, p.K2, tid);
      load_mn_tile<BN, BK, PB, 2, T>(sb, p.B2, p.ldb2, 0, N, (kt - e1) * BK, p.K2, tid);
    } else if (kt < e3) {
      load_mn_tile<BM, BK, PA, 2, T>(sa, p.A3, p.lda3, m0, p.M, (kt - e2) * BK, K3, tid);
      load_mn_tile<BN, BK, PB, 2, T>(sb, p.B3, p.ldb3, 0, N, (kt - e2) * BK, K3, tid);
    } else {
      load_x_tile<BN, PB, T>(sb, p.X, p.ldx, N, (kt - e3) * BK, N, tid);
    }
  };
  // mask: W's columns >= N (an odd N's straddling pair reads one gathered row
  // past the block) are zeroed before they become phase 4's A operand
  auto park_acc = [&](bool mask) {
#pragma unroll
    for (int i = 0; i < FM; ++i)
#pragma unroll
      for (int j = 0; j < FN; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const bool dead = mask && 16 * (j / 2) + 4 * t + 2 * h + (j % 2) >= N;
          park[((i * FN + j) * 2 + h) * T] = dead ? 0.0 : acc[i][j][h];
          acc[i][j][h] = 0.0;
        }
  };

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nkt) issue(s);
    cp_async_commit();
  }
  for (int kt = 0; kt < nkt; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    if (kt + STAGES - 1 < nkt) issue(kt + STAGES - 1);
    cp_async_commit();
    const double* sa = smem + (kt % STAGES) * Cfg::STAGE_ELEMS;
    const double* sb = sa + BK * PA;
    if (kt < e3) {
      const bool neg = kt >= e2;
#pragma unroll
      for (int kk = 0; kk < BK; kk += 4) {
        double af[FM], bf[FN];
#pragma unroll
        for (int j = 0; j < FM / 2; ++j) {
          const double2 v = *reinterpret_cast<const double2*>(sa + (kk + t) * PA + wm + 16 * j + 2 * g);
          af[2 * j] = neg ? -v.x : v.x;
          af[2 * j + 1] = neg ? -v.y : v.y;
        }
#pragma unroll
        for (int j = 0; j < FN / 2; ++j) {
          const double2 v = *reinterpret_cast<const double2*>(sb + (kk + t) * PB + 16 * j + 2 * g);
          bf[2 * j] = v.x;
          bf[2 * j + 1] = v.y;
        }
        dmma_block<FM, FN>(acc, af, bf);
      }
    } else {
      // phase 4: W's columns 16 q .. 16 q + 15 as the k range (q = kt - e3)
      const int q = kt - e3;
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        double af[FM], bf[FN];
        const int jn = 2 * q + (s & 1), h = s >> 1;
#pragma unroll
        for (int i = 0; i < FM; ++i) af[i] = park[((i * FN + jn) * 2 + h) * T];
#pragma unroll
        for (int j = 0; j < FN / 2; ++j) {
          const double2 v = *reinterpret_cast<const double2*>(sb + (4 * s + t) * PB + 16 * j + 2 * g);
          bf[2 * j] = v.x;
          bf[2 * j + 1] = v.y;
        }
        dmma_block<FM, FN>(acc, af, bf);
      }
    }
    if (kt == e1 - 1) park_acc(false);
    if (kt == e2 - 1) {
#pragma unroll
      for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j) {
          acc[i][j][0] *= park[((i * FN + j) * 2 + 0) * T];
          acc[i][j][1] *= park[((i * FN + j) * 2 + 1) * T];
        }
    }
    if (kt == e3 - 1) park_acc(true);
  }
  cp_async_wait<0>();

  // Epilogue: L_blk rows (paired layout: MMA tile 2j (+1) holds rows 2g (2g + 1)
  // of a 16-row group; n-tile jn column 16 (jn / 2) + 4 t + 2 h + (jn % 2)) and
  // the downdate over the 4 lanes of a row pair.
#pragma unroll
  for (int j = 0; j < FM / 2; ++j) {
    const int m = m0 + wm + 16 * j + 2 * g;
    double sq0 = 0.0, sq1 = 0.0;
#pragma unroll
    for (int jn = 0; jn < FN; ++jn)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int n = 16 * (jn / 2) + 4 * t + 2 * h + (jn % 2);
        if (n >= N) continue;
        const double v0 = acc[2 * j][jn][h], v1 = acc[2 * j + 1][jn][h];
        sq0 = fma(v0, v0, sq0);
        sq1 = fma(v1, v1, sq1);
        double* c = cout + m + (long long)n * p.ldc;
        if (m + 1 < p.M) {
          *reinterpret_cast<double2*>(c) = make_double2(v0, v1);
        } else if (m < p.M) {
          c[0] = v0;
        }
      }
    sq0 += __shfl_xor_sync(0xffffffffu, sq0, 1);
    sq1 += __shfl_xor_sync(0xffffffffu, sq1, 1);
    sq0 += __shfl_xor_sync(0xffffffffu, sq0, 2);
    sq1 += __shfl_xor_sync(0xffffffffu, sq1, 2);
    if (t == 0) {
      if (m < p.M && p.pos[m] >= kend) p.d[m] -= sq0;
      if (m + 1 < p.M && p.pos[m + 1] >= kend) p.d[m + 1] -= sq1;
    }
  }
}

// The tile configuration of width 16 Q.
template <int Q>
struct PanelQ;
template <> struct PanelQ<2> { using C = PanelCfg<2, 3, 2>; };
template <> struct PanelQ<3> { using C = PanelCfg<3, 3, 2>; };
template <> struct PanelQ<4> { using C = PanelCfg<4, 3, 2>; };
template <> struct PanelQ<5> { using C = PanelCfg<5, 2, 2>; };
template <> struct PanelQ<6> { using C = PanelCfg<6, 2, 2>; };
template <> struct PanelQ<7> { using C = PanelCfg<7, 2, 2>; };
template <> struct PanelQ<8> { using C = PanelCfg<8, 3, 1>; };

// Width 16 ceil(N / 16) for a block whose N is known on the device only
// (QMAX from the accept cap), else width 16 QMAX.
template <int Q, bool DISPATCH>
__device__ __forceinline__ void panel_pick(const PanelParams& p, double* smem, int N, int K3, int kend,
                                           double* cout) {
  if constexpr (DISPATCH && Q > 2) {
    if (N <= 16 * (Q - 1)) {
      panel_pick<Q - 1, true>(p, smem, N, K3, kend, cout);
      return;
    }
  }
  panel_body<typename PanelQ<Q>::C>(p, smem, N, K3, kend, cout);
}

template <int Q>
constexpr int panel_smem_max() {
  if constexpr (Q <= 2)
    return PanelQ<2>::C::SMEM_BYTES;
  else
    return PanelQ<Q>::C::SMEM_BYTES > panel_smem_max<Q - 1>() ? PanelQ<Q>::C::SMEM_BYTES : panel_smem_max<Q - 1>();
}

// resident CTAs per SM the register budget is sized for (PanelQ<Q>::C::MINB)
template <int Q>
constexpr int panel_minb() {
  return Q >= 8 ? 1 : 2;
}

template <int Q, bool DISPATCH>
__global__ void __launch_bounds__(128, panel_minb<Q>()) panel_kernel(PanelParams p) {
  static_assert(PanelQ<Q>::C::MINB == panel_minb<Q>(), "register budget");
  extern __shared__ __align__(16) double smem[];
  int N = p.N, K3 = p.K3, kend = p.kend;
  double* cout = p.C;
  if (p.kdev) {
    K3 = *p.kdev;
    N = min(N, *p.ndev);
    kend = K3 + N;
    cout += (long long)K3 * p.ldc;
  }
  if (N <= 0) return;
  panel_pick<Q, DISPATCH>(p, smem, N, K3, kend, cout);
}

template <int Q>
cudaError_t launch_panel(cudaStream_t st, const PanelParams& p, bool dispatch) {
  const int grid = (p.M + 63) / 64;
  if (grid == 0) return cudaSuccess;
  const int smem = dispatch ? panel_smem_max<Q>() : PanelQ<Q>::C::SMEM_BYTES;
  auto kern = dispatch ? panel_kernel<Q, true> : panel_kernel<Q, false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  kern<<<grid, 128, smem, st>>>(p);
  count_launches(1);
  return cudaGetLastError();
}

bool aligned16p(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace

// LRGW_PANEL=0 / 1 forces the choice. By default the fused panel runs where
// it beats the three launches (measured, profiles/r02/): on the TMA engine
// (panel4.cu) at every Hadamard depth — Si64 select 10.11 -> 9.40 ms, C60
// 41.9 -> 35.2 ms, Si216 229.5 -> 220 ms, Si512 2739 -> 2708 ms (the 96-wide
// body loads its B halves one at a time to stay within the 2-CTA register
// budget); the cp.async panel (panel.cu) only up to a depth of 512.
bool select_panel_enabled(int n1, int n2) {
  static const int v = getenv("LRGW_PANEL") ? atoi(getenv("LRGW_PANEL")) : -1;
  if (v >= 0) return v != 0;
  return select_panel_tma_enabled() || n1 + n2 <= 512;
}

cudaError_t select_panel(cudaStream_t st, int M, int N, const double* a1, long long lda1, const double* b1,
                         long long ldb1, int k1, const double* a2, long long lda2, const double* b2, long long ldb2,
                         int k2, const double* l, long long ldl, const double* lrow, long long ldlr, int k,
                         const double* x, long long ldx, double* c, long long ldc, double* d, const int* pos,
                         int kend, const int* k_dev, const int* n_dev) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  if (N < 17 || N > 128 || k1 < 1 || k2 < 1 || k < 0) return cudaErrorNotSupported;
  const bool vec = aligned16p(a1) && aligned16p(b1) && aligned16p(a2) && aligned16p(b2) && aligned16p(x) &&
                   aligned16p(c) && (k == 0 || (aligned16p(l) && aligned16p(lrow))) && lda1 % 2 == 0 &&
                   ldb1 % 2 == 0 && lda2 % 2 == 0 && ldb2 % 2 == 0 && ldx % 2 == 0 && ldc % 2 == 0 &&
                   ((k == 0 && !k_dev) || (ldl % 2 == 0 && ldlr % 2 == 0)) &&
                   (M % 2 == 0 || (lda1 > M && lda2 > M && ldl > M));
  if (!vec) return cudaErrorNotSupported;
  PanelParams p{};
  p.M = M, p.N = N, p.K1 = k1, p.K2 = k2, p.K3 = k;
  p.A1 = a1, p.lda1 = lda1, p.B1 = b1, p.ldb1 = ldb1;
  p.A2 = a2, p.lda2 = lda2, p.B2 = b2, p.ldb2 = ldb2;
  p.A3 = l, p.lda3 = ldl, p.B3 = lrow, p.ldb3 = ldlr;
  p.X = x, p.ldx = ldx, p.C = c, p.ldc = ldc, p.d = d, p.pos = pos, p.kend = kend;
  p.kdev = k_dev, p.ndev = n_dev;
  const bool dispatch = k_dev != nullptr;  // the block's width is known on the device only
  switch ((N + 15) / 16) {
    case 2: return launch_panel<2>(st, p, dispatch);
    case 3: return launch_panel<3>(st, p, dispatch);
    case 4: return launch_panel<4>(st, p, dispatch);
    case 5: return launch_panel<5>(st, p, dispatch);
    case 6: return launch_panel<6>(st, p, dispatch);
    case 7: return launch_panel<7>(st, p, dispatch);
    default: return launch_panel<8>(st, p, dispatch);
  }
}

}  // namespace lrgw_dev
