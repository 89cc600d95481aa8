// gemm2.cuh — second-generation FP64 DMMA GEMM mainloop for MN-contiguous
// operands (C = alpha A B^T [o (A2 B2^T)] + beta C, A: M x K and B: N x K both
// column-major with M / N contiguous).
//
// Two changes against gemm.cuh's engine, both aimed at the shared-memory /
// issue limits ncu showed (tensor pipe 65-84%):
//  * fragment pairing: within every 16-row group, 8x8 MMA tile 2j takes rows
//    2g and tile 2j+1 rows 2g+1 (g = lane / 4), so a thread's two A (or B)
//    fragments of a k-step are adjacent in the [k][m] tile -> one LDS.128
//    instead of two LDS.64 (conflict-free with a pitch of BM + 4 doubles), and
//    the epilogue stores adjacent row pairs as double2 (coalesced 128-byte
//    segments);
//  * bigger warp tiles (up to 64x32: 32 DMMA per 6 LDS.128 per k4 step).
// Optional fused epilogues: Hadamard of two K phases (the ISDF Gram pair),
// column scatter (colmap), device-side N bound (n_dev), and a triangular
// B (tri_b: B(n, k) = 0 for k < n) that starts K at the tile's n0.
#pragma once

#include "common.cuh"

namespace lrgw_dev {

struct Dgemm2Params {
  int M, N, K, K2;  // K2 > 0: second (Hadamard) phase with A2, B2
  const double* A;
  long long lda;
  const double* B;
  long long ldb;
  const double* A2;
  long long lda2;
  const double* B2;
  long long ldb2;
  double* C;
  long long ldc;
  double alpha, beta;
  int tri_b;
  const int* colmap;
  const int* n_dev;
  // fused residual downdate of the selection (one warp column per CTA only):
  // dd[m] -= sum_n C(m, n)^2 for rows with dpos[m] >= dkend
  double* dd;
  const int* dpos;
  int dkend;
};

template <int BM_, int BN_, int WM_, int WN_, int STAGES_, int VEC_, bool HAD_, int BK_ = 16, int MINB_ = 1,
          bool SKIP_ = false, bool PARK_ = false>
struct Gemm2Cfg {
  static constexpr int BM = BM_, BN = BN_, BK = BK_, WM = WM_, WN = WN_, STAGES = STAGES_, VEC = VEC_;
  static constexpr int MINB = MINB_;  // resident CTAs per SM the register budget is sized for
  static constexpr bool SKIP = SKIP_;  // warps wholly past a device-bounded N skip their MMAs
  static constexpr bool HAD = HAD_;
  // PARK: the first Hadamard product waits in shared memory (thread-private
  // slots) instead of a second register accumulator set — wide warp tiles
  // without spills.
  static constexpr bool PARK = HAD_ && PARK_;
  static constexpr int WARPS_M = BM / WM, WARPS_N = BN / WN;
  static constexpr int THREADS = 32 * WARPS_M * WARPS_N;
  static constexpr int FM = WM / 8, FN = WN / 8;
  static constexpr int PA = BM + 4, PB = BN + 4;  // doubles; == 4 (mod 16): conflict-free LDS.128
  static constexpr int STAGE_ELEMS = BK * (PA + PB);
  static constexpr int PARK_ELEMS = PARK ? FM * FN * 2 * THREADS : 0;
  static constexpr int SMEM_BYTES = (STAGES * STAGE_ELEMS + PARK_ELEMS) * 8;
  static_assert(WM % 16 == 0 && WN % 16 == 0, "paired fragments need 16-row groups");
};

// [BK][ROWS + 4] tile of an MN-contiguous operand, 16-byte (VEC 2) or 8-byte chunks.
template <int ROWS, int BK, int PITCH, int VEC, int THREADS>
__device__ __forceinline__ void load_mn_tile(double* s, const double* g, long long ld, int row0, int rows, int k0,
                                             int kend, int tid) {
  constexpr int CHUNKS = ROWS * BK / VEC;
#pragma unroll
  for (int i = 0; i < (CHUNKS + THREADS - 1) / THREADS; ++i) {
    const int c = tid + i * THREADS;
    if (CHUNKS % THREADS != 0 && c >= CHUNKS) break;
    const int k = c / (ROWS / VEC);
    const int r = (c % (ROWS / VEC)) * VEC;
    const int gr = row0 + r, gk = k0 + k;
    const bool ok = gr < rows && gk < kend;
    const double* src = ok ? g + gr + (long long)gk * ld : g;
    if (VEC == 2)
      cp_async16(s + k * PITCH + r, src, ok);
    else
      cp_async8(s + k * PITCH + r, src, ok);
  }
}

template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS, Cfg::MINB) dgemm2_kernel(Dgemm2Params p) {
  extern __shared__ __align__(16) double smem[];
  constexpr int BM = Cfg::BM, BN = Cfg::BN, BK = Cfg::BK, STAGES = Cfg::STAGES;
  constexpr int FM = Cfg::FM, FN = Cfg::FN, PA = Cfg::PA, PB = Cfg::PB;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;  // N tiles fastest (A panel reuse in L2)
  int N = p.N;
  if (p.n_dev) N = min(N, *p.n_dev);
  if (n0 >= N) return;
  const int kb = p.tri_b ? (n0 / BK) * BK : 0;
  const int kt1 = p.K > kb ? (p.K - kb + BK - 1) / BK : 0;
  const int kt2 = Cfg::HAD ? (p.K2 + BK - 1) / BK : 0;
  const int nkt = kt1 + kt2;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp % Cfg::WARPS_M) * Cfg::WM, wn = (warp / Cfg::WARPS_M) * Cfg::WN;
  const int g = lane >> 2, t = lane & 3;
  const bool live = !Cfg::SKIP || n0 + wn < N;

  double acc[FM][FN][2];
  constexpr bool REG1 = Cfg::HAD && !Cfg::PARK;  // first product in registers
  double first[REG1 ? FM : 1][REG1 ? FN : 1][2];
  double* park = smem + STAGES * Cfg::STAGE_ELEMS + tid;  // slot q of this thread: park[q * THREADS]
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  auto issue = [&](int kt) {
    double* sa = smem + (kt % STAGES) * Cfg::STAGE_ELEMS;
    double* sb = sa + BK * PA;
    if (kt < kt1) {
      load_mn_tile<BM, BK, PA, Cfg::VEC, Cfg::THREADS>(sa, p.A, p.lda, m0, p.M, kb + kt * BK, p.K, tid);
      load_mn_tile<BN, BK, PB, Cfg::VEC, Cfg::THREADS>(sb, p.B, p.ldb, n0, N, kb + kt * BK, p.K, tid);
    } else {
      load_mn_tile<BM, BK, PA, Cfg::VEC, Cfg::THREADS>(sa, p.A2, p.lda2, m0, p.M, (kt - kt1) * BK, p.K2, tid);
      load_mn_tile<BN, BK, PB, Cfg::VEC, Cfg::THREADS>(sb, p.B2, p.ldb2, n0, N, (kt - kt1) * BK, p.K2, tid);
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
    if (Cfg::SKIP && !live) continue;
    const double* sa = smem + (kt % STAGES) * Cfg::STAGE_ELEMS;
    const double* sb = sa + BK * PA;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[FM], bf[FN];
#pragma unroll
      for (int j = 0; j < FM / 2; ++j) {
        const double2 v = *reinterpret_cast<const double2*>(sa + (kk + t) * PA + wm + 16 * j + 2 * g);
        af[2 * j] = v.x;
        af[2 * j + 1] = v.y;
      }
#pragma unroll
      for (int j = 0; j < FN / 2; ++j) {
        const double2 v = *reinterpret_cast<const double2*>(sb + (kk + t) * PB + wn + 16 * j + 2 * g);
        bf[2 * j] = v.x;
        bf[2 * j + 1] = v.y;
      }
      dmma_block<FM, FN>(acc, af, bf);
    }
    if (Cfg::HAD && kt == kt1 - 1) {
#pragma unroll
      for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j) {
          if (Cfg::PARK) {
            park[((i * FN + j) * 2 + 0) * Cfg::THREADS] = acc[i][j][0];
            park[((i * FN + j) * 2 + 1) * Cfg::THREADS] = acc[i][j][1];
          } else {
            first[REG1 ? i : 0][REG1 ? j : 0][0] = acc[i][j][0];
            first[REG1 ? i : 0][REG1 ? j : 0][1] = acc[i][j][1];
          }
          acc[i][j][0] = acc[i][j][1] = 0.0;
        }
    }
  }
  cp_async_wait<0>();

  // Epilogue. MMA tile 2j (+1) of a 16-row group holds rows 2g (2g + 1);
  // tile column c of n-tile jn is column 16 (jn / 2) + 2 c + (jn % 2).
#pragma unroll
  for (int j = 0; j < FM / 2; ++j) {
    const int m = m0 + wm + 16 * j + 2 * g;
    double sq0 = 0.0, sq1 = 0.0;  // fused downdate: this thread's share of the rows' squared sums
#pragma unroll
    for (int jn = 0; jn < FN; ++jn)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int n = n0 + wn + 16 * (jn / 2) + 4 * t + 2 * h + (jn % 2);
        if (n >= N) continue;
        double v0 = acc[2 * j][jn][h], v1 = acc[2 * j + 1][jn][h];
        if (Cfg::PARK) {
          v0 *= park[(((2 * j) * FN + jn) * 2 + h) * Cfg::THREADS];
          v1 *= park[(((2 * j + 1) * FN + jn) * 2 + h) * Cfg::THREADS];
        } else if (Cfg::HAD) {
          v0 *= first[REG1 ? 2 * j : 0][REG1 ? jn : 0][h];
          v1 *= first[REG1 ? 2 * j + 1 : 0][REG1 ? jn : 0][h];
        }
        v0 *= p.alpha;
        v1 *= p.alpha;
        sq0 = fma(v0, v0, sq0);
        sq1 = fma(v1, v1, sq1);
        const int nc = p.colmap ? __ldg(p.colmap + n) : n;
        double* c = p.C + m + (long long)nc * p.ldc;
        if (m + 1 < p.M && ((reinterpret_cast<uintptr_t>(c) & 15) == 0)) {
          double2 out = make_double2(v0, v1);
          if (p.beta != 0.0) {
            const double2 old = *reinterpret_cast<const double2*>(c);
            out.x += p.beta * old.x;
            out.y += p.beta * old.y;
          }
          *reinterpret_cast<double2*>(c) = out;
        } else {
          if (m < p.M) c[0] = (p.beta == 0.0) ? v0 : v0 + p.beta * c[0];
          if (m + 1 < p.M) c[1] = (p.beta == 0.0) ? v1 : v1 + p.beta * c[1];
        }
      }
    if (p.dd) {  // the 4 lanes of a row pair (t = 0..3) hold disjoint columns; WARPS_N == 1
      sq0 += __shfl_xor_sync(0xffffffffu, sq0, 1);
      sq1 += __shfl_xor_sync(0xffffffffu, sq1, 1);
      sq0 += __shfl_xor_sync(0xffffffffu, sq0, 2);
      sq1 += __shfl_xor_sync(0xffffffffu, sq1, 2);
      if (t == 0) {
        if (m < p.M && p.dpos[m] >= p.dkend) p.dd[m] -= sq0;
        if (m + 1 < p.M && p.dpos[m + 1] >= p.dkend) p.dd[m + 1] -= sq1;
      }
    }
  }
}

}  // namespace lrgw_dev
