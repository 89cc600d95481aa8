// gemm.cuh — FP64 DMMA GEMM engine for the lrgw hot path (sm_100a).
//
//   C(m,n) = alpha * sum_k A(m,k) * s(k) * B(n,k) + beta * C(m,n)
//
// A is logically M x K and B is N x K; each is stored either MN-contiguous
// (column-major M x K: A[m + k*lda]) or K-contiguous (A[m*lda + k]). That one
// engine covers every dense contraction of the path:
//   fit GEMMs  (Phi Phi_mu^T)       A: MN,  B: MN            (isdf.hpp:132)
//   Theta      (lhs G^-1)           A: MN,  B: K             (isdf.hpp:143)
//   Theta^T V Theta in G-space      A: K,   B: K, s = v(G)   (smw.hpp:61)
//   probe      (Theta^T X, Theta y) skinny variants          (smw.hpp:101)
// The diagonal s(k) is fused into the B-operand load (never materialised).
// Tiles stream global -> shared through a STAGES-deep cp.async ring; warps
// issue DMMA.8x8x4 from padded, bank-conflict-free shared tiles.
#pragma once

#include <type_traits>

#include "common.cuh"

namespace lrgw_dev {

struct DgemmParams {
  int M, N, K;
  const double* A;
  long long lda;
  const double* B;
  long long ldb;
  double* C;
  long long ldc;
  double alpha, beta;
  const double* scale;   // length K, or nullptr
  int lower;             // 1: only tiles with tile_n <= tile_m (BM == BN)
  int k_chunk;           // split-K chunk (multiple of BK) when gridDim.z > 1
  double* partial;       // split-K: raw alpha*acc to partial + z*part_stride (ld = M)
  long long part_stride;
  int tri_b;             // B(n, k) == 0 for k < n (lower-triangular operand): K starts at n0
  const int* colmap;     // output column n is written to column colmap[n] of C
  const int* n_dev;      // if set: N = min(N, *n_dev), read on the device (no host sync)
  const double* Cin;     // if set: the beta term reads Cin[m + cin_map[n] ldcin] instead of C
  long long ldcin;
  const int* cin_map;
  int batch;             // > 1: gridDim.z runs independent products at A + z bsa, B + z bsb, C + z bsc
  long long bsa, bsb, bsc;
};

// Tile loader for one operand. ROWS = BM or BN.
template <int ROWS, int BK, bool KMAJOR, int VEC, int THREADS>
struct TileLoader {
  static constexpr int PITCH = KMAJOR ? (BK + 4) : (ROWS + 4);   // doubles
  static constexpr int ELEMS = KMAJOR ? ROWS * PITCH : BK * PITCH;
  static constexpr int CHUNKS = ROWS * BK / VEC;
  static constexpr int PER_THREAD = (CHUNKS + THREADS - 1) / THREADS;

  // row0: first logical row of the tile; k0: first k; rows/kend: bounds.
  __device__ __forceinline__ static void load(double* s, const double* g, long long ld, int row0,
                                              int rows, int k0, int kend, int tid) {
#pragma unroll
    for (int i = 0; i < PER_THREAD; ++i) {
      const int c = tid + i * THREADS;
      if (CHUNKS % THREADS != 0 && c >= CHUNKS) break;
      int r, k;
      if (KMAJOR) {
        r = c / (BK / VEC);
        k = (c % (BK / VEC)) * VEC;
      } else {
        k = c / (ROWS / VEC);
        r = (c % (ROWS / VEC)) * VEC;
      }
      const int gr = row0 + r, gk = k0 + k;
      const bool ok = (gr < rows) && (gk < kend);
      const double* src = ok ? (KMAJOR ? g + (long long)gr * ld + gk : g + gr + (long long)gk * ld) : g;
      double* dst = KMAJOR ? s + r * PITCH + k : s + k * PITCH + r;
      if (VEC == 2)
        cp_async16(dst, src, ok);
      else
        cp_async8(dst, src, ok);
    }
  }

  // Fragment element [row][kk] of the staged tile.
  __device__ __forceinline__ static double frag(const double* s, int row, int kk) {
    return KMAJOR ? s[row * PITCH + kk] : s[kk * PITCH + row];
  }
};

template <int BM_, int BN_, int WM_, int WN_, int STAGES_, bool AK_, bool BK_MAJ_, int VA_, int VB_, int BK_ = 16,
          int MINB_ = 1>
struct GemmCfg {
  static constexpr int BM = BM_, BN = BN_, BK = BK_, WM = WM_, WN = WN_, STAGES = STAGES_;
  static constexpr int MINB = MINB_;  // resident CTAs per SM the register budget is sized for
  static constexpr bool A_KMAJOR = AK_, B_KMAJOR = BK_MAJ_;
  static constexpr int WARPS_M = BM / WM, WARPS_N = BN / WN;
  static constexpr int THREADS = 32 * WARPS_M * WARPS_N;
  static constexpr int FM = WM / 8, FN = WN / 8;
  using LA = TileLoader<BM, BK, A_KMAJOR, VA_, THREADS>;
  using LB = TileLoader<BN, BK, B_KMAJOR, VB_, THREADS>;
  static constexpr int STAGE_ELEMS = LA::ELEMS + LB::ELEMS + BK;  // + the k-slice of the diagonal scale
  static constexpr int SMEM_BYTES = STAGES * STAGE_ELEMS * 8;
};

template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS, Cfg::MINB) dgemm_kernel(DgemmParams p) {
  extern __shared__ __align__(16) double smem[];
  constexpr int BM = Cfg::BM, BN = Cfg::BN, BK = Cfg::BK, STAGES = Cfg::STAGES;
  constexpr int FM = Cfg::FM, FN = Cfg::FN;
  using LA = typename Cfg::LA;
  using LB = typename Cfg::LB;

  int tm, tn;
  if (p.lower) {
    lower_tile(blockIdx.x, tm, tn);
  } else {
    // N tiles fastest: the CTAs sharing an A row panel run together, so A is
    // read from HBM once (then L2) instead of once per N tile
    tn = blockIdx.x;
    tm = blockIdx.y;
  }
  const int m0 = tm * BM, n0 = tn * BN;
  if (p.n_dev) {
    const int nd = *p.n_dev;
    if (nd < p.N) p.N = nd;
    if (n0 >= p.N) return;
  }
  if (p.batch > 1) {
    p.A += blockIdx.z * p.bsa;
    p.B += blockIdx.z * p.bsb;
    p.C += blockIdx.z * p.bsc;
  }
  const int kb = p.k_chunk > 0 ? blockIdx.z * p.k_chunk : (p.tri_b ? (n0 / BK) * BK : 0);
  const int ke = p.k_chunk > 0 ? min(p.K, kb + p.k_chunk) : p.K;
  const int nkt = ke > kb ? (ke - kb + BK - 1) / BK : 0;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp % Cfg::WARPS_M) * Cfg::WM, wn = (warp / Cfg::WARPS_M) * Cfg::WN;
  const int g = lane >> 2, t = lane & 3;
  const bool live = n0 + wn < p.N;  // warps wholly past the (device-bounded) N skip their MMAs

  double acc[FM][FN][2];
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  auto stageA = [&](int s) { return smem + s * Cfg::STAGE_ELEMS; };
  auto stageB = [&](int s) { return smem + s * Cfg::STAGE_ELEMS + LA::ELEMS; };
  auto stageS = [&](int s) { return smem + s * Cfg::STAGE_ELEMS + LA::ELEMS + LB::ELEMS; };
  // the diagonal scale travels with its k-tile (no global load on the MMA path)
  auto load_scale = [&](int s, int k0) {
    if (p.scale && tid < BK) {
      const int gk = k0 + tid;
      cp_async8(stageS(s) + tid, gk < ke ? p.scale + gk : p.scale, gk < ke);
    }
  };

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nkt) {
      LA::load(stageA(s), p.A, p.lda, m0, p.M, kb + s * BK, ke, tid);
      LB::load(stageB(s), p.B, p.ldb, n0, p.N, kb + s * BK, ke, tid);
      load_scale(s, kb + s * BK);
    }
    cp_async_commit();
  }

  auto mainloop = [&](auto with_mma) {
    for (int kt = 0; kt < nkt; ++kt) {
      cp_async_wait<STAGES - 2>();
      __syncthreads();
      {
        const int nx = kt + STAGES - 1;
        if (nx < nkt) {
          const int s = nx % STAGES;
          LA::load(stageA(s), p.A, p.lda, m0, p.M, kb + nx * BK, ke, tid);
          LB::load(stageB(s), p.B, p.ldb, n0, p.N, kb + nx * BK, ke, tid);
          load_scale(s, kb + nx * BK);
        }
        cp_async_commit();
      }
      if (!decltype(with_mma)::value) continue;
      const double* sa = stageA(kt % STAGES);
      const double* sb = stageB(kt % STAGES);
      const double* ss = stageS(kt % STAGES);
#pragma unroll
      for (int kk = 0; kk < BK; kk += 4) {
        double af[FM], bf[FN];
#pragma unroll
        for (int i = 0; i < FM; ++i) af[i] = LA::frag(sa, wm + i * 8 + g, kk + t);
#pragma unroll
        for (int j = 0; j < FN; ++j) bf[j] = LB::frag(sb, wn + j * 8 + g, kk + t);
        if (p.scale) {
          const double sc = ss[kk + t];
#pragma unroll
          for (int j = 0; j < FN; ++j) bf[j] *= sc;
        }
        dmma_block<FM, FN>(acc, af, bf);
      }
    }
  };
  // warps wholly past a device-bounded N only keep the copy / barrier cadence
  if (live)
    mainloop(std::true_type{});
  else
    mainloop(std::false_type{});
  cp_async_wait<0>();

  // Epilogue: c0 = C[m = g][n = 2t], c1 = C[g][2t+1] per 8x8 fragment.
  if (p.partial) {
    double* out = p.partial + (long long)blockIdx.z * p.part_stride;
#pragma unroll
    for (int i = 0; i < FM; ++i)
#pragma unroll
      for (int j = 0; j < FN; ++j) {
        const int m = m0 + wm + i * 8 + g;
        const int n = n0 + wn + j * 8 + 2 * t;
        if (m < p.M) {
          if (n < p.N) out[m + (long long)n * p.M] = p.alpha * acc[i][j][0];
          if (n + 1 < p.N) out[m + (long long)(n + 1) * p.M] = p.alpha * acc[i][j][1];
        }
      }
    return;
  }
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j) {
      const int m = m0 + wm + i * 8 + g;
      const int n = n0 + wn + j * 8 + 2 * t;
      if (m < p.M) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (n + h < p.N) {
            const int nc = p.colmap ? __ldg(p.colmap + n + h) : n + h;
            double* c = p.C + m + (long long)nc * p.ldc;
            const double v = p.alpha * acc[i][j][h];
            if (p.beta == 0.0)
              *c = v;
            else
              *c = v + p.beta * (p.Cin ? p.Cin[m + (long long)__ldg(p.cin_map + n + h) * p.ldcin] : *c);
          }
        }
      }
    }
}

// C = alpha * (A1 B1^T) o (A2 B2^T) + beta * C — the ISDF fit GEMM pair with
// the Hadamard product fused into the epilogue (isdf.hpp:132): the two
// N_r x N_mu Gram factors never reach HBM. Both pairs MN-contiguous. The
// k-tile stream runs over K1 then K2; at the switch the first product is
// parked in registers.
struct HadamardParams {
  int M, N, K1, K2;
  const double *A1, *B1, *A2, *B2;
  long long lda1, ldb1, lda2, ldb2;
  double* C;
  long long ldc;
  double alpha, beta;
};

template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS) hadamard_kernel(HadamardParams p) {
  extern __shared__ __align__(16) double smem[];
  constexpr int BM = Cfg::BM, BN = Cfg::BN, BK = Cfg::BK, STAGES = Cfg::STAGES;
  constexpr int FM = Cfg::FM, FN = Cfg::FN;
  using LA = typename Cfg::LA;
  using LB = typename Cfg::LB;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;  // N tiles fastest (A panel reuse in L2)
  const int kt1 = (p.K1 + BK - 1) / BK, kt2 = (p.K2 + BK - 1) / BK;
  const int nkt = kt1 + kt2;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp % Cfg::WARPS_M) * Cfg::WM, wn = (warp / Cfg::WARPS_M) * Cfg::WN;
  const int g = lane >> 2, t = lane & 3;

  double acc[FM][FN][2], first[FM][FN][2];
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = first[i][j][0] = first[i][j][1] = 0.0;

  auto issue = [&](int kt) {
    double* sa = smem + (kt % STAGES) * Cfg::STAGE_ELEMS;
    double* sb = sa + LA::ELEMS;
    // pick the phase's operands first so one load sequence serves both phases
    const double *a = p.A1, *b = p.B1;
    long long lda = p.lda1, ldb = p.ldb1;
    int k0 = kt * BK, kend = p.K1;
    if (kt >= kt1) a = p.A2, b = p.B2, lda = p.lda2, ldb = p.ldb2, k0 = (kt - kt1) * BK, kend = p.K2;
    LA::load(sa, a, lda, m0, p.M, k0, kend, tid);
    LB::load(sb, b, ldb, n0, p.N, k0, kend, tid);
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
    const double* sb = sa + LA::ELEMS;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[FM], bf[FN];
#pragma unroll
      for (int i = 0; i < FM; ++i) af[i] = LA::frag(sa, wm + i * 8 + g, kk + t);
#pragma unroll
      for (int j = 0; j < FN; ++j) bf[j] = LB::frag(sb, wn + j * 8 + g, kk + t);
      dmma_block<FM, FN>(acc, af, bf);
    }
    if (kt == kt1 - 1) {
#pragma unroll
      for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j) {
          first[i][j][0] = acc[i][j][0];
          first[i][j][1] = acc[i][j][1];
          acc[i][j][0] = acc[i][j][1] = 0.0;
        }
    }
  }
  cp_async_wait<0>();
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j) {
      const int m = m0 + wm + i * 8 + g;
      const int n = n0 + wn + j * 8 + 2 * t;
      if (m < p.M) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (n + h < p.N) {
            double* c = p.C + m + (long long)(n + h) * p.ldc;
            const double v = p.alpha * (first[i][j][h] * acc[i][j][h]);
            *c = (p.beta == 0.0) ? v : v + p.beta * (*c);
          }
        }
      }
    }
}

}  // namespace lrgw_dev
