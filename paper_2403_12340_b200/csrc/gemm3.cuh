// gemm3.cuh — third-generation FP64 DMMA GEMM mainloop: paired fragments for
// either operand layout.
//
//   C = alpha * sum_k A(m,k) s(k) B(n,k) + beta * C      (DgemmParams, gemm.cuh)
//
// Every thread loads two k4 steps' fragments at once: the k order inside a
// tile is permuted so that lane t's k indices of steps 2p and 2p+1 are the
// adjacent pair 8p + 2t, 8p + 2t + 1 (a sum is order-free). Then
//  * a K-contiguous operand (smem [row][BK + 8]) gives both steps' values of
//    a fragment with one LDS.128;
//  * an MN-contiguous operand (smem [k][rows + 2]) pairs rows 2g, 2g + 1 of a
//    16-row group (MMA tiles 2j, 2j + 1) with one LDS.128 per step;
// both pitches keep each quarter-warp's LDS.128 on distinct banks. The
// diagonal scale s(k) travels with its k-tile (double2 per pair). Supports
// lower-triangle tiles, split-K partials, triangular-B K skipping, output
// column scatter, a device-side N bound and a gathered beta term, so it can
// replace the v1 engine (gemm.cuh) for every contraction of the path.
// CTAs of 4 warps, several resident per SM (the library DGEMM's occupancy).
#pragma once

#include "common.cuh"
#include "gemm.cuh"

namespace lrgw_dev {

template <int BM_, int BN_, int WM_, int WN_, int STAGES_, bool AK_, bool BKM_, int VEC_, int BK_, int MINB_>
struct Gemm3Cfg {
  static constexpr int BM = BM_, BN = BN_, BK = BK_, WM = WM_, WN = WN_, STAGES = STAGES_, VEC = VEC_;
  static constexpr int MINB = MINB_;
  static constexpr bool AK = AK_, BKM = BKM_;  // K-contiguous operands
  static constexpr int WARPS_M = BM / WM, WARPS_N = BN / WN;
  static constexpr int THREADS = 32 * WARPS_M * WARPS_N;
  static constexpr int FM = WM / 8, FN = WN / 8;
  static constexpr int PA = AK ? BK + 8 : BM + 2;  // doubles
  static constexpr int PB = BKM ? BK + 8 : BN + 2;
  static constexpr int EA = AK ? BM * PA : BK * PA;
  static constexpr int EB = BKM ? BN * PB : BK * PB;
  static constexpr int STAGE_ELEMS = EA + EB + BK;  // + the k-slice of the diagonal scale
  static constexpr int SMEM_BYTES = STAGES * STAGE_ELEMS * 8;
  static_assert(BK % 8 == 0, "k pairs");
  static_assert(AK || WM % 16 == 0, "row pairs");
  static_assert(BKM || WN % 16 == 0, "column pairs");
};

// [rows][BK + 8] tile of a K-contiguous operand (chunks of VEC consecutive k).
template <int ROWS, int BK, int PITCH, int VEC, int THREADS>
__device__ __forceinline__ void load_k_tile(double* s, const double* g, long long ld, int row0, int rows, int k0,
                                            int kend, int tid) {
  constexpr int CHUNKS = ROWS * BK / VEC;
#pragma unroll
  for (int i = 0; i < (CHUNKS + THREADS - 1) / THREADS; ++i) {
    const int c = tid + i * THREADS;
    if (CHUNKS % THREADS != 0 && c >= CHUNKS) break;
    const int r = c / (BK / VEC);
    const int k = (c % (BK / VEC)) * VEC;
    const int gr = row0 + r, gk = k0 + k;
    const bool ok = gr < rows && gk < kend;
    const double* src = ok ? g + (long long)gr * ld + gk : g;
    if (VEC == 2)
      cp_async16(s + r * PITCH + k, src, ok);
    else
      cp_async8(s + r * PITCH + k, src, ok);
  }
}

// [BK][rows + 2] tile of an MN-contiguous operand.
template <int ROWS, int BK, int PITCH, int VEC, int THREADS>
__device__ __forceinline__ void load_mn_tile3(double* s, const double* g, long long ld, int row0, int rows, int k0,
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

// Fragments of steps 2p and 2p+1 for FR 8-row tiles starting at local row w.
// KMAJ: tile i = rows w + 8i + g (natural); else tiles 2j / 2j+1 = rows
// w + 16j + 2g / + 1 (paired).
template <bool KMAJ, int FR, int PITCH>
__device__ __forceinline__ void load_frag_pair(const double* s, int w, int p, int g, int t, double (&f0)[FR],
                                               double (&f1)[FR]) {
  if (KMAJ) {
#pragma unroll
    for (int i = 0; i < FR; ++i) {
      const double2 v = *reinterpret_cast<const double2*>(s + (w + 8 * i + g) * PITCH + 8 * p + 2 * t);
      f0[i] = v.x;
      f1[i] = v.y;
    }
  } else {
#pragma unroll
    for (int j = 0; j < FR / 2; ++j) {
      const double2 v0 = *reinterpret_cast<const double2*>(s + (8 * p + 2 * t) * PITCH + w + 16 * j + 2 * g);
      const double2 v1 = *reinterpret_cast<const double2*>(s + (8 * p + 2 * t + 1) * PITCH + w + 16 * j + 2 * g);
      f0[2 * j] = v0.x;
      f0[2 * j + 1] = v0.y;
      f1[2 * j] = v1.x;
      f1[2 * j + 1] = v1.y;
    }
  }
}

template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS, Cfg::MINB) dgemm3_kernel(DgemmParams p) {
  extern __shared__ __align__(16) double smem[];
  constexpr int BM = Cfg::BM, BN = Cfg::BN, BK = Cfg::BK, STAGES = Cfg::STAGES;
  constexpr int FM = Cfg::FM, FN = Cfg::FN, PA = Cfg::PA, PB = Cfg::PB;
  int tm, tn;
  if (p.lower) {
    lower_tile(blockIdx.x, tm, tn);
  } else {
    tn = blockIdx.x;  // N tiles fastest (A panel reuse in L2)
    tm = blockIdx.y;
  }
  const int m0 = tm * BM, n0 = tn * BN;
  if (p.n_dev) {
    const int nd = *p.n_dev;
    if (nd < p.N) p.N = nd;
    if (n0 >= p.N) return;
  }
  const int kb = p.k_chunk > 0 ? blockIdx.z * p.k_chunk : (p.tri_b ? (n0 / BK) * BK : 0);
  const int ke = p.k_chunk > 0 ? min(p.K, kb + p.k_chunk) : p.K;
  const int nkt = ke > kb ? (ke - kb + BK - 1) / BK : 0;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp % Cfg::WARPS_M) * Cfg::WM, wn = (warp / Cfg::WARPS_M) * Cfg::WN;
  const int g = lane >> 2, t = lane & 3;
  // warps wholly past a device-bounded N skip their MMAs, and so do the warps
  // of a diagonal lower tile that sit strictly above the diagonal (every
  // lower-tile caller mirrors the lower triangle over the upper one)
  const bool live = n0 + wn < p.N && !(p.lower && tm == tn && wn >= wm + Cfg::WM);

  double acc[FM][FN][2];
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  auto issue = [&](int kt) {
    double* sa = smem + (kt % STAGES) * Cfg::STAGE_ELEMS;
    double* sb = sa + Cfg::EA;
    const int k0 = kb + kt * BK;
    if (Cfg::AK)
      load_k_tile<BM, BK, PA, Cfg::VEC, Cfg::THREADS>(sa, p.A, p.lda, m0, p.M, k0, ke, tid);
    else
      load_mn_tile3<BM, BK, PA, Cfg::VEC, Cfg::THREADS>(sa, p.A, p.lda, m0, p.M, k0, ke, tid);
    if (Cfg::BKM)
      load_k_tile<BN, BK, PB, Cfg::VEC, Cfg::THREADS>(sb, p.B, p.ldb, n0, p.N, k0, ke, tid);
    else
      load_mn_tile3<BN, BK, PB, Cfg::VEC, Cfg::THREADS>(sb, p.B, p.ldb, n0, p.N, k0, ke, tid);
    if (p.scale && tid < BK) {
      const int gk = k0 + tid;
      cp_async8(sb + Cfg::EB + tid, gk < ke ? p.scale + gk : p.scale, gk < ke);
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
    if (!live) continue;
    const double* sa = smem + (kt % STAGES) * Cfg::STAGE_ELEMS;
    const double* sb = sa + Cfg::EA;
    const double* ss = sb + Cfg::EB;
#pragma unroll
    for (int pp = 0; pp < BK / 8; ++pp) {
      double a0[FM], a1[FM], b0[FN], b1[FN];
      load_frag_pair<Cfg::AK, FM, PA>(sa, wm, pp, g, t, a0, a1);
      load_frag_pair<Cfg::BKM, FN, PB>(sb, wn, pp, g, t, b0, b1);
      if (p.scale) {
        const double2 sc = *reinterpret_cast<const double2*>(ss + 8 * pp + 2 * t);
#pragma unroll
        for (int j = 0; j < FN; ++j) {
          b0[j] *= sc.x;
          b1[j] *= sc.y;
        }
      }
      dmma_block<FM, FN>(acc, a0, b0);
      dmma_block<FM, FN>(acc, a1, b1);
    }
  }
  cp_async_wait<0>();

  // Epilogue: accumulator (i, j, h) = C(row(i), col(j, h)).
  auto row_of = [&](int i) { return Cfg::AK ? wm + 8 * i + g : wm + 16 * (i / 2) + 2 * g + (i & 1); };
  auto col_of = [&](int j, int h) {
    return Cfg::BKM ? wn + 8 * j + 2 * t + h : wn + 16 * (j / 2) + 4 * t + 2 * h + (j & 1);
  };
  if (p.partial) {
    double* out = p.partial + (long long)blockIdx.z * p.part_stride;
#pragma unroll
    for (int i = 0; i < FM; ++i)
#pragma unroll
      for (int j = 0; j < FN; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int m = m0 + row_of(i), n = n0 + col_of(j, h);
          if (m < p.M && n < p.N) out[m + (long long)n * p.M] = p.alpha * acc[i][j][h];
        }
    return;
  }
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int m = m0 + row_of(i), n = n0 + col_of(j, h);
        if (m >= p.M || n >= p.N) continue;
        const int nc = p.colmap ? __ldg(p.colmap + n) : n;
        double* c = p.C + m + (long long)nc * p.ldc;
        const double v = p.alpha * acc[i][j][h];
        if (p.beta == 0.0)
          *c = v;
        else
          *c = v + p.beta * (p.Cin ? p.Cin[m + (long long)__ldg(p.cin_map + n) * p.ldcin] : *c);
      }
}

}  // namespace lrgw_dev
