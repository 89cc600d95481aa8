// panel4.cu — the selection's block panel (panel.cu) on the TMA engine
// (gemm4.cuh): one producer warp streams the four K phases' boxes
//   phase 1  Phi_a rows / Phi_a[R]        (A and B boxes)
//   phase 2  Phi_b rows / Phi_b[R]
//   phase 3  L[:, :k] rows / L[R, :k]     (A fragments negated)
//   phase 4  X boxes only: W (parked in shared memory) is the A operand
// into a 3-stage mbarrier ring; four compute warps (16 rows x all 16Q
// columns each) run the DMMA mainloop on swizzled fragments. Phase 4 reuses
// the accumulator layout as the A fragment: thread t of a quad holds W
// columns 16q + 4t + u, u = 2pp + h, while gemm4's k-step (pp, h) reads the
// stage's k row 8pp + 2t + h — so the greedy writes X with its columns
// permuted inside every 16-group (k_mem 8pp + 2t + h <- k 4t + 2pp + h,
// select.cu) and TMA lands them where the fragments look. B rows past nb are
// zero-filled by TMA, so W's dead columns are exact zeros. Epilogue: L_blk
// and the residual downdate as in panel.cu.
#include <cstdlib>

#include "gemm4.cuh"
#include "kernels.h"

namespace lrgw_dev {

namespace {

// load_frag_swz for one k of the pair (h = 0: k = 8p + 2t, h = 1: k + 1): the
// wide bodies load the B halves one at a time (fewer live registers)
template <int FR, int BK>
__device__ __forceinline__ void load_frag_swz1(const double* s, int w, int p, int h, int g, int t, double (&f)[FR]) {
  const int k = 8 * p + 2 * t + h;
#pragma unroll
  for (int j = 0; j < FR / 2; ++j) {
    const double* box = s + ((w >> 4) + j) * (BK * 16);
    const double2 v = *reinterpret_cast<const double2*>(box + k * 16 + 2 * (g ^ (k & 7)));
    f[2 * j] = v.x;
    f[2 * j + 1] = v.y;
  }
}

// dmma_block over the column fragments j >= j0 only (warp-uniform j0): phase 4
// multiplies by X = L_sel^-1, lower triangular, so k-tile q (W columns
// 16 q .. 16 q + 15) contributes nothing to output columns below 16 q — the
// skipped products are exact zeros, the results stay bit for bit.
template <int FM, int FN>
__device__ __forceinline__ void dmma_block_from(double (&acc)[FM][FN][2], const double (&af)[FM],
                                                const double (&bf)[FN], int j0) {
#pragma unroll
  for (int j = 0; j < FN; ++j)
    if (j >= j0) {
#pragma unroll
      for (int i = 0; i < FM; ++i) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
}

struct Panel4Params {
  int M, N, K1, K2, K3;
  double* C;
  long long ldc;
  double* d;
  const int* pos;
  int kend;
};

template <int Q, int STAGES_>
struct P4Cfg {
  static constexpr int BM = 64, BN = 16 * Q, BK = 16, STAGES = STAGES_;
  static constexpr int CWARPS = 4, THREADS = 32 * (CWARPS + 1), CT = 32 * CWARPS;
  static constexpr int FM = 2, FN = 2 * Q;
  static constexpr int BOX = BK * 16;
  static constexpr int A_BOXES = BM / 16, B_BOXES = BN / 16;
  static constexpr int STAGE_ELEMS = (A_BOXES + B_BOXES) * BOX;
  static constexpr unsigned AB_BYTES = STAGE_ELEMS * 8, B_BYTES = B_BOXES * BOX * 8;
  static constexpr int PARK_ELEMS = FM * FN * 2 * CT;
  static constexpr int SMEM_BYTES = (STAGES * STAGE_ELEMS + PARK_ELEMS) * 8 + 1024 + 2 * STAGES * 8;
};

template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS, 2)
    panel4_kernel(const __grid_constant__ CUtensorMap a1, const __grid_constant__ CUtensorMap b1,
                  const __grid_constant__ CUtensorMap a2, const __grid_constant__ CUtensorMap b2,
                  const __grid_constant__ CUtensorMap a3, const __grid_constant__ CUtensorMap b3,
                  const __grid_constant__ CUtensorMap xm, Panel4Params p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int BK = Cfg::BK, STAGES = Cfg::STAGES, FM = Cfg::FM, FN = Cfg::FN, CT = Cfg::CT;
  double* ring = smem_ring_1024(smem_raw);
  double* park_base = ring + STAGES * Cfg::STAGE_ELEMS;
  uint64_t* full = reinterpret_cast<uint64_t*>(park_base + Cfg::PARK_ELEMS);
  uint64_t* empty = full + STAGES;
  const int m0 = blockIdx.x * Cfg::BM;
  const int N = p.N;
  const int e1 = (p.K1 + BK - 1) / BK, e2 = e1 + (p.K2 + BK - 1) / BK, e3 = e2 + (p.K3 + BK - 1) / BK;
  const int nkt = e3 + (N + BK - 1) / BK;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, Cfg::CWARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (warp == Cfg::CWARPS) {  // ===== TMA producer =====
    if (lane == 0) {
      for (int kt = 0; kt < nkt; ++kt) {
        const int s = kt % STAGES;
        if (kt >= STAGES) mbar_wait(empty + s, ((kt / STAGES) - 1) & 1);
        double* sa = ring + s * Cfg::STAGE_ELEMS;
        double* sb = sa + Cfg::A_BOXES * Cfg::BOX;
        if (kt >= e3) {  // phase 4: X boxes only
          mbar_arrive_expect_tx(full + s, Cfg::B_BYTES);
#pragma unroll
          for (int b = 0; b < Cfg::B_BOXES; ++b) tma_load_2d(sb + b * Cfg::BOX, &xm, full + s, 16 * b, (kt - e3) * BK);
          continue;
        }
        const CUtensorMap* ma = kt < e1 ? &a1 : kt < e2 ? &a2 : &a3;
        const CUtensorMap* mb = kt < e1 ? &b1 : kt < e2 ? &b2 : &b3;
        const int k0 = (kt < e1 ? kt : kt < e2 ? kt - e1 : kt - e2) * BK;
        mbar_arrive_expect_tx(full + s, Cfg::AB_BYTES);
#pragma unroll
        for (int b = 0; b < Cfg::A_BOXES; ++b) tma_load_2d(sa + b * Cfg::BOX, ma, full + s, m0 + 16 * b, k0);
#pragma unroll
        for (int b = 0; b < Cfg::B_BOXES; ++b) tma_load_2d(sb + b * Cfg::BOX, mb, full + s, 16 * b, k0);
      }
    }
    return;
  }
  // ===== consumers: warp w owns rows 16 w .. 16 w + 15, all columns =====
  const int wm = warp * 16;
  const int g = lane >> 2, t = lane & 3;
  double* park = park_base + tid;  // slot q of this thread: park[q * CT]
  double acc[FM][FN][2];
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  auto park_acc = [&]() {
#pragma unroll
    for (int i = 0; i < FM; ++i)
#pragma unroll
      for (int j = 0; j < FN; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          park[((i * FN + j) * 2 + h) * CT] = acc[i][j][h];
          acc[i][j][h] = 0.0;
        }
  };
  for (int kt = 0; kt < nkt; ++kt) {
    const int s = kt % STAGES;
    mbar_wait(full + s, (kt / STAGES) & 1);
    if (kt > 0) release_prev(empty + (kt - 1) % STAGES, lane);  // gemm4.cuh: never right behind the slot's own loads
    const double* sa = ring + s * Cfg::STAGE_ELEMS;
    const double* sb = sa + Cfg::A_BOXES * Cfg::BOX;
    if (kt < e3) {
      const bool neg = kt >= e2;
#pragma unroll
      for (int pp = 0; pp < BK / 8; ++pp) {
        double a0[FM], a1_[FM];
        load_frag_swz<FM, BK>(sa, wm, pp, g, t, a0, a1_);
        if (neg) {
#pragma unroll
          for (int i = 0; i < FM; ++i) {
            a0[i] = -a0[i];
            a1_[i] = -a1_[i];
          }
        }
        if constexpr (FN > 10) {
          double bf[FN];
          load_frag_swz1<FN, BK>(sb, 0, pp, 0, g, t, bf);
          dmma_block<FM, FN>(acc, a0, bf);
          load_frag_swz1<FN, BK>(sb, 0, pp, 1, g, t, bf);
          dmma_block<FM, FN>(acc, a1_, bf);
        } else {
          double b0[FN], b1_[FN];
          load_frag_swz<FN, BK>(sb, 0, pp, g, t, b0, b1_);
          dmma_block<FM, FN>(acc, a0, b0);
          dmma_block<FM, FN>(acc, a1_, b1_);
        }
      }
    } else {
      // phase 4, W columns 16 q .. 16 q + 15: k-step (pp, h) <- W column 16 q + 4 t + 2 pp + h
      const int q = kt - e3;
#pragma unroll
      for (int pp = 0; pp < BK / 8; ++pp) {
        double a0[FM], a1_[FM];
#pragma unroll
        for (int i = 0; i < FM; ++i) {
          a0[i] = park[((i * FN + 2 * q) * 2 + pp) * CT];
          a1_[i] = park[((i * FN + 2 * q + 1) * 2 + pp) * CT];
        }
        if constexpr (FN > 10) {
          double bf[FN];
          load_frag_swz1<FN, BK>(sb, 0, pp, 0, g, t, bf);
          dmma_block_from<FM, FN>(acc, a0, bf, 2 * q);
          load_frag_swz1<FN, BK>(sb, 0, pp, 1, g, t, bf);
          dmma_block_from<FM, FN>(acc, a1_, bf, 2 * q);
        } else {
          double b0[FN], b1_[FN];
          load_frag_swz<FN, BK>(sb, 0, pp, g, t, b0, b1_);
          dmma_block_from<FM, FN>(acc, a0, b0, 2 * q);
          dmma_block_from<FM, FN>(acc, a1_, b1_, 2 * q);
        }
      }
    }
    if (kt == e1 - 1) park_acc();
    if (kt == e2 - 1) {
#pragma unroll
      for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j) {
          acc[i][j][0] *= park[((i * FN + j) * 2 + 0) * CT];
          acc[i][j][1] *= park[((i * FN + j) * 2 + 1) * CT];
        }
    }
    if (kt == e3 - 1) park_acc();
  }
  // epilogue: L_blk and the downdate over the 4 lanes of a row pair
#pragma unroll
  for (int ii = 0; ii < FM / 2; ++ii) {
    const int m = m0 + wm + 16 * ii + 2 * g;
    double sq0 = 0.0, sq1 = 0.0;
#pragma unroll
    for (int jn = 0; jn < FN; ++jn)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int n = 16 * (jn / 2) + 4 * t + 2 * h + (jn & 1);
        if (n >= N) continue;
        const double v0 = acc[2 * ii][jn][h], v1 = acc[2 * ii + 1][jn][h];
        sq0 = fma(v0, v0, sq0);
        sq1 = fma(v1, v1, sq1);
        double* c = p.C + m + (long long)n * p.ldc;
        if (m + 1 < p.M)
          *reinterpret_cast<double2*>(c) = make_double2(v0, v1);
        else if (m < p.M)
          c[0] = v0;
      }
    sq0 += __shfl_xor_sync(0xffffffffu, sq0, 1);
    sq1 += __shfl_xor_sync(0xffffffffu, sq1, 1);
    sq0 += __shfl_xor_sync(0xffffffffu, sq0, 2);
    sq1 += __shfl_xor_sync(0xffffffffu, sq1, 2);
    if (t == 0) {
      if (m < p.M && p.pos[m] >= p.kend) p.d[m] -= sq0;
      if (m + 1 < p.M && p.pos[m + 1] >= p.kend) p.d[m + 1] -= sq1;
    }
  }
}

template <class Cfg>
cudaError_t launch_p4(cudaStream_t st, const CUtensorMap (&m)[7], const Panel4Params& p) {
  auto kern = panel4_kernel<Cfg>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES);
  if (e != cudaSuccess) return e;
  kern<<<(p.M + Cfg::BM - 1) / Cfg::BM, Cfg::THREADS, Cfg::SMEM_BYTES, st>>>(m[0], m[1], m[2], m[3], m[4], m[5],
                                                                            m[6], p);
  count_launches(1);
  return cudaGetLastError();
}

}  // namespace

bool select_panel_tma_enabled() {
  static const bool on = !(getenv("LRGW_PANEL_TMA") && atoi(getenv("LRGW_PANEL_TMA")) == 0);
  return on && tma_gemm_enabled();
}

// The X columns inside each 16-group in the order panel4's fragments read
// them: memory column 16 q + r holds X column 16 q + perm(r).
int select_panel_xperm(int r) { return 4 * ((r >> 1) & 3) + 2 * (r >> 3) + (r & 1); }

cudaError_t select_panel_tma(cudaStream_t st, int M, int N, const double* a1, long long lda1, const double* b1,
                             long long ldb1, int k1, const double* a2, long long lda2, const double* b2,
                             long long ldb2, int k2, const double* l, long long ldl, const double* lrow,
                             long long ldlr, int k, const double* xperm, long long ldx, double* c, long long ldc,
                             double* d, const int* pos, int kend) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  if (N < 17 || N > 112 || k1 < 1 || k2 < 1 || k < 0 || ldc % 2 != 0 || (reinterpret_cast<uintptr_t>(c) & 15) != 0)
    return cudaErrorNotSupported;
  CUtensorMap m[7];
  const int kx = (N + 15) / 16 * 16;
  if (!tma_encode_mn(&m[0], a1, M, k1, lda1, 16) || !tma_encode_mn(&m[1], b1, N, k1, ldb1, 16) ||
      !tma_encode_mn(&m[2], a2, M, k2, lda2, 16) || !tma_encode_mn(&m[3], b2, N, k2, ldb2, 16) ||
      !tma_encode_mn(&m[6], xperm, N, kx, ldx, 16) || kx > ldx)
    return cudaErrorNotSupported;
  if (k > 0) {
    if (!tma_encode_mn(&m[4], l, M, k, ldl, 16) || !tma_encode_mn(&m[5], lrow, N, k, ldlr, 16))
      return cudaErrorNotSupported;
  } else {
    m[4] = m[0];
    m[5] = m[1];
  }
  Panel4Params p{M, N, k1, k2, k, c, ldc, d, pos, kend};
  switch ((N + 15) / 16) {
    case 2: return launch_p4<P4Cfg<2, 3>>(st, m, p);
    case 3: return launch_p4<P4Cfg<3, 3>>(st, m, p);
    case 4: return launch_p4<P4Cfg<4, 3>>(st, m, p);
    case 5: return launch_p4<P4Cfg<5, 3>>(st, m, p);
    case 6: return launch_p4<P4Cfg<6, 3>>(st, m, p);
    default: return launch_p4<P4Cfg<7, 2>>(st, m, p);
  }
}

}  // namespace lrgw_dev
