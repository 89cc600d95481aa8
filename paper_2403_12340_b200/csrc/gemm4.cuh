// gemm4.cuh — TMA-fed FP64 DMMA GEMM for MN-contiguous operands.
//
//   C = alpha * A B^T [o (A2 B2^T)] + beta * C,   A: M x K, B: N x K column-major
//
// The Blackwell-native staging of the path's tall GEMMs (the fused fit
// Theta = L L_P^-1, the selection's L-pass and W columns): one producer warp
// issues cp.async.bulk.tensor (TMA) loads of 16-row x BK-deep boxes of A and B
// into a STAGES-deep shared-memory ring and arms an mbarrier per stage with
// the stage's byte count; the consumer warps wait on that barrier, run the
// DMMA.8x8x4 mainloop and release the slot through a second mbarrier. No
// per-thread address arithmetic or LDGSTS in the mainloop, no CTA barrier
// per k-tile; out-of-range rows / k are zero-filled by the TMA unit.
//
// Shared layout: each box is BK rows of 128 bytes (16 doubles) written with
// CU_TENSOR_MAP_SWIZZLE_128B — 16-byte chunk c of row k lands at chunk
// c ^ (k & 7). The paired fragments of gemm2.cuh (rows 2g, 2g + 1 of a
// 16-row group in one LDS.128; k order permuted to 8p + 2t, 8p + 2t + 1) read
// chunk g of rows k: across a quarter-warp (g in {2q, 2q+1}, t = 0..3,
// k & 7 = 2t or 2t + 1) the swizzled chunks g ^ (k & 7) are 8 distinct
// chunks — conflict-free without padding.
#pragma once

#include <cuda.h>

#include "common.cuh"

namespace lrgw_dev {

struct Dgemm4Params {
  int M, N, K, K2;  // K2 > 0: Hadamard second phase (maps A2 / B2)
  double* C;
  long long ldc;
  double alpha, beta;
  int tri_b;           // B(n, k) == 0 for k < n: K starts at the tile's n0
  const int* colmap;   // output column n -> colmap[n]
  const int* n_dev;    // device-side bound on N
  int vec_store;       // C 16-byte aligned with even ldc: paired double2 stores
};

// PROD: one extra warp does nothing but issue the TMAs (its lane 0 waits on
// the empty barriers); otherwise thread 0 of the compute warps refills the
// ring after each k-tile.
template <int BM_, int BN_, int WM_, int WN_, int BK_, int STAGES_, bool HAD_, int MINB_, bool PROD_ = true>
struct Gemm4Cfg {
  static constexpr int BM = BM_, BN = BN_, WM = WM_, WN = WN_, BK = BK_, STAGES = STAGES_, MINB = MINB_;
  static constexpr bool HAD = HAD_, PROD = PROD_;
  static constexpr int WARPS_M = BM / WM, WARPS_N = BN / WN;
  static constexpr int CWARPS = WARPS_M * WARPS_N;  // compute warps
  static constexpr int THREADS = 32 * (CWARPS + (PROD ? 1 : 0));
  static constexpr int FM = WM / 8, FN = WN / 8;
  static constexpr int BOX = BK * 16;  // doubles per 16-row box
  static constexpr int A_BOXES = BM / 16, B_BOXES = BN / 16;
  static constexpr int STAGE_ELEMS = (A_BOXES + B_BOXES) * BOX;
  static constexpr unsigned STAGE_BYTES = STAGE_ELEMS * 8;
  static constexpr int SMEM_BYTES = STAGES * STAGE_ELEMS * 8 + 1024 /* 1024-B alignment */ + 2 * STAGES * 8;
  static_assert(BM % 16 == 0 && BN % 16 == 0 && WM % 16 == 0 && WN % 16 == 0, "16-row boxes / pairs");
  static_assert(BK % 8 == 0, "k pairs, 1024-B aligned boxes");
};

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// Releasing a ring slot. A consumer warp must not arrive on a slot's empty
// barrier while its own shared-memory loads from that slot can still be in
// flight: ptxas schedules the arrive right behind the last LDS (the MMAs that
// consume the loaded registers follow it), and a producer blocked on that
// barrier refills the slot at once — measured on the B200 as run-to-run
// differences of ~1e-6 (tools/stress_quad.py, tools/bench_quad.py). Every
// consumer therefore releases k-tile j - 1 right after its wait for k-tile j:
// the wait's spin loop ends the basic block, so every MMA of tile j - 1 — and
// with it every load it depends on — has issued. The last k-tile of a kernel
// is never refilled and needs no release.
__device__ __forceinline__ void release_prev(uint64_t* empty_prev, int lane) {
  __syncwarp();
  if (lane == 0) mbar_arrive(empty_prev);
}

// 2-D TMA load of box (c0 = row, c1 = k) into shared memory, completing on bar.
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// Paired fragments of k steps 8p + 2t and 8p + 2t + 1 for FR 8-row MMA tiles
// whose 16-row groups start at local row w (tile 2j: rows w + 16j + 2g,
// tile 2j + 1: the next row), from a swizzled [box][BK][16] stage.
template <int FR, int BK>
__device__ __forceinline__ void load_frag_swz(const double* s, int w, int p, int g, int t, double (&f0)[FR],
                                              double (&f1)[FR]) {
  const int k0 = 8 * p + 2 * t, k1 = k0 + 1;
#pragma unroll
  for (int j = 0; j < FR / 2; ++j) {
    const double* box = s + ((w >> 4) + j) * (BK * 16);
    const double2 v0 = *reinterpret_cast<const double2*>(box + k0 * 16 + 2 * (g ^ (k0 & 7)));
    const double2 v1 = *reinterpret_cast<const double2*>(box + k1 * 16 + 2 * (g ^ (k1 & 7)));
    f0[2 * j] = v0.x;
    f0[2 * j + 1] = v0.y;
    f1[2 * j] = v1.x;
    f1[2 * j + 1] = v1.y;
  }
}

template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS, Cfg::MINB)
    dgemm4_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                  const __grid_constant__ CUtensorMap map_a2, const __grid_constant__ CUtensorMap map_b2,
                  Dgemm4Params p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int BM = Cfg::BM, BN = Cfg::BN, BK = Cfg::BK, STAGES = Cfg::STAGES;
  constexpr int FM = Cfg::FM, FN = Cfg::FN;
  double* ring = smem_ring_1024(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + STAGES * Cfg::STAGE_ELEMS);
  uint64_t* empty = full + STAGES;

  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;  // N tiles fastest (A panel reuse in L2)
  int N = p.N;
  if (p.n_dev) N = min(N, *p.n_dev);
  if (n0 >= N) return;
  const int kb = p.tri_b ? (n0 / BK) * BK : 0;
  const int kt1 = p.K > kb ? (p.K - kb + BK - 1) / BK : 0;
  const int kt2 = Cfg::HAD ? (p.K2 + BK - 1) / BK : 0;
  const int nkt = kt1 + kt2;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, Cfg::CWARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  // thread 0 keeps the ring full: stage s of k-tile kt + STAGES is refilled
  // once every warp has released k-tile kt (the empty barrier)
  auto issue = [&](int kt) {
    const int s = kt % STAGES;
    double* sa = ring + s * Cfg::STAGE_ELEMS;
    double* sb = sa + Cfg::A_BOXES * Cfg::BOX;
    mbar_arrive_expect_tx(full + s, Cfg::STAGE_BYTES);
    const bool ph2 = Cfg::HAD && kt >= kt1;
    const CUtensorMap* ma = ph2 ? &map_a2 : &map_a;
    const CUtensorMap* mb = ph2 ? &map_b2 : &map_b;
    const int k0 = ph2 ? (kt - kt1) * BK : kb + kt * BK;
#pragma unroll
    for (int b = 0; b < Cfg::A_BOXES; ++b) tma_load_2d(sa + b * Cfg::BOX, ma, full + s, m0 + 16 * b, k0);
#pragma unroll
    for (int b = 0; b < Cfg::B_BOXES; ++b) tma_load_2d(sb + b * Cfg::BOX, mb, full + s, n0 + 16 * b, k0);
  };
  if (tid == (Cfg::PROD ? 32 * Cfg::CWARPS : 0)) {
    tma_prefetch_desc(&map_a);
    tma_prefetch_desc(&map_b);
    if (Cfg::HAD) {
      tma_prefetch_desc(&map_a2);
      tma_prefetch_desc(&map_b2);
    }
    for (int kt = 0; kt < STAGES && kt < nkt; ++kt) issue(kt);
    if (Cfg::PROD)
      for (int kt = STAGES; kt < nkt; ++kt) {
        mbar_wait(empty + kt % STAGES, ((kt / STAGES) - 1) & 1);
        issue(kt);
      }
  }
  if (Cfg::PROD && warp == Cfg::CWARPS) return;

  // ===== consumers =====
  const int wm = (warp % Cfg::WARPS_M) * Cfg::WM, wn = (warp / Cfg::WARPS_M) * Cfg::WN;
  const int g = lane >> 2, t = lane & 3;
  const bool live = n0 + wn < N;
  // leading k-tiles that are zero for this warp's columns (triangular B)
  const int kz = p.tri_b ? max(0, (n0 + wn - kb) / BK) : 0;
  double acc[FM][FN][2];
  double first[Cfg::HAD ? FM : 1][Cfg::HAD ? FN : 1][2];
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  for (int kt = 0; kt < nkt; ++kt) {
    const int s = kt % STAGES;
    if (Cfg::HAD && kt == kt1) {  // the first product waits in registers
#pragma unroll
      for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j) {
          first[i][j][0] = acc[i][j][0];
          first[i][j][1] = acc[i][j][1];
          acc[i][j][0] = acc[i][j][1] = 0.0;
        }
    }
    mbar_wait(full + s, (kt / STAGES) & 1);
    if (kt > 0) {
      release_prev(empty + (kt - 1) % STAGES, lane);
      if (!Cfg::PROD && tid == 0 && kt - 1 + STAGES < nkt) {
        mbar_wait(empty + (kt - 1) % STAGES, ((kt - 1) / STAGES) & 1);
        issue(kt - 1 + STAGES);
      }
    }
    // triangular B: a k-tile wholly left of the warp's first column is zero
    // for the whole warp (the tile-level skip only starts K at n0) — skip its
    // MMAs (exact: the skipped products are zeros)
    if (live && kt >= kz) {
      const double* sa = ring + s * Cfg::STAGE_ELEMS;
      const double* sb = sa + Cfg::A_BOXES * Cfg::BOX;
#pragma unroll
      for (int pp = 0; pp < BK / 8; ++pp) {
        double a0[FM], a1[FM], b0[FN], b1[FN];
        load_frag_swz<FM, BK>(sa, wm, pp, g, t, a0, a1);
        load_frag_swz<FN, BK>(sb, wn, pp, g, t, b0, b1);
        dmma_block<FM, FN>(acc, a0, b0);
        dmma_block<FM, FN>(acc, a1, b1);
      }
    }
  }
  if (!live) return;
  if (Cfg::HAD) {
#pragma unroll
    for (int i = 0; i < FM; ++i)
#pragma unroll
      for (int j = 0; j < FN; ++j) {
        acc[i][j][0] *= first[i][j][0];
        acc[i][j][1] *= first[i][j][1];
      }
  }
  // epilogue: accumulator (i, j, h) = C(m0 + wm + 16 (i/2) + 2g + (i&1), n0 + wn + 16 (j/2) + 4t + 2h + (j&1))
#pragma unroll
  for (int j = 0; j < FN; ++j)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int n = n0 + wn + 16 * (j / 2) + 4 * t + 2 * h + (j & 1);
      if (n >= N) continue;
      const long long nc = p.colmap ? __ldg(p.colmap + n) : n;
      double* col = p.C + nc * p.ldc;
#pragma unroll
      for (int ii = 0; ii < FM / 2; ++ii) {
        const int m = m0 + wm + 16 * ii + 2 * g;
        double v0 = p.alpha * acc[2 * ii][j][h], v1 = p.alpha * acc[2 * ii + 1][j][h];
        if (p.vec_store && m + 1 < p.M) {
          double2* c2 = reinterpret_cast<double2*>(col + m);
          if (p.beta != 0.0) {
            const double2 o = *c2;
            v0 += p.beta * o.x;
            v1 += p.beta * o.y;
          }
          *c2 = make_double2(v0, v1);
        } else {
          if (m < p.M) col[m] = p.beta != 0.0 ? v0 + p.beta * col[m] : v0;
          if (m + 1 < p.M) col[m + 1] = p.beta != 0.0 ? v1 + p.beta * col[m + 1] : v1;
        }
      }
    }
}

// Persistent form of dgemm4_kernel (no Hadamard phase, no device N): each CTA
// walks a contiguous run of tiles (N tiles fastest), and the TMA
// warp's ring runs on across tile boundaries (global k-tile count g for the
// stage and phase), so the next tile's first boxes load during this tile's
// epilogue — the per-tile fill / drain the one-tile-per-CTA grid pays on
// short K (the Si64 fit: K 128..1024 by the triangular skip).
template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS, Cfg::MINB)
    dgemm4p_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                   Dgemm4Params p, int tiles_m, int tiles_n) {
  static_assert(Cfg::PROD && !Cfg::HAD, "persistent: TMA warp, single phase");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int BM = Cfg::BM, BN = Cfg::BN, BK = Cfg::BK, STAGES = Cfg::STAGES;
  constexpr int FM = Cfg::FM, FN = Cfg::FN;
  double* ring = smem_ring_1024(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + STAGES * Cfg::STAGE_ELEMS);
  uint64_t* empty = full + STAGES;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, Cfg::CWARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const int ntiles = tiles_m * tiles_n, N = p.N;
  // a contiguous run of tiles per CTA (N fastest): whole tile rows, so the
  // triangular-B work per CTA balances and a row's A panel stays in L2
  const int t_begin = static_cast<int>((long long)ntiles * blockIdx.x / gridDim.x);
  const int t_end = static_cast<int>((long long)ntiles * (blockIdx.x + 1) / gridDim.x);
  if (warp == Cfg::CWARPS) {  // ===== TMA producer =====
    if (lane != 0) return;
    tma_prefetch_desc(&map_a);
    tma_prefetch_desc(&map_b);
    long long gk = 0;
    for (int tile = t_begin; tile < t_end; ++tile) {
      const int m0 = (tile / tiles_n) * BM, n0 = (tile % tiles_n) * BN;
      const int kb = p.tri_b ? (n0 / BK) * BK : 0;
      const int kt1 = p.K > kb ? (p.K - kb + BK - 1) / BK : 0;
      for (int kt = 0; kt < kt1; ++kt, ++gk) {
        const int s = static_cast<int>(gk % STAGES);
        if (gk >= STAGES) mbar_wait(empty + s, static_cast<unsigned>(((gk / STAGES) - 1) & 1));
        double* sa = ring + s * Cfg::STAGE_ELEMS;
        double* sb = sa + Cfg::A_BOXES * Cfg::BOX;
        mbar_arrive_expect_tx(full + s, Cfg::STAGE_BYTES);
        const int k0 = kb + kt * BK;
#pragma unroll
        for (int b = 0; b < Cfg::A_BOXES; ++b) tma_load_2d(sa + b * Cfg::BOX, &map_a, full + s, m0 + 16 * b, k0);
#pragma unroll
        for (int b = 0; b < Cfg::B_BOXES; ++b) tma_load_2d(sb + b * Cfg::BOX, &map_b, full + s, n0 + 16 * b, k0);
      }
    }
    return;
  }
  // ===== consumers =====
  const int wm = (warp % Cfg::WARPS_M) * Cfg::WM, wn = (warp / Cfg::WARPS_M) * Cfg::WN;
  const int g = lane >> 2, t = lane & 3;
  long long gk = 0;
  for (int tile = t_begin; tile < t_end; ++tile) {
    const int m0 = (tile / tiles_n) * BM, n0 = (tile % tiles_n) * BN;
    const int kb = p.tri_b ? (n0 / BK) * BK : 0;
    const int kt1 = p.K > kb ? (p.K - kb + BK - 1) / BK : 0;
    const bool live = n0 + wn < N;
    const int kz = p.tri_b ? max(0, (n0 + wn - kb) / BK) : 0;
    double acc[FM][FN][2];
#pragma unroll
    for (int i = 0; i < FM; ++i)
#pragma unroll
      for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    for (int kt = 0; kt < kt1; ++kt, ++gk) {
      const int s = static_cast<int>(gk % STAGES);
      mbar_wait(full + s, static_cast<unsigned>((gk / STAGES) & 1));
      if (gk > 0) release_prev(empty + static_cast<int>((gk - 1) % STAGES), lane);
      if (live && kt >= kz) {
        const double* sa = ring + s * Cfg::STAGE_ELEMS;
        const double* sb = sa + Cfg::A_BOXES * Cfg::BOX;
#pragma unroll
        for (int pp = 0; pp < BK / 8; ++pp) {
          double a0[FM], a1[FM], b0[FN], b1[FN];
          load_frag_swz<FM, BK>(sa, wm, pp, g, t, a0, a1);
          load_frag_swz<FN, BK>(sb, wn, pp, g, t, b0, b1);
          dmma_block<FM, FN>(acc, a0, b0);
          dmma_block<FM, FN>(acc, a1, b1);
        }
      }
    }
    if (!live) continue;
#pragma unroll
    for (int j = 0; j < FN; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int n = n0 + wn + 16 * (j / 2) + 4 * t + 2 * h + (j & 1);
        if (n >= N) continue;
        const long long nc = p.colmap ? __ldg(p.colmap + n) : n;
        double* col = p.C + nc * p.ldc;
#pragma unroll
        for (int ii = 0; ii < FM / 2; ++ii) {
          const int m = m0 + wm + 16 * ii + 2 * g;
          double v0 = p.alpha * acc[2 * ii][j][h], v1 = p.alpha * acc[2 * ii + 1][j][h];
          if (p.vec_store && m + 1 < p.M) {
            double2* c2 = reinterpret_cast<double2*>(col + m);
            if (p.beta != 0.0) {
              const double2 o = *c2;
              v0 += p.beta * o.x;
              v1 += p.beta * o.y;
            }
            *c2 = make_double2(v0, v1);
          } else {
            if (m < p.M) col[m] = p.beta != 0.0 ? v0 + p.beta * col[m] : v0;
            if (m + 1 < p.M) col[m + 1] = p.beta != 0.0 ? v1 + p.beta * col[m + 1] : v1;
          }
        }
      }
  }
}

// ---------------------------------------------------------------------------
// K-contiguous operands (the G-space SYRK Theta^T V Theta over the half
// spectrum: X is 2K x n_mu with each column's k contiguous):
//   C = alpha * sum_k A(m, k) s(k) B(n, k) (+ beta C),   A(m, k) at m * lda + k
// Boxes are {16 k, BM rows}: each row's 16 k values are one 128-byte line,
// 128B-swizzled (chunk c of row r at c ^ (r & 7)). A thread's k pair
// (8p + 2t, 8p + 2t + 1) is chunk 4p + t; to keep a quarter-warp's 8 LDS.128
// on 8 distinct chunks, the MMA fragment row g maps to the physical row
// rp(g) = (g >> 1) + 4 (g & 1) of its 8-row group (the two rows a
// quarter-warp touches then differ in bit 2 of the swizzle key). The same
// permutation is undone in the epilogue (C's row g -> rp(g); its columns
// 2t, 2t + 1 -> t, t + 4). Lower-triangle tiles, the diagonal scale s(k)
// (read through L1, one double2 per k pair) and split-K partials as in the
// v3 engine (gemm3.cuh).
// ---------------------------------------------------------------------------
struct Dgemm4kParams {
  int M, N, K;
  double* C;
  long long ldc;
  double alpha, beta;
  const double* scale;  // length K or nullptr
  int lower;            // only tiles with tile_n <= tile_m (BM == BN)
  int k_chunk;          // split-K chunk (multiple of 16) when gridDim.z > 1
  double* partial;      // split-K: alpha * acc to partial + z * part_stride (ld M)
  long long part_stride;
};

template <int BM_, int BN_, int WM_, int WN_, int STAGES_, int MINB_, bool PROD_ = false>
struct Gemm4kCfg {
  static constexpr int BM = BM_, BN = BN_, WM = WM_, WN = WN_, BK = 16, STAGES = STAGES_, MINB = MINB_;
  static constexpr bool PROD = PROD_;
  static constexpr int WARPS_M = BM / WM, WARPS_N = BN / WN;
  static constexpr int CWARPS = WARPS_M * WARPS_N;  // compute warps (+ 1 TMA warp when PROD)
  static constexpr int THREADS = 32 * (CWARPS + (PROD ? 1 : 0));
  static constexpr int FM = WM / 8, FN = WN / 8;
  static constexpr int STAGE_ELEMS = (BM + BN) * 16;
  static constexpr unsigned STAGE_BYTES = STAGE_ELEMS * 8;
  static constexpr int SMEM_BYTES = STAGES * STAGE_ELEMS * 8 + 1024 + 2 * STAGES * 8;
  static_assert(BM % 8 == 0 && BN % 8 == 0 && BM <= 256 && BN <= 256, "one box of <= 256 rows per operand");
};

__device__ __forceinline__ int perm_row(int g) { return (g >> 1) + 4 * (g & 1); }

// k-pair fragments (steps 2p, 2p+1) of FR 8-row tiles from a swizzled [rows][16] stage
template <int FR>
__device__ __forceinline__ void load_frag_kswz(const double* s, int w, int p, int g, int t, double (&f0)[FR],
                                               double (&f1)[FR]) {
  const int rp = perm_row(g);
  const int chunk = (4 * p + t) ^ rp;  // (w + 8 i) is a multiple of 8: row & 7 == rp
#pragma unroll
  for (int i = 0; i < FR; ++i) {
    const double2 v = *reinterpret_cast<const double2*>(s + (w + 8 * i + rp) * 16 + 2 * chunk);
    f0[i] = v.x;
    f1[i] = v.y;
  }
}

template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS, Cfg::MINB)
    dgemm4k_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                   Dgemm4kParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int BM = Cfg::BM, BN = Cfg::BN, STAGES = Cfg::STAGES, FM = Cfg::FM, FN = Cfg::FN;
  double* ring = smem_ring_1024(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + STAGES * Cfg::STAGE_ELEMS);
  uint64_t* empty = full + STAGES;
  int tm, tn;
  if (p.lower) {
    lower_tile(blockIdx.x, tm, tn);
  } else {
    tn = blockIdx.x;
    tm = blockIdx.y;
  }
  const int m0 = tm * BM, n0 = tn * BN;
  const int kb = p.k_chunk > 0 ? blockIdx.z * p.k_chunk : 0;
  const int ke = p.k_chunk > 0 ? min(p.K, kb + p.k_chunk) : p.K;
  const int nkt = ke > kb ? (ke - kb + 15) / 16 : 0;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, Cfg::CWARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int kt) {
    const int s = kt % STAGES;
    double* sa = ring + s * Cfg::STAGE_ELEMS;
    mbar_arrive_expect_tx(full + s, Cfg::STAGE_BYTES);
    tma_load_2d(sa, &map_a, full + s, kb + kt * 16, m0);
    tma_load_2d(sa + BM * 16, &map_b, full + s, kb + kt * 16, n0);
  };
  if (tid == (Cfg::PROD ? 32 * Cfg::CWARPS : 0)) {
    tma_prefetch_desc(&map_a);
    tma_prefetch_desc(&map_b);
    for (int kt = 0; kt < STAGES && kt < nkt; ++kt) issue(kt);
    if (Cfg::PROD)
      for (int kt = STAGES; kt < nkt; ++kt) {
        mbar_wait(empty + kt % STAGES, ((kt / STAGES) - 1) & 1);
        issue(kt);
      }
  }
  if (Cfg::PROD && warp == Cfg::CWARPS) return;
  const int wm = (warp % Cfg::WARPS_M) * Cfg::WM, wn = (warp / Cfg::WARPS_M) * Cfg::WN;
  const int g = lane >> 2, t = lane & 3;
  // warps of a diagonal lower tile strictly above the diagonal skip their MMAs
  const bool live = !(p.lower && tm == tn && wn >= wm + Cfg::WM);
  double acc[FM][FN][2];
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  for (int kt = 0; kt < nkt; ++kt) {
    const int s = kt % STAGES;
    const int kg = kb + kt * 16;
    double2 sc[2] = {make_double2(1.0, 1.0), make_double2(1.0, 1.0)};
    if (p.scale) {
#pragma unroll
      for (int pp = 0; pp < 2; ++pp) {
        const int k = kg + 8 * pp + 2 * t;
        sc[pp] = k + 1 < ke ? __ldg(reinterpret_cast<const double2*>(p.scale + k))
                            : make_double2(k < ke ? __ldg(p.scale + k) : 0.0, 0.0);
      }
    }
    mbar_wait(full + s, (kt / STAGES) & 1);
    if (kt > 0) {
      release_prev(empty + (kt - 1) % STAGES, lane);
      if (!Cfg::PROD && tid == 0 && kt - 1 + STAGES < nkt) {
        mbar_wait(empty + (kt - 1) % STAGES, ((kt - 1) / STAGES) & 1);
        issue(kt - 1 + STAGES);
      }
    }
    if (live) {
      const double* sa = ring + s * Cfg::STAGE_ELEMS;
      const double* sb = sa + BM * 16;
#pragma unroll
      for (int pp = 0; pp < 2; ++pp) {
        double a0[FM], a1[FM], b0[FN], b1[FN];
        load_frag_kswz<FM>(sa, wm, pp, g, t, a0, a1);
        load_frag_kswz<FN>(sb, wn, pp, g, t, b0, b1);
        if (p.scale) {
#pragma unroll
          for (int j = 0; j < FN; ++j) {
            b0[j] *= sc[pp].x;
            b1[j] *= sc[pp].y;
          }
        }
        dmma_block<FM, FN>(acc, a0, b0);
        dmma_block<FM, FN>(acc, a1, b1);
      }
    }
  }
  if (!live) return;
  const int rp = perm_row(g);
  double* out = p.partial ? p.partial + (long long)blockIdx.z * p.part_stride : p.C;
  const long long ldo = p.partial ? p.M : p.ldc;
#pragma unroll
  for (int i = 0; i < FM; ++i) {
    const int m = m0 + wm + 8 * i + rp;
    if (m >= p.M) continue;
#pragma unroll
    for (int j = 0; j < FN; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int n = n0 + wn + 8 * j + t + 4 * h;
        if (n >= p.N) continue;
        double* c = out + m + (long long)n * ldo;
        const double v = p.alpha * acc[i][j][h];
        *c = (p.partial || p.beta == 0.0) ? v : v + p.beta * *c;
      }
  }
}

}  // namespace lrgw_dev
