// quad4.cu — K3 on the TMA engine: the fused Cauchy-quadrature / Hadamard
// FP64 DMMA kernel of quadrature.cu with Blackwell-native staging.
//
// Same contract as quad_kernel (contour_node_term + sum_node_terms,
// contour.hpp:144-222): per lower 64 x 64 tile of T and per node k
//   Jc = Phi_c,mu diag(1/(z_k - e_c)) Phi_c,mu^T,  Jv likewise (complex)
//   acc += (w g)_re Im(Jv o Jc) + (w g)_im Re(Jv o Jc)
// on the same persistent schedule (one contiguous run of (tile, node) units
// per CTA, one 64 x 64 partial per tile segment, fixed-order reduction by
// quad_reduce_kernel): the node and segment summation order is the cp.async
// kernel's; only the order of the bands inside a product differs (k-tile
// depth and the paired-fragment k permutation).
//
// What changes is the feed: a producer warp (one elected lane) issues
// cp.async.bulk.tensor boxes of the Phi_mu row panels (16 rows x BK bands,
// 128-byte swizzle, gemm4.cuh's MN-contiguous layout) into an mbarrier ring
// that runs on across node and tile boundaries; the eight compute warps
// (32 x 16 tiles, paired fragments) never compute an address or meet at a CTA
// barrier. The k-tile's slice of the node's diagonal 1/(z_k - e) rides in the
// same stage (a 1-D bulk copy on the stage's barrier) and is fused into the B
// fragments. The conduction factors P1, P2 wait out the valence phase in a
// per-thread shared-memory park (conflict-free [value][thread] layout) instead
// of 64 registers (a TMA warp beside eight compute warps caps the kernel at 168
// registers), so the mainloop holds three accumulator tiles and ptxas has room
// to run the fragment loads ahead of the MMAs.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>

#include "gemm4.cuh"
#include "kernels.h"

namespace lrgw_dev {

namespace {

constexpr int Q4BM = 64;                    // tile edge (== quadrature.cu's QBM: shared partial layout)
constexpr int Q4WM = 32, Q4WN = 16;         // warp tile
constexpr int Q4WARPS_M = Q4BM / Q4WM;      // 2 (x 4 warp columns)
constexpr int Q4CWARPS = Q4WARPS_M * (Q4BM / Q4WN);  // 8 compute warps
constexpr int Q4THREADS = 32 * (Q4CWARPS + 1);       // + the TMA warp
constexpr int Q4FM = Q4WM / 8, Q4FN = Q4WN / 8;      // 4 x 2 fragments
constexpr int Q4ACC = Q4FM * Q4FN * 2;               // 16 values per accumulator tile and thread
constexpr int Q4BOXES = 2 * (Q4BM / 16);             // 4 A + 4 B boxes per stage

template <int BK>
struct Q4 {
  static constexpr int STAGES = BK <= 16 ? 8 : BK <= 24 ? 6 : BK <= 32 ? 4 : BK <= 48 ? 3 : 2;
  static constexpr int NPP = BK / 8;  // k-pair steps (8 bands) per k-tile
  static constexpr int BOX = BK * 16;
  static constexpr int STAGE_ELEMS = Q4BOXES * BOX;
  static constexpr unsigned BOX_BYTES = STAGE_ELEMS * 8;
  static constexpr int PARK_ELEMS = 2 * Q4ACC * 32 * Q4CWARPS;  // P1, P2 of every compute thread
  static constexpr int DIAG_ELEMS = STAGES * BK * 2;            // the k-tiles' complex diagonals
  static constexpr int SMEM_BYTES = (STAGES * STAGE_ELEMS + PARK_ELEMS + DIAG_ELEMS) * 8 + 1024 + 2 * STAGES * 8;
  static_assert(BK % 8 == 0, "k pairs, 1024-B aligned boxes");
  static_assert(SMEM_BYTES <= 232448, "227 KB of shared memory per CTA");
};

struct Quad4Params {
  int n_v, n_c, n_nodes;
  long long units;
  const double2* dv;  // [node][n_v]
  const double2* dc;  // [node][n_c]
  const double2* gw;  // [node]
  const int* seg_base;
  double* partial;
};

__host__ __device__ __forceinline__ long long q4_run_begin(long long units, int ctas, int c) {
  return units * c / ctas;
}

__device__ __forceinline__ void q4_bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// One k-pair step's operands: the paired A / B fragments (gemm4.cuh's
// load_frag_swz addressing) of bands 8pp + 2t and 8pp + 2t + 1 and their
// complex diagonal entries.
struct Q4Frag {
  double2 a[Q4FM];  // [2 * group + (k1 ? 1 : 0)]
  double2 b[Q4FN];
  double2 d[2];
};

__device__ __forceinline__ double2 q4_lds2(const double* p) { return *reinterpret_cast<const double2*>(p); }

template <int BK>
__device__ __forceinline__ void q4_load(Q4Frag& f, const double* sa, const double* sb, const double* sd, int wm,
                                        int wn, int pp, int g, int t) {
  const int k0 = 8 * pp + 2 * t, k1 = k0 + 1;
  const int c0 = 2 * (g ^ (k0 & 7)), c1 = 2 * (g ^ (k1 & 7));
#pragma unroll
  for (int j = 0; j < Q4FM / 2; ++j) {
    const double* box = sa + ((wm >> 4) + j) * (BK * 16);
    f.a[2 * j] = q4_lds2(box + k0 * 16 + c0);
    f.a[2 * j + 1] = q4_lds2(box + k1 * 16 + c1);
  }
#pragma unroll
  for (int j = 0; j < Q4FN / 2; ++j) {
    const double* box = sb + ((wn >> 4) + j) * (BK * 16);
    f.b[2 * j] = q4_lds2(box + k0 * 16 + c0);
    f.b[2 * j + 1] = q4_lds2(box + k1 * 16 + c1);
  }
  f.d[0] = q4_lds2(sd + 2 * k0);
  f.d[1] = q4_lds2(sd + 2 * k1);
}

__device__ __forceinline__ void q4_mma(double (&accR)[Q4FM][Q4FN][2], double (&accI)[Q4FM][Q4FN][2],
                                       const Q4Frag& f) {
#pragma unroll
  for (int h = 0; h < 2; ++h) {  // the step's two bands
    double a[Q4FM], br[Q4FN], bi[Q4FN];
#pragma unroll
    for (int j = 0; j < Q4FM / 2; ++j) {
      a[2 * j] = f.a[2 * j + h].x;
      a[2 * j + 1] = f.a[2 * j + h].y;
    }
#pragma unroll
    for (int j = 0; j < Q4FN / 2; ++j) {
      br[2 * j] = f.b[2 * j + h].x * f.d[h].x;
      br[2 * j + 1] = f.b[2 * j + h].y * f.d[h].x;
      bi[2 * j] = f.b[2 * j + h].x * f.d[h].y;
      bi[2 * j + 1] = f.b[2 * j + h].y * f.d[h].y;
    }
    dmma_block<Q4FM, Q4FN>(accR, a, br);
    dmma_block<Q4FM, Q4FN>(accI, a, bi);
  }
}

template <int BK>
__global__ void __launch_bounds__(Q4THREADS, 1)
    quad4_kernel(const __grid_constant__ CUtensorMap map_c, const __grid_constant__ CUtensorMap map_v,
                 Quad4Params p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  using C = Q4<BK>;
  constexpr int STAGES = C::STAGES, NPP = C::NPP;
  double* ring = smem_ring_1024(smem_raw);
  double* park = ring + STAGES * C::STAGE_ELEMS;
  double* diag = park + C::PARK_ELEMS;
  uint64_t* full = reinterpret_cast<uint64_t*>(diag + C::DIAG_ELEMS);
  uint64_t* empty = full + STAGES;

  const long long u0 = q4_run_begin(p.units, gridDim.x, blockIdx.x);
  const long long u1 = q4_run_begin(p.units, gridDim.x, blockIdx.x + 1);
  if (u1 <= u0) return;
  const int ktc = (p.n_c + BK - 1) / BK, ktv = (p.n_v + BK - 1) / BK, ktt = ktc + ktv;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, Q4CWARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  // a band tail copies fewer than BK diagonal entries: the rest of the slot
  // must hold finite values (they meet zero-filled Phi bands)
  for (int i = tid; i < C::DIAG_ELEMS; i += Q4THREADS) diag[i] = 0.0;
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  __syncthreads();

  if (warp == Q4CWARPS) {  // ===== TMA producer: the flattened (unit, {c, v}, k-tile) stream =====
    if (lane != 0) return;
    tma_prefetch_desc(&map_c);
    tma_prefetch_desc(&map_v);
    long long gk = 0;
    int tile = static_cast<int>(u0 / p.n_nodes), node = static_cast<int>(u0 % p.n_nodes);
    int tm, tn;
    lower_tile(tile, tm, tn);
    for (long long u = u0; u < u1; ++u) {
      for (int kt = 0; kt < ktt; ++kt, ++gk) {
        const int s = static_cast<int>(gk % STAGES);
        if (gk >= STAGES) mbar_wait(empty + s, static_cast<unsigned>(((gk / STAGES) - 1) & 1));
        double* sa = ring + s * C::STAGE_ELEMS;
        double* sb = sa + (Q4BM / 16) * C::BOX;
        const bool cph = kt < ktc;
        const CUtensorMap* m = cph ? &map_c : &map_v;
        const int k0 = (cph ? kt : kt - ktc) * BK;
        const int kk = min(BK, (cph ? p.n_c : p.n_v) - k0);
        const double2* dtab = cph ? p.dc + (long long)node * p.n_c : p.dv + (long long)node * p.n_v;
        mbar_arrive_expect_tx(full + s, C::BOX_BYTES + 16u * kk);
        q4_bulk_g2s(diag + s * BK * 2, dtab + k0, 16u * kk, full + s);
#pragma unroll
        for (int b = 0; b < Q4BM / 16; ++b) tma_load_2d(sa + b * C::BOX, m, full + s, tm * Q4BM + 16 * b, k0);
#pragma unroll
        for (int b = 0; b < Q4BM / 16; ++b) tma_load_2d(sb + b * C::BOX, m, full + s, tn * Q4BM + 16 * b, k0);
      }
      if (++node == p.n_nodes) {
        node = 0;
        lower_tile(++tile, tm, tn);
      }
    }
    return;
  }

  // ===== consumers =====
  const int wm = (warp % Q4WARPS_M) * Q4WM, wn = (warp / Q4WARPS_M) * Q4WN;
  const int g = lane >> 2, t = lane & 3;
  double* mypark = park + tid;  // value v of this thread at mypark[v * 256]
  constexpr int PSTR = 32 * Q4CWARPS;

  double accR[Q4FM][Q4FN][2], accI[Q4FM][Q4FN][2], tac[Q4FM][Q4FN][2];
#pragma unroll
  for (int i = 0; i < Q4FM; ++i)
#pragma unroll
    for (int j = 0; j < Q4FN; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) accR[i][j][h] = accI[i][j][h] = tac[i][j][h] = 0.0;

  int slot = p.seg_base[blockIdx.x];
  int node = static_cast<int>(u0 % p.n_nodes);
  auto stage_a = [&](long long j) { return ring + static_cast<int>(j % STAGES) * C::STAGE_ELEMS; };
  auto stage_d = [&](long long j) { return diag + static_cast<int>(j % STAGES) * (BK * 2); };
  long long gk = 0;
  for (long long u = u0; u < u1; ++u) {
    for (int kt = 0; kt < ktt; ++kt, ++gk) {
      const double* sa = stage_a(gk);
      const double* sd = stage_d(gk);
      mbar_wait(full + static_cast<int>(gk % STAGES), static_cast<unsigned>((gk / STAGES) & 1));
      // the previous k-tile's slot goes back only now (gemm4.cuh:release_prev):
      // released right behind its own loads, the refill raced them — bit
      // differences between runs at Si216 / Si512
      if (gk > 0) release_prev(empty + static_cast<int>((gk - 1) % STAGES), lane);
      // plain loads: ptxas runs them ahead of the MMAs (an explicit register
      // double buffer with pinned loads measured 4-8 points slower)
#pragma unroll
      for (int pp = 0; pp < NPP; ++pp) {
        Q4Frag f;
        q4_load<BK>(f, sa, sa + (Q4BM / 16) * C::BOX, sd, wm, wn, pp, g, t);
        q4_mma(accR, accI, f);
      }

      if (kt == ktc - 1) {
        // end of the c phase: fold the node's w*g into the conduction factors and park them
        const double2 wg = __ldg(p.gw + node);
#pragma unroll
        for (int i = 0; i < Q4FM; ++i)
#pragma unroll
          for (int j = 0; j < Q4FN; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const double cr = accR[i][j][h], ci = accI[i][j][h];
              const int v = (i * Q4FN + j) * 2 + h;
              mypark[v * PSTR] = wg.x * ci + wg.y * cr;
              mypark[(Q4ACC + v) * PSTR] = wg.x * cr - wg.y * ci;
              accR[i][j][h] = accI[i][j][h] = 0.0;
            }
      } else if (kt == ktt - 1) {
        // end of the v phase: weighted complex-Hadamard accumulation
#pragma unroll
        for (int i = 0; i < Q4FM; ++i)
#pragma unroll
          for (int j = 0; j < Q4FN; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int v = (i * Q4FN + j) * 2 + h;
              const double p1 = mypark[v * PSTR], p2 = mypark[(Q4ACC + v) * PSTR];
              tac[i][j][h] = fma(accR[i][j][h], p1, fma(accI[i][j][h], p2, tac[i][j][h]));
              accR[i][j][h] = accI[i][j][h] = 0.0;
            }
        // last node of this CTA's segment of the tile: flush the partial
        if (u + 1 == u1 || node + 1 == p.n_nodes) {
          double* out = p.partial + (long long)slot * Q4BM * Q4BM;
          // accumulator (i, j, h) = tile(wm + 16 (i/2) + 2g + (i&1), wn + 16 (j/2) + 4t + 2h + (j&1))
#pragma unroll
          for (int i = 0; i < Q4FM; ++i)
#pragma unroll
            for (int jj = 0; jj < Q4FN / 2; ++jj)
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int m = wm + 16 * (i / 2) + 2 * g + (i & 1), n = wn + 16 * jj + 4 * t + 2 * h;
                *reinterpret_cast<double2*>(out + m * Q4BM + n) =
                    make_double2(tac[i][2 * jj][h], tac[i][2 * jj + 1][h]);
                tac[i][2 * jj][h] = tac[i][2 * jj + 1][h] = 0.0;
              }
          ++slot;
        }
      }
    }
    if (++node == p.n_nodes) node = 0;
  }
}

template <int BK>
cudaError_t launch_quad4(cudaStream_t st, int ctas, const CUtensorMap& mc, const CUtensorMap& mv,
                         const Quad4Params& p) {
  auto kern = quad4_kernel<BK>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Q4<BK>::SMEM_BYTES);
  if (e != cudaSuccess) return e;
  kern<<<ctas, Q4THREADS, Q4<BK>::SMEM_BYTES, st>>>(mc, mv, p);
  count_launches(1);
  return cudaGetLastError();
}

}  // namespace

bool quad_tma_enabled() {
  const char* v = getenv("LRGW_QUAD_TMA");  // read per call: tools compare the two feeds in one process
  return !(v && atoi(v) == 0);
}

// The node kernel of quad_nodes on the TMA feed (the caller runs the plan
// upload before and quad_reduce_kernel after). cudaErrorNotSupported: the
// Phi_mu panels do not qualify for a tensor map (odd leading dimension or
// unaligned base) — the caller keeps the cp.async kernel.
cudaError_t quad_nodes_tma(cudaStream_t st, int n_mu, int n_v, int n_c, const double* pv, long long ldv,
                           const double* pc, long long ldc, int n_nodes, long long units, const double* dv,
                           const double* dc, const double* gw, const int* seg_base, int ctas,
                           double* partial) {
  // k-tile depth: the deepest of 64 / 48 / 40 / 32 / 24 / 16 among those that pad the two
  // bands least (C60's 120 = 3 x 40, Si216's 432 = 9 x 48)
  auto waste = [&](int bk) { return (n_v + bk - 1) / bk * bk - n_v + (n_c + bk - 1) / bk * bk - n_c; };
  int bk = 16;
  for (int cand : {24, 32, 40, 48, 64})
    if (waste(cand) <= waste(bk)) bk = cand;
  if (const char* v = getenv("LRGW_QUAD_BK")) bk = atoi(v);  // experiments
  CUtensorMap mc, mv;
  if (!tma_encode_mn(&mc, pc, n_mu, n_c, ldc, bk) || !tma_encode_mn(&mv, pv, n_mu, n_v, ldv, bk))
    return cudaErrorNotSupported;
  Quad4Params p;
  p.n_v = n_v;
  p.n_c = n_c;
  p.n_nodes = n_nodes;
  p.units = units;
  p.dv = reinterpret_cast<const double2*>(dv);
  p.dc = reinterpret_cast<const double2*>(dc);
  p.gw = reinterpret_cast<const double2*>(gw);
  p.seg_base = seg_base;
  p.partial = partial;
  switch (bk) {
    case 64: return launch_quad4<64>(st, ctas, mc, mv, p);
    case 48: return launch_quad4<48>(st, ctas, mc, mv, p);
    case 40: return launch_quad4<40>(st, ctas, mc, mv, p);
    case 32: return launch_quad4<32>(st, ctas, mc, mv, p);
    case 24: return launch_quad4<24>(st, ctas, mc, mv, p);
    case 16: return launch_quad4<16>(st, ctas, mc, mv, p);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace lrgw_dev
