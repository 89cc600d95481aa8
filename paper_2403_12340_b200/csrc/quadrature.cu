// quadrature.cu — K3: fused Cauchy-quadrature / Hadamard FP64 DMMA kernel.
//
// Replaces contour_node_term + sum_node_terms (contour.hpp:144-222). For every
// lower-triangle 64x64 tile of T and every quadrature node k of its node group:
//   Jc = Phi_c,mu diag(1/(z_k - e_c)) Phi_c,mu^T      (complex: re, im parts)
//   Jv = Phi_v,mu diag(1/(z_k - e_v)) Phi_v,mu^T
//   acc += (w g)_re * Im(Jv o Jc) + (w g)_im * Re(Jv o Jc)
// with the diagonal scaling fused into the B-fragment load and the complex
// Hadamard + weighted node accumulation fused into the epilogue, so no
// N_mu x N_mu intermediate of any node ever reaches HBM. The complex product is
// refactored as Jv_re o P1 + Jv_im o P2 with P1 = (wg)_re Jc_im + (wg)_im Jc_re,
// P2 = (wg)_re Jc_re - (wg)_im Jc_im, so 5 accumulator tiles are live.
// Persistent schedule: the (tile, node) work units, tile-major, are cut into
// one contiguous run per SM; each CTA streams its run's operand k-tiles
// through a 4-stage cp.async ring over the flattened (unit, {c, v}, k-tile)
// sequence (the pipeline never drains at node or tile boundaries) and writes
// one 64 x 64 partial per tile segment it touches; a fixed-order reduction
// sums the segments of each tile. Phi_mu panels are L2-resident (2 MB at Si64).
//
// This file holds the schedule (quad_plan), the reduction and the cp.async
// feed of the node kernel; quad_nodes runs the node kernel on the TMA feed
// (quad4.cu: same schedule, partial layout and node order) whenever the
// Phi_mu panels qualify for a tensor map (16-byte aligned base, even leading
// dimension) and keeps the cp.async kernel below for the rest.
#include <algorithm>
#include <type_traits>
#include <vector>

#include "common.cuh"
#include "kernels.h"

namespace lrgw_dev {

namespace {

constexpr int QBM = 64;
constexpr int QWM = 32, QWN = 16;                      // warp tile
constexpr int QWARPS_M = QBM / QWM, QWARPS_N = QBM / QWN;  // 2 x 4
constexpr int QTHREADS = 32 * QWARPS_M * QWARPS_N;     // 256
constexpr int QFM = QWM / 8, QFN = QWN / 8;            // 4 x 2 fragments
constexpr int QPITCH = QBM + 4;                        // conflict-free pitch (doubles)
// k-tile depth: 64 (3-stage ring) when both bands reach it, else 32 / 16 (4 stages)
template <int BK>
struct QK {
  static constexpr int QBK = BK, QSTAGES = BK >= 64 ? 3 : 4;
  static constexpr int QTILE = QBK * QPITCH;
  static constexpr int QSTAGE_ELEMS = 2 * QTILE + 2 * QBK;  // + the k-tile's complex diagonal
  static constexpr int QSMEM = QSTAGES * QSTAGE_ELEMS * 8;
};

struct QuadParams {
  int n_mu, n_v, n_c;
  const double* pv;
  long long ldv;
  const double* pc;
  long long ldc;
  int n_nodes;
  long long units;     // tiles x n_nodes
  const double2* dv;   // [node][n_v]
  const double2* dc;   // [node][n_c]
  const double2* gw;   // [node]
  const int* seg_base; // [cta]: first partial slot of the CTA
  double* partial;     // [slot][QBM * QBM]
};

// Work run of CTA c: units [u0, u1).
__host__ __device__ __forceinline__ long long quad_run_begin(long long units, int ctas, int c) {
  return units * c / ctas;
}

template <int VEC, int QBK>
__device__ __forceinline__ void load_panel(double* s, const double* g, long long ld, int row0,
                                           int rows, int k0, int kend, int tid) {
  constexpr int CHUNKS = QBM * QBK / VEC;
#pragma unroll
  for (int i = 0; i < CHUNKS / QTHREADS; ++i) {
    const int c = tid + i * QTHREADS;
    const int k = c / (QBM / VEC);
    const int r = (c % (QBM / VEC)) * VEC;
    const int gr = row0 + r, gk = k0 + k;
    const bool ok = gr < rows && gk < kend;
    const double* src = ok ? g + gr + (long long)gk * ld : g;
    if (VEC == 2)
      cp_async16(s + k * QPITCH + r, src, ok);
    else
      cp_async8(s + k * QPITCH + r, src, ok);
  }
}

template <int VEC, int BK>
__global__ void __launch_bounds__(QTHREADS, 1) quad_kernel(QuadParams p) {
  extern __shared__ __align__(16) double smem[];
  constexpr int QBK = QK<BK>::QBK, QSTAGES = QK<BK>::QSTAGES, QTILE = QK<BK>::QTILE;
  constexpr int QSTAGE_ELEMS = QK<BK>::QSTAGE_ELEMS;
  const long long u0 = quad_run_begin(p.units, gridDim.x, blockIdx.x);
  const long long u1 = quad_run_begin(p.units, gridDim.x, blockIdx.x + 1);
  if (u1 <= u0) return;
  const int ktc = (p.n_c + QBK - 1) / QBK, ktv = (p.n_v + QBK - 1) / QBK, ktt = ktc + ktv;
  const int total = static_cast<int>(u1 - u0) * ktt;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp % QWARPS_M) * QWM, wn = (warp / QWARPS_M) * QWN;
  const int g = lane >> 2, t = lane & 3;

  // producer cursor (unit = tile * n_nodes + node, k-tile), advanced in order
  int i_tile = static_cast<int>(u0 / p.n_nodes), i_node = static_cast<int>(u0 % p.n_nodes), i_kt = 0;
  int i_tm, i_tn;
  lower_tile(i_tile, i_tm, i_tn);
  auto issue = [&](int j) {
    const int kt = i_kt, node = i_node, tm = i_tm, tn = i_tn;
    if (++i_kt == ktt) {
      i_kt = 0;
      if (++i_node == p.n_nodes) {
        i_node = 0;
        lower_tile(++i_tile, i_tm, i_tn);
      }
    }
    double* s = smem + (j % QSTAGES) * QSTAGE_ELEMS;
    const bool cph = kt < ktc;
    const double* src = cph ? p.pc : p.pv;
    const long long ld = cph ? p.ldc : p.ldv;
    const int k0 = (cph ? kt : kt - ktc) * QBK;
    const int kend = cph ? p.n_c : p.n_v;
    load_panel<VEC, QBK>(s, src, ld, tm * QBM, p.n_mu, k0, kend, tid);
    load_panel<VEC, QBK>(s + QTILE, src, ld, tn * QBM, p.n_mu, k0, kend, tid);
    // the node's diagonal 1/(z_k - e) for this k-tile (zero-filled past the band count)
    if (tid < QBK) {
      const double2* dtab = cph ? p.dc + (long long)node * p.n_c : p.dv + (long long)node * p.n_v;
      const int gk = k0 + tid;
      cp_async16(s + 2 * QTILE + 2 * tid, gk < kend ? dtab + gk : dtab, gk < kend);
    }
  };

  double accR[QFM][QFN][2], accI[QFM][QFN][2], p1[QFM][QFN][2], p2[QFM][QFN][2], tac[QFM][QFN][2];
#pragma unroll
  for (int i = 0; i < QFM; ++i)
#pragma unroll
    for (int j = 0; j < QFN; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) accR[i][j][h] = accI[i][j][h] = tac[i][j][h] = p1[i][j][h] = p2[i][j][h] = 0.0;

#pragma unroll
  for (int s = 0; s < QSTAGES - 1; ++s) {
    if (s < total) issue(s);
    cp_async_commit();
  }

  int slot = p.seg_base[blockIdx.x];
  // consumer cursor
  long long unit = u0;
  int kt = 0, c_node = static_cast<int>(u0 % p.n_nodes);
  for (int j = 0; j < total; ++j) {
    cp_async_wait<QSTAGES - 2>();
    __syncthreads();
    if (j + QSTAGES - 1 < total) issue(j + QSTAGES - 1);
    cp_async_commit();

    const double* sa = smem + (j % QSTAGES) * QSTAGE_ELEMS;
    const double* sb = sa + QTILE;
    const double2* sd = reinterpret_cast<const double2*>(sa + 2 * QTILE);
#pragma unroll
    for (int kk = 0; kk < QBK; kk += 4) {
      const double2 d = sd[kk + t];
      double af[QFM], br[QFN], bi[QFN];
#pragma unroll
      for (int i = 0; i < QFM; ++i) af[i] = sa[(kk + t) * QPITCH + wm + i * 8 + g];
#pragma unroll
      for (int jn = 0; jn < QFN; ++jn) {
        const double b = sb[(kk + t) * QPITCH + wn + jn * 8 + g];
        br[jn] = b * d.x;
        bi[jn] = b * d.y;
      }
#pragma unroll
      for (int i = 0; i < QFM; ++i)
#pragma unroll
        for (int jn = 0; jn < QFN; ++jn) {
          dmma884(accR[i][jn][0], accR[i][jn][1], af[i], br[jn]);
          dmma884(accI[i][jn][0], accI[i][jn][1], af[i], bi[jn]);
        }
    }
    if (kt == ktc - 1) {
      // end of the c phase: fold the node's w*g into the conduction factors
      const double2 wg = __ldg(p.gw + c_node);
#pragma unroll
      for (int i = 0; i < QFM; ++i)
#pragma unroll
        for (int jn = 0; jn < QFN; ++jn)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const double cr = accR[i][jn][h], ci = accI[i][jn][h];
            p1[i][jn][h] = wg.x * ci + wg.y * cr;
            p2[i][jn][h] = wg.x * cr - wg.y * ci;
            accR[i][jn][h] = accI[i][jn][h] = 0.0;
          }
    } else if (kt == ktt - 1) {
      // end of the v phase: weighted complex-Hadamard accumulation
#pragma unroll
      for (int i = 0; i < QFM; ++i)
#pragma unroll
        for (int jn = 0; jn < QFN; ++jn)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            tac[i][jn][h] = fma(accR[i][jn][h], p1[i][jn][h], fma(accI[i][jn][h], p2[i][jn][h], tac[i][jn][h]));
            accR[i][jn][h] = accI[i][jn][h] = 0.0;
          }
      // last node of this CTA's segment of the tile: flush the partial
      if (unit + 1 == u1 || c_node + 1 == p.n_nodes) {
        double* out = p.partial + (long long)slot * QBM * QBM;
#pragma unroll
        for (int i = 0; i < QFM; ++i)
#pragma unroll
          for (int jn = 0; jn < QFN; ++jn) {
            const int m = wm + i * 8 + g, n = wn + jn * 8 + 2 * t;
            *reinterpret_cast<double2*>(out + m * QBM + n) = make_double2(tac[i][jn][0], tac[i][jn][1]);
#pragma unroll
            for (int h = 0; h < 2; ++h) tac[i][jn][h] = 0.0;
          }
        ++slot;
      }
    }
    if (++kt == ktt) {
      kt = 0;
      ++unit;
      if (++c_node == p.n_nodes) c_node = 0;
    }
  }
  cp_async_wait<0>();
}

// running(m,n) = beta * running(m,n) + sum over the tile's segment partials
// (in CTA order, fixed), T(m,n) = T(n,m) = pref * running(m,n)   (m >= n).
__global__ void quad_reduce_kernel(const double* partial, const int* tile_ptr, int n_mu, double* running,
                                   double beta, double pref, double* t, long long ldt) {
  const long long total = (long long)n_mu * n_mu;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int m = static_cast<int>(idx % n_mu), n = static_cast<int>(idx / n_mu);
    if (m < n) continue;
    const int tm = m / QBM, tn = n / QBM, tile = tm * (tm + 1) / 2 + tn;
    const int local = (m % QBM) * QBM + (n % QBM);
    double s = 0.0;
    for (int sl = tile_ptr[tile]; sl < tile_ptr[tile + 1]; ++sl) s += partial[(long long)sl * QBM * QBM + local];
    if (running) {
      s = (beta == 0.0) ? s : beta * running[idx] + s;
      running[idx] = s;
    }
    const double v = pref * s;
    t[m + n * ldt] = v;
    t[n + m * ldt] = v;
  }
}

}  // namespace

namespace {

struct QuadPlan {
  int ctas = 0, slots = 0;
  std::vector<int> seg_base;  // [cta + 1]
  std::vector<int> tile_ptr;  // [tiles + 1] -> slot ranges (slots are tile-major by construction)
};

// Segments of each CTA's contiguous run of (tile, node) units.
QuadPlan quad_plan(int n_mu, int n_nodes, int sm_count) {
  QuadPlan q;
  const int tdim = (n_mu + QBM - 1) / QBM;
  const int tiles = tdim * (tdim + 1) / 2;
  const long long units = (long long)tiles * n_nodes;
  q.ctas = (int)std::min<long long>(units, sm_count);
  q.seg_base.assign(q.ctas + 1, 0);
  q.tile_ptr.assign(tiles + 1, 0);
  std::vector<int> count(tiles, 0);
  for (int c = 0; c < q.ctas; ++c) {
    const long long a = quad_run_begin(units, q.ctas, c), b = quad_run_begin(units, q.ctas, c + 1);
    int segs = 0;
    if (b > a) {
      const long long t0 = a / n_nodes, t1 = (b - 1) / n_nodes;
      segs = (int)(t1 - t0 + 1);
      for (long long tt = t0; tt <= t1; ++tt) ++count[tt];
    }
    q.seg_base[c + 1] = q.seg_base[c] + segs;
  }
  for (int tt = 0; tt < tiles; ++tt) q.tile_ptr[tt + 1] = q.tile_ptr[tt] + count[tt];
  q.slots = q.seg_base[q.ctas];
  return q;
}

}  // namespace

size_t quad_partial_elems(int n_mu, int n_nodes, int sm_count) {
  const QuadPlan q = quad_plan(n_mu, n_nodes, sm_count);
  return (size_t)q.slots * QBM * QBM + 2 * (size_t)(q.ctas + 1) + (q.tile_ptr.size() + 1) / 2 + 2;
}

cudaError_t quad_nodes(cudaStream_t st, int n_mu, int n_v, int n_c, const double* pv, long long ldv,
                       const double* pc, long long ldc, int n_nodes, const double* dv,
                       const double* dc, const double* gw, int sm_count, double* partial,
                       double* running, double beta, double pref, double* t, long long ldt,
                       cudaEvent_t k_begin, cudaEvent_t k_end) {
  if (n_mu <= 0 || n_nodes <= 0) return cudaSuccess;
  const QuadPlan q = quad_plan(n_mu, n_nodes, sm_count);
  // plan tables live after the partial slots in the same workspace
  int* seg_base = reinterpret_cast<int*>(partial + (size_t)q.slots * QBM * QBM);
  int* tile_ptr = seg_base + q.seg_base.size();
  cudaError_t e = cudaMemcpyAsync(seg_base, q.seg_base.data(), q.seg_base.size() * sizeof(int),
                                  cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return e;
  e = cudaMemcpyAsync(tile_ptr, q.tile_ptr.data(), q.tile_ptr.size() * sizeof(int), cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return e;
  QuadParams p;
  p.n_mu = n_mu;
  p.n_v = n_v;
  p.n_c = n_c;
  p.pv = pv;
  p.ldv = ldv;
  p.pc = pc;
  p.ldc = ldc;
  p.n_nodes = n_nodes;
  const int tdim = (n_mu + QBM - 1) / QBM;
  p.units = (long long)(tdim * (tdim + 1) / 2) * n_nodes;
  p.dv = reinterpret_cast<const double2*>(dv);
  p.dc = reinterpret_cast<const double2*>(dc);
  p.gw = reinterpret_cast<const double2*>(gw);
  p.seg_base = seg_base;
  p.partial = partial;
  const bool vec = (n_mu % 2 == 0) && (ldv % 2 == 0) && (ldc % 2 == 0) &&
                   (reinterpret_cast<uintptr_t>(pv) % 16 == 0) &&
                   (reinterpret_cast<uintptr_t>(pc) % 16 == 0);
  if (k_begin) cudaEventRecord(k_begin, st);
  // the TMA feed (quad4.cu) wherever the Phi_mu panels qualify for a tensor map
  bool done = false;
  if (quad_tma_enabled()) {
    e = quad_nodes_tma(st, n_mu, n_v, n_c, pv, ldv, pc, ldc, n_nodes, p.units, dv, dc, gw, seg_base, q.ctas,
                       partial);
    if (e == cudaSuccess)
      done = true;
    else if (e != cudaErrorNotSupported)
      return e;
  }
  auto go = [&](auto vec_c, auto bk_c) {
    constexpr int V = decltype(vec_c)::value, B = decltype(bk_c)::value;
    cudaFuncSetAttribute(quad_kernel<V, B>, cudaFuncAttributeMaxDynamicSharedMemorySize, QK<B>::QSMEM);
    quad_kernel<V, B><<<q.ctas, QTHREADS, QK<B>::QSMEM, st>>>(p);
    count_launches(1);
  };
  using V1 = std::integral_constant<int, 1>;
  using V2 = std::integral_constant<int, 2>;
  const int nb = std::min(n_v, n_c);
  // k-tile depth: the deepest of 64 / 48 / 40 that pads the two bands least
  // (C60's 120 = 3 x 40: no dead k; Si216's 432 = 9 x 48)
  auto waste = [&](int bk) { return (n_v + bk - 1) / bk * bk - n_v + (n_c + bk - 1) / bk * bk - n_c; };
  int bk = 64;
  if (nb >= 40)
    for (int cand : {48, 40})
      if (waste(cand) < waste(bk)) bk = cand;
  if (done) {
  } else if (nb >= 64 && bk == 64) {
    using B = std::integral_constant<int, 64>;
    vec ? go(V2{}, B{}) : go(V1{}, B{});
  } else if (nb >= 48 && bk == 48) {
    using B = std::integral_constant<int, 48>;
    vec ? go(V2{}, B{}) : go(V1{}, B{});
  } else if (nb >= 40 && bk == 40) {
    using B = std::integral_constant<int, 40>;
    vec ? go(V2{}, B{}) : go(V1{}, B{});
  } else if (nb >= 32) {
    using B = std::integral_constant<int, 32>;
    vec ? go(V2{}, B{}) : go(V1{}, B{});
  } else {
    using B = std::integral_constant<int, 16>;
    vec ? go(V2{}, B{}) : go(V1{}, B{});
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (k_end) cudaEventRecord(k_end, st);
  quad_reduce_kernel<<<1184, 256, 0, st>>>(partial, tile_ptr, n_mu, running, beta, pref, t, ldt);
  count_launches(1);
  return cudaGetLastError();
}

}  // namespace lrgw_dev
