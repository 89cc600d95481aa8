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
// Operand k-tiles stream through a 4-stage cp.async ring over the flattened
// (node, {c, v}, k-tile) sequence, so the pipeline never drains at node
// boundaries. Phi_mu panels are L2-resident (2 MB at Si64).
#include "common.cuh"
#include "kernels.h"

namespace lrgw_dev {

namespace {

constexpr int QBM = 64, QBK = 16, QSTAGES = 4;
constexpr int QWM = 32, QWN = 16;                      // warp tile
constexpr int QWARPS_M = QBM / QWM, QWARPS_N = QBM / QWN;  // 2 x 4
constexpr int QTHREADS = 32 * QWARPS_M * QWARPS_N;     // 256
constexpr int QFM = QWM / 8, QFN = QWN / 8;            // 4 x 2 fragments
constexpr int QPITCH = QBM + 4;                        // conflict-free pitch (doubles)
constexpr int QTILE = QBK * QPITCH;
constexpr int QSTAGE_ELEMS = 2 * QTILE + 2 * QBK;  // + the k-tile's complex diagonal
constexpr int QSMEM = QSTAGES * QSTAGE_ELEMS * 8;

struct QuadParams {
  int n_mu, n_v, n_c;
  const double* pv;
  long long ldv;
  const double* pc;
  long long ldc;
  int n_nodes, nodes_per_group;
  const double2* dv;  // [node][n_v]
  const double2* dc;  // [node][n_c]
  const double2* gw;  // [node]
  double* partial;    // [group][n_mu * n_mu]
};

template <int VEC>
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

template <int VEC>
__global__ void __launch_bounds__(QTHREADS, 1) quad_kernel(QuadParams p) {
  extern __shared__ __align__(16) double smem[];
  int tm, tn;
  lower_tile(blockIdx.x, tm, tn);
  const int m0 = tm * QBM, n0 = tn * QBM;
  const int node0 = blockIdx.y * p.nodes_per_group;
  const int nn = min(p.nodes_per_group, p.n_nodes - node0);
  if (nn <= 0) return;
  const int ktc = (p.n_c + QBK - 1) / QBK, ktv = (p.n_v + QBK - 1) / QBK, ktt = ktc + ktv;
  const int total = nn * ktt;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp % QWARPS_M) * QWM, wn = (warp / QWARPS_M) * QWN;
  const int g = lane >> 2, t = lane & 3;

  auto issue = [&](int j) {
    const int kt = j % ktt;
    double* s = smem + (j % QSTAGES) * QSTAGE_ELEMS;
    const bool cph = kt < ktc;
    const double* src = cph ? p.pc : p.pv;
    const long long ld = cph ? p.ldc : p.ldv;
    const int k0 = (cph ? kt : kt - ktc) * QBK;
    const int kend = cph ? p.n_c : p.n_v;
    load_panel<VEC>(s, src, ld, m0, p.n_mu, k0, kend, tid);
    load_panel<VEC>(s + QTILE, src, ld, n0, p.n_mu, k0, kend, tid);
    // the node's diagonal 1/(z_k - e) for this k-tile (zero-filled past the band count)
    if (tid < QBK) {
      const int node = node0 + j / ktt;
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

  for (int j = 0; j < total; ++j) {
    cp_async_wait<QSTAGES - 2>();
    __syncthreads();
    if (j + QSTAGES - 1 < total) issue(j + QSTAGES - 1);
    cp_async_commit();

    const int node = node0 + j / ktt;
    const int kt = j % ktt;
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
      const double2 wg = __ldg(p.gw + node);
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
    }
  }
  cp_async_wait<0>();

  double* out = p.partial + (long long)blockIdx.y * p.n_mu * p.n_mu;
#pragma unroll
  for (int i = 0; i < QFM; ++i)
#pragma unroll
    for (int jn = 0; jn < QFN; ++jn) {
      const int m = m0 + wm + i * 8 + g;
      const int n = n0 + wn + jn * 8 + 2 * t;
      if (m < p.n_mu) {
        if (n < p.n_mu) out[m + (long long)n * p.n_mu] = tac[i][jn][0];
        if (n + 1 < p.n_mu) out[m + (long long)(n + 1) * p.n_mu] = tac[i][jn][1];
      }
    }
}

// running(m,n) = beta * running(m,n) + sum_g partial[g](m,n)   (m >= n)
// T(m,n) = T(n,m) = pref * running(m,n)
__global__ void quad_reduce_kernel(const double* partial, int groups, int n_mu, double* running,
                                   double beta, double pref, double* t, long long ldt) {
  const long long total = (long long)n_mu * n_mu;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int m = static_cast<int>(idx % n_mu), n = static_cast<int>(idx / n_mu);
    if (m < n) continue;
    double s = 0.0;
    for (int gi = 0; gi < groups; ++gi) s += partial[gi * total + idx];
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

int quad_partial_groups(int n_mu, int n_nodes, int sm_count) {
  const int tiles = ((n_mu + QBM - 1) / QBM) * ((n_mu + QBM - 1) / QBM + 1) / 2;
  // one resident 256-thread CTA per SM (register bound); split nodes until
  // the grid covers ~2 waves, never below 4 nodes per group
  int groups = 1;
  while (groups < n_nodes && tiles * groups < 2 * sm_count && (n_nodes + groups) / (groups + 1) >= 4)
    ++groups;
  return groups;
}

cudaError_t quad_nodes(cudaStream_t st, int n_mu, int n_v, int n_c, const double* pv, long long ldv,
                       const double* pc, long long ldc, int n_nodes, const double* dv,
                       const double* dc, const double* gw, int groups, double* partial,
                       double* running, double beta, double pref, double* t, long long ldt) {
  if (n_mu <= 0 || n_nodes <= 0) return cudaSuccess;
  QuadParams p;
  p.n_mu = n_mu;
  p.n_v = n_v;
  p.n_c = n_c;
  p.pv = pv;
  p.ldv = ldv;
  p.pc = pc;
  p.ldc = ldc;
  p.n_nodes = n_nodes;
  p.nodes_per_group = (n_nodes + groups - 1) / groups;
  groups = (n_nodes + p.nodes_per_group - 1) / p.nodes_per_group;
  p.dv = reinterpret_cast<const double2*>(dv);
  p.dc = reinterpret_cast<const double2*>(dc);
  p.gw = reinterpret_cast<const double2*>(gw);
  p.partial = partial;
  const int tdim = (n_mu + QBM - 1) / QBM;
  dim3 grid(tdim * (tdim + 1) / 2, groups);
  const bool vec = (n_mu % 2 == 0) && (ldv % 2 == 0) && (ldc % 2 == 0) &&
                   (reinterpret_cast<uintptr_t>(pv) % 16 == 0) &&
                   (reinterpret_cast<uintptr_t>(pc) % 16 == 0);
  if (vec) {
    cudaFuncSetAttribute(quad_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, QSMEM);
    quad_kernel<2><<<grid, QTHREADS, QSMEM, st>>>(p); count_launches(1);
  } else {
    cudaFuncSetAttribute(quad_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, QSMEM);
    quad_kernel<1><<<grid, QTHREADS, QSMEM, st>>>(p); count_launches(1);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  quad_reduce_kernel<<<1184, 256, 0, st>>>(partial, groups, n_mu, running, beta, pref, t, ldt); count_launches(1);
  return cudaGetLastError();
}

}  // namespace lrgw_dev
