// skinny.cu — K7: the probe apply's two passes over Theta (smw.hpp:97-103).
//
//   u = Theta^T x   (N_mu x m, K = N_r)     z = Theta w   (N_r x m, K = N_mu)
//
// with m <= 16 probe columns. Both are HBM-bound streams over Theta
// (N_r x N_mu FP64, 906 MB at Si64); a DMMA tile would waste >90% of its
// columns, so these are coalesced FMA streams: one pass over Theta each,
// the small operand (x chunk / w) staged in shared memory.
#include <cstdint>

#include "kernels.h"

namespace lrgw_dev {

namespace {

constexpr int TN_MU_W = 4;                // Theta columns per warp
constexpr int TN_THREADS = 256;           // 8 warps
constexpr int TN_MU = TN_MU_W * TN_THREADS / 32;  // Theta columns per CTA

// partial[chunk][mu][c] = sum over the chunk's rows of Theta[r, mu] x[r, c].
// Lane = grid row (coalesced 256-byte row segments of each Theta column and
// of x), warp = 4 Theta columns, accumulators in registers over the whole
// row chunk and one warp reduction at the end; x is re-read by the CTA's 8
// warps from L1. Theta is streamed from HBM exactly once.
template <int M>
__global__ void __launch_bounds__(TN_THREADS) tn_kernel(const double* theta, long long ldt, int n_r, int n_mu,
                                                        const double* x, long long ldx, int rows_per_chunk,
                                                        double* partial) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int mu0 = blockIdx.x * TN_MU + warp * TN_MU_W;
  const int r0 = blockIdx.y * rows_per_chunk;
  const int r1 = min(n_r, r0 + rows_per_chunk);
  const double* th[TN_MU_W];
  bool ok[TN_MU_W];
#pragma unroll
  for (int i = 0; i < TN_MU_W; ++i) {
    ok[i] = mu0 + i < n_mu;
    th[i] = theta + (long long)(ok[i] ? mu0 + i : 0) * ldt;
  }
  double acc[TN_MU_W][M];
#pragma unroll
  for (int i = 0; i < TN_MU_W; ++i)
#pragma unroll
    for (int c = 0; c < M; ++c) acc[i][c] = 0.0;
  // pairs of rows per lane (16-byte loads) when the layout allows, then the tail
  const bool vec = ((ldt | ldx | r0) & 1) == 0 && ((reinterpret_cast<uintptr_t>(theta) |
                                                    reinterpret_cast<uintptr_t>(x)) & 15) == 0;
  int r = r0 + 2 * lane;
  if (vec) {
    for (; r + 1 < r1; r += 64) {
      double2 xv[M], tv[TN_MU_W];
#pragma unroll
      for (int c = 0; c < M; ++c) xv[c] = __ldg(reinterpret_cast<const double2*>(x + r + (long long)c * ldx));
#pragma unroll
      for (int i = 0; i < TN_MU_W; ++i)
        tv[i] = ok[i] ? __ldcs(reinterpret_cast<const double2*>(th[i] + r)) : make_double2(0.0, 0.0);
#pragma unroll
      for (int i = 0; i < TN_MU_W; ++i)
#pragma unroll
        for (int c = 0; c < M; ++c) acc[i][c] = fma(tv[i].y, xv[c].y, fma(tv[i].x, xv[c].x, acc[i][c]));
    }
  } else {
    r = r0 + lane;
  }
  for (; r < r1; r += vec ? 64 : 32) {  // scalar rows (the odd tail, or an unaligned layout)
    const int rr = r;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int q = rr + h;
      if (q >= r1 || (!vec && h == 1)) break;
      double xv[M], tv[TN_MU_W];
#pragma unroll
      for (int c = 0; c < M; ++c) xv[c] = __ldg(x + q + (long long)c * ldx);
#pragma unroll
      for (int i = 0; i < TN_MU_W; ++i) tv[i] = ok[i] ? __ldcs(th[i] + q) : 0.0;
#pragma unroll
      for (int i = 0; i < TN_MU_W; ++i)
#pragma unroll
        for (int c = 0; c < M; ++c) acc[i][c] = fma(tv[i], xv[c], acc[i][c]);
    }
  }
#pragma unroll
  for (int i = 0; i < TN_MU_W; ++i)
#pragma unroll
    for (int c = 0; c < M; ++c) {
      double v = acc[i][c];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
      if (lane == 0 && ok[i]) partial[((long long)blockIdx.y * n_mu + mu0 + i) * M + c] = v;
    }
}

template <int M>
__global__ void tn_reduce_kernel(const double* partial, int chunks, int n_mu, double* u, long long ldu) {
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < n_mu * M; idx += gridDim.x * blockDim.x) {
    double v = 0.0;
    for (int ch = 0; ch < chunks; ++ch) v += partial[(long long)ch * n_mu * M + idx];
    const int mu = idx / M, c = idx % M;
    u[mu + (long long)c * ldu] = v;
  }
}

// z[r, c] = sum_mu Theta[r, mu] w[mu, c]; w (n_mu x M) staged in shared memory.
template <int M>
__global__ void __launch_bounds__(256) nn_kernel(const double* theta, long long ldt, int n_r, int n_mu,
                                                 const double* w, long long ldw, double* z, long long ldz) {
  extern __shared__ double ws[];  // n_mu x M, row-major (ws[mu * M + c])
  for (int idx = threadIdx.x; idx < n_mu * M; idx += blockDim.x) {
    const int mu = idx / M, c = idx % M;
    ws[idx] = w[mu + (long long)c * ldw];
  }
  __syncthreads();
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n_r; r += gridDim.x * blockDim.x) {
    double acc[M];
#pragma unroll
    for (int c = 0; c < M; ++c) acc[c] = 0.0;
    int mu = 0;
    for (; mu + 4 <= n_mu; mu += 4) {
      double th[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) th[u] = __ldg(theta + r + (long long)(mu + u) * ldt);
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int c = 0; c < M; ++c) acc[c] = fma(th[u], ws[(mu + u) * M + c], acc[c]);
    }
    for (; mu < n_mu; ++mu) {
      const double th = __ldg(theta + r + (long long)mu * ldt);
#pragma unroll
      for (int c = 0; c < M; ++c) acc[c] = fma(th, ws[mu * M + c], acc[c]);
    }
#pragma unroll
    for (int c = 0; c < M; ++c) z[r + (long long)c * ldz] = acc[c];
  }
}

template <int M>
cudaError_t tn_launch(cudaStream_t st, const double* theta, long long ldt, int n_r, int n_mu, const double* x,
                      long long ldx, double* u, long long ldu, double* work, size_t work_elems, int sm_count) {
  const int mus = (n_mu + TN_MU - 1) / TN_MU;
  // ~8 resident CTAs per SM, bounded by the workspace
  int chunks = std::max(1, (8 * sm_count + mus - 1) / mus);
  while (chunks > 1 && (size_t)chunks * n_mu * M > work_elems) --chunks;
  const int rows = (n_r + chunks - 1) / chunks;
  chunks = (n_r + rows - 1) / rows;
  tn_kernel<M><<<dim3(mus, chunks), TN_THREADS, 0, st>>>(theta, ldt, n_r, n_mu, x, ldx, rows, work);
  count_launches(1);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  tn_reduce_kernel<M><<<(n_mu * M + 255) / 256, 256, 0, st>>>(work, chunks, n_mu, u, ldu);
  count_launches(1);
  return cudaGetLastError();
}

template <int M>
cudaError_t nn_launch(cudaStream_t st, const double* theta, long long ldt, int n_r, int n_mu, const double* w,
                      long long ldw, double* z, long long ldz, int sm_count) {
  const size_t smem = (size_t)n_mu * M * sizeof(double);
  if (smem > 200 * 1024) return cudaErrorInvalidConfiguration;
  cudaFuncSetAttribute(nn_kernel<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int blocks = std::min((n_r + 255) / 256, 4 * sm_count);
  nn_kernel<M><<<blocks, 256, smem, st>>>(theta, ldt, n_r, n_mu, w, ldw, z, ldz);
  count_launches(1);
  return cudaGetLastError();
}

}  // namespace

bool skinny_supported(int m) { return m == 1 || m == 2 || m == 4 || m == 8; }

cudaError_t skinny_tn(cudaStream_t st, const double* theta, long long ldt, int n_r, int n_mu, const double* x,
                      long long ldx, int m, double* u, long long ldu, double* work, size_t work_elems, int sm_count) {
  switch (m) {
    case 1: return tn_launch<1>(st, theta, ldt, n_r, n_mu, x, ldx, u, ldu, work, work_elems, sm_count);
    case 2: return tn_launch<2>(st, theta, ldt, n_r, n_mu, x, ldx, u, ldu, work, work_elems, sm_count);
    case 4: return tn_launch<4>(st, theta, ldt, n_r, n_mu, x, ldx, u, ldu, work, work_elems, sm_count);
    case 8: return tn_launch<8>(st, theta, ldt, n_r, n_mu, x, ldx, u, ldu, work, work_elems, sm_count);
    case 16: return tn_launch<16>(st, theta, ldt, n_r, n_mu, x, ldx, u, ldu, work, work_elems, sm_count);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t skinny_nn(cudaStream_t st, const double* theta, long long ldt, int n_r, int n_mu, const double* w,
                      long long ldw, int m, double* z, long long ldz, int sm_count) {
  switch (m) {
    case 1: return nn_launch<1>(st, theta, ldt, n_r, n_mu, w, ldw, z, ldz, sm_count);
    case 2: return nn_launch<2>(st, theta, ldt, n_r, n_mu, w, ldw, z, ldz, sm_count);
    case 4: return nn_launch<4>(st, theta, ldt, n_r, n_mu, w, ldw, z, ldz, sm_count);
    case 8: return nn_launch<8>(st, theta, ldt, n_r, n_mu, w, ldw, z, ldz, sm_count);
    case 16: return nn_launch<16>(st, theta, ldt, n_r, n_mu, w, ldw, z, ldz, sm_count);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace lrgw_dev
