// skinny.cu — K7: the probe apply's two passes over Theta (smw.hpp:97-103).
//
//   u = Theta^T x   (N_mu x m, K = N_r)     z = Theta w   (N_r x m, K = N_mu)
//
// with m <= 16 probe columns. Both are HBM-bound streams over Theta
// (N_r x N_mu FP64, 906 MB at Si64); a DMMA tile would waste >90% of its
// columns, so these are coalesced FMA streams: one pass over Theta each,
// the small operand (x chunk / w) staged in shared memory.
#include <cstdint>

#include <cstdlib>

#include "gemm4.cuh"
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

// Bulk-copy variant of tn_kernel: a producer warp streams 128-row stages of
// the CTA's 32 Theta columns and of x into a 4-deep shared-memory ring with
// 1-D cp.async.bulk copies (1 KB per column segment) completing on "full"
// mbarriers; the 8 consumer warps release slots through "empty" mbarriers.
// The bytes in flight per SM are bounded by shared memory (~190 KB) instead
// of by the registers the load-to-use version can hold (~32 KB, which capped
// it at ~3.4 TB/s). Needs 16-byte aligned columns (even n_r, ldt, ldx).
constexpr int TB_S = 2;       // stages
constexpr int TB_W = 4;       // Theta columns per consumer warp
constexpr int TB_CN = 16;     // Theta columns per CTA
constexpr int TB_PARTS = TN_THREADS / 32 / (TB_CN / TB_W);  // warps sharing a column group
template <int M>
struct TbCfg {
  static constexpr int R = M <= 8 ? 512 : 256;      // rows per stage (4 KB / 2 KB column segments)
  static constexpr int TH = TB_CN * R;            // Theta doubles per stage
  static constexpr int ST = TH + M * R;           // doubles per stage
  static constexpr int SMEM = TB_S * ST * 8 + 2 * TB_S * 8;
};

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

template <int M>
__global__ void __launch_bounds__(TN_THREADS + 32) tn_bulk_kernel(const double* theta, long long ldt, int n_r,
                                                                  int n_mu, const double* x, long long ldx,
                                                                  int rows_per_chunk, double* partial) {
  using C = TbCfg<M>;
  extern __shared__ __align__(128) double tb_smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(tb_smem + TB_S * C::ST);
  uint64_t* empty = full + TB_S;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int mub = blockIdx.x * TB_CN;
  const int ncol = min(TB_CN, n_mu - mub);
  const int r0 = blockIdx.y * rows_per_chunk;
  const int r1 = min(n_r, r0 + rows_per_chunk);
  const int nst = (r1 - r0 + C::R - 1) / C::R;
  if (threadIdx.x == 0) {
    for (int s = 0; s < TB_S; ++s) mbar_init(full + s, 1), mbar_init(empty + s, TN_THREADS / 32);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (warp == TN_THREADS / 32) {  // producer warp: lane i copies column segment i
    for (int k = 0; k < nst; ++k) {
      const int s = k % TB_S;
      if (k >= TB_S) mbar_wait(empty + s, (unsigned)(((k / TB_S) - 1) & 1));
      const int rb = r0 + k * C::R, nrow = min(C::R, r1 - rb);
      double* buf = tb_smem + s * C::ST;
      if (lane == 0) mbar_arrive_expect_tx(full + s, (unsigned)((ncol + M) * nrow * 8));
      __syncwarp();
      if (lane < ncol) bulk_g2s(buf + lane * C::R, theta + rb + (long long)(mub + lane) * ldt, nrow * 8, full + s);
      if (lane < M) bulk_g2s(buf + C::TH + lane * C::R, x + rb + (long long)lane * ldx, nrow * 8, full + s);
    }
    return;
  }
  const int c0 = (warp % (TB_CN / TB_W)) * TB_W, part = warp / (TB_CN / TB_W);
  bool ok[TB_W];
#pragma unroll
  for (int i = 0; i < TB_W; ++i) ok[i] = c0 + i < ncol;
  double acc[TB_W][M];
#pragma unroll
  for (int i = 0; i < TB_W; ++i)
#pragma unroll
    for (int c = 0; c < M; ++c) acc[i][c] = 0.0;
  for (int k = 0; k < nst; ++k) {
    const int s = k % TB_S;
    const int nrow = min(C::R, r1 - (r0 + k * C::R));
    const double* buf = tb_smem + s * C::ST;
    mbar_wait(full + s, (unsigned)((k / TB_S) & 1));
    // the previous stage goes back only now: an arrive right behind the
    // stage's own loads lets the refill race them (gemm4.cuh:release_prev)
    if (k > 0) {
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + (k - 1) % TB_S);
    }
    for (int q = 2 * lane + 64 * part; q < nrow; q += 64 * TB_PARTS) {
      double2 tv[TB_W];
#pragma unroll
      for (int i = 0; i < TB_W; ++i)
        tv[i] = ok[i] ? *reinterpret_cast<const double2*>(buf + (c0 + i) * C::R + q) : make_double2(0.0, 0.0);
#pragma unroll
      for (int c = 0; c < M; ++c) {
        const double2 xv = *reinterpret_cast<const double2*>(buf + C::TH + c * C::R + q);
#pragma unroll
        for (int i = 0; i < TB_W; ++i) acc[i][c] = fma(tv[i].y, xv.y, fma(tv[i].x, xv.x, acc[i][c]));
      }
    }
  }
#pragma unroll
  for (int i = 0; i < TB_W; ++i)
#pragma unroll
    for (int c = 0; c < M; ++c) {
      double v = acc[i][c];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
      if (lane == 0 && ok[i]) partial[(((long long)blockIdx.y * TB_PARTS + part) * n_mu + mub + c0 + i) * M + c] = v;
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
    // 8 Theta loads in flight per thread (HBM-latency bound at 4)
    for (; mu + 8 <= n_mu; mu += 8) {
      double th[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) th[u] = __ldcs(theta + r + (long long)(mu + u) * ldt);
#pragma unroll
      for (int u = 0; u < 8; ++u)
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

// Bulk-copy variant of nn_kernel: a CTA owns 256 grid rows (one per consumer
// thread); a producer warp streams the
// Theta columns through a 2-deep ring of 32-column x 256-row stages (2 KB
// column segments) with 1-D cp.async.bulk copies; w sits in shared memory.
constexpr int NB_R = 256, NB_S = 2, NB_CONS = NB_R;  // rows per CTA, stages, consumer threads (1 row each)
template <int M>
struct NbCfg {
  static constexpr int CN = M <= 8 ? 32 : 16;   // Theta columns per stage
  static constexpr int ST = CN * NB_R;          // doubles per stage
  static size_t smem(int n_mu) { return (size_t)NB_S * ST * 8 + 2 * NB_S * 8 + (size_t)n_mu * M * 8; }
};

template <int M>
__global__ void __launch_bounds__(NB_CONS + 32) nn_bulk_kernel(const double* theta, long long ldt, int n_r, int n_mu,
                                                               const double* w, long long ldw, double* z,
                                                               long long ldz) {
  using C = NbCfg<M>;
  extern __shared__ __align__(128) double nb_smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(nb_smem + NB_S * C::ST);
  uint64_t* empty = full + NB_S;
  double* ws = reinterpret_cast<double*>(empty + NB_S);  // n_mu x M, row-major
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int rb = blockIdx.x * NB_R, nrow = min(NB_R, n_r - rb);
  const int nst = (n_mu + C::CN - 1) / C::CN;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NB_S; ++s) mbar_init(full + s, 1), mbar_init(empty + s, NB_CONS / 32);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (warp == NB_CONS / 32) {  // producer warp: lane j copies column segment j of the stage
    for (int k = 0; k < nst; ++k) {
      const int s = k % NB_S, mu0 = k * C::CN, ncol = min(C::CN, n_mu - mu0);
      if (k >= NB_S) mbar_wait(empty + s, (unsigned)(((k / NB_S) - 1) & 1));
      if (lane == 0) mbar_arrive_expect_tx(full + s, (unsigned)(ncol * nrow * 8));
      __syncwarp();
      if (lane < ncol)
        bulk_g2s(nb_smem + s * C::ST + lane * NB_R, theta + rb + (long long)(mu0 + lane) * ldt, nrow * 8, full + s);
    }
    return;
  }
  for (int idx = threadIdx.x; idx < n_mu * M; idx += NB_CONS) {
    const int mu = idx / M, c = idx % M;
    ws[idx] = w[mu + (long long)c * ldw];
  }
  asm volatile("bar.sync 1, %0;\n" ::"n"(NB_CONS));  // consumers only
  const int q = threadIdx.x;
  double a0[M];
#pragma unroll
  for (int c = 0; c < M; ++c) a0[c] = 0.0;
  for (int k = 0; k < nst; ++k) {
    const int s = k % NB_S, mu0 = k * C::CN, ncol = min(C::CN, n_mu - mu0);
    const double* buf = nb_smem + s * C::ST;
    mbar_wait(full + s, (unsigned)((k / NB_S) & 1));
    if (k > 0) {  // deferred release, as in tn_bulk_kernel
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + (k - 1) % NB_S);
    }
    if (q < nrow) {
#pragma unroll 8
      for (int j = 0; j < ncol; ++j) {
        const double tv = buf[j * NB_R + q];
        const double* wv = ws + (mu0 + j) * M;
#pragma unroll
        for (int c = 0; c < M; ++c) a0[c] = fma(tv, wv[c], a0[c]);
      }
    }
  }
  if (q < nrow) {
#pragma unroll
    for (int c = 0; c < M; ++c) z[rb + q + (long long)c * ldz] = a0[c];
  }
}

template <int M>
cudaError_t tn_launch(cudaStream_t st, const double* theta, long long ldt, int n_r, int n_mu, const double* x,
                      long long ldx, double* u, long long ldu, double* work, size_t work_elems, int sm_count) {
  int mus = (n_mu + TN_MU - 1) / TN_MU;
  int chunks, parts = 1;
  const char* env = std::getenv("LRGW_TN_BULK");  // 0: the load-to-use kernel
  const bool bulk = !(env && env[0] == '0') && ((ldt | ldx | n_r) & 1) == 0 &&
                    ((reinterpret_cast<uintptr_t>(theta) | reinterpret_cast<uintptr_t>(x)) & 15) == 0;
  if (bulk) {
    // whole waves of the resident CTAs, chunks a multiple of the stage rows
    mus = (n_mu + TB_CN - 1) / TB_CN;
    parts = TB_PARTS;
    int per_sm = 0;
    cudaFuncSetAttribute(tn_bulk_kernel<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, TbCfg<M>::SMEM);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tn_bulk_kernel<M>, TN_THREADS + 32, TbCfg<M>::SMEM);
    const int slots = std::max(1, per_sm) * sm_count;
    int best = 1;
    double best_eff = -1.0;
    for (int ch = std::max(1, slots / mus); ch <= std::max(1, 4 * slots / mus); ++ch) {
      const long long tiles = (long long)mus * ch;
      const double eff = (double)tiles / ((double)((tiles + slots - 1) / slots) * slots);
      if (eff > best_eff + 0.02) best_eff = eff, best = ch;
    }
    chunks = best;
    while (chunks > 1 && (size_t)chunks * parts * n_mu * M > work_elems) --chunks;
    int rows = (n_r + chunks - 1) / chunks;
    rows = (rows + TbCfg<M>::R - 1) / TbCfg<M>::R * TbCfg<M>::R;
    chunks = (n_r + rows - 1) / rows;
    tn_bulk_kernel<M><<<dim3(mus, chunks), TN_THREADS + 32, TbCfg<M>::SMEM, st>>>(theta, ldt, n_r, n_mu, x, ldx, rows,
                                                                            work);
  } else {
    // ~8 resident CTAs per SM, bounded by the workspace
    chunks = std::max(1, (8 * sm_count + mus - 1) / mus);
    while (chunks > 1 && (size_t)chunks * n_mu * M > work_elems) --chunks;
    const int rows = (n_r + chunks - 1) / chunks;
    chunks = (n_r + rows - 1) / rows;
    tn_kernel<M><<<dim3(mus, chunks), TN_THREADS, 0, st>>>(theta, ldt, n_r, n_mu, x, ldx, rows, work);
  }
  count_launches(1);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  tn_reduce_kernel<M><<<(n_mu * M + 255) / 256, 256, 0, st>>>(work, chunks * parts, n_mu, u, ldu);
  count_launches(1);
  return cudaGetLastError();
}

template <int M>
cudaError_t nn_launch(cudaStream_t st, const double* theta, long long ldt, int n_r, int n_mu, const double* w,
                      long long ldw, double* z, long long ldz, int sm_count) {
  {
    const char* env = std::getenv("LRGW_NN_BULK");  // 0: the load-to-use kernel
    const size_t smem = NbCfg<M>::smem(n_mu);
    if (!(env && env[0] == '0') && ((ldt | n_r) & 1) == 0 && (reinterpret_cast<uintptr_t>(theta) & 15) == 0 &&
        smem <= 227 * 1024) {
      cudaFuncSetAttribute(nn_bulk_kernel<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      nn_bulk_kernel<M><<<(n_r + NB_R - 1) / NB_R, NB_CONS + 32, smem, st>>>(theta, ldt, n_r, n_mu, w, ldw, z, ldz);
      count_launches(1);
      return cudaGetLastError();
    }
  }
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
