// trtri.cu — in-place inverse of a lower-triangular N x N matrix (N_mu-sized
// leaves of the fit and of the SMW core, isdf.hpp:143 / smw.hpp:61).
//
// Recursive 2 x 2 blocking on the DMMA GEMM engine:
//   [L11  0 ]^-1   [ X11            0  ]
//   [L21 L22]    = [ -X22 L21 X11   X22 ],
// bottom-up from 64 x 64 diagonal leaves inverted one CTA each (32 x 32
// diagonal blocks by one warp per block — lane = column, unrolled forward
// substitution with reciprocal pivots — then the leaf's block rows), then
// levels 64, 128, ... with two (batched) GEMMs per level. log2(N / 64) levels,
// all compute on tensor cores; replaces cuSOLVER's trsm / trmm cascade.
#include <cfloat>

#include "common.cuh"
#include "kernels.h"

namespace lrgw_dev {

namespace {

constexpr int LEAF = 64;
constexpr int LEAF_THREADS = 512;

// One CTA per diagonal leaf q: a[q LEAF + i, q LEAF + j] (size nb <= LEAF).
// `bad` receives (first zero pivot + 1) if any.
__global__ void __launch_bounds__(LEAF_THREADS) trtri_leaf_kernel(double* a, int n, long long lda, int* bad) {
  extern __shared__ __align__(16) double sm[];
  double* X = sm;                          // LEAF x (LEAF + 1), row-major [i][m]
  double* Lp = X + LEAF * (LEAF + 1);       // packed lower L: (i, m) at i (i + 1) / 2 + m
  __shared__ double rdiag[LEAF];
  __shared__ double P[3 * 32 * 32];
  const int o = blockIdx.x * LEAF;
  const int nb = min(LEAF, n - o);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  constexpr int LP = LEAF + 1;
  // identity padding beyond nb keeps the block arithmetic uniform
  for (int idx = tid; idx < LEAF * LEAF; idx += blockDim.x) {
    const int i = idx % LEAF, m = idx / LEAF;  // column-major walk: coalesced reads
    double v;
    if (i < nb && m < nb)
      v = m <= i ? a[(o + i) + (long long)(o + m) * lda] : 0.0;
    else
      v = i == m ? 1.0 : 0.0;
    if (m <= i) Lp[i * (i + 1) / 2 + m] = v;
    X[i * LP + m] = 0.0;
  }
  __syncthreads();
  for (int i = tid; i < LEAF; i += blockDim.x) {
    const double d = Lp[i * (i + 1) / 2 + i];
    rdiag[i] = d != 0.0 ? 1.0 / d : 0.0;
    if (d == 0.0 && i < nb) atomicMin(bad, o + i + 1);
  }
  __syncthreads();
  const int nblk = (nb + 31) / 32;
  // diagonal 32 x 32 blocks: warp w inverts block w (lane j: column 32 w + j)
  if (wid < nblk) {
    const int b0 = 32 * wid;
    double x[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      double acc = (i == lane) ? 1.0 : 0.0;
#pragma unroll
      for (int m = 0; m < i; ++m) acc = fma(-Lp[(b0 + i) * (b0 + i + 1) / 2 + b0 + m], x[m], acc);
      x[i] = (i >= lane) ? acc * rdiag[b0 + i] : 0.0;
    }
#pragma unroll
    for (int i = 0; i < 32; ++i) X[(b0 + i) * LP + b0 + lane] = x[i];
  }
  __syncthreads();
  // block rows I: X_Ik = -X_II sum_{m=32k}^{32I-1} L_Im X_mk (k < I)
  for (int I = 1; I < nblk; ++I) {
    for (int idx = tid; idx < I * 1024; idx += blockDim.x) {
      const int k = idx / 1024, i = (idx / 32) % 32, j = idx % 32;
      double acc = 0.0;
      const double* li = Lp + (32 * I + i) * (32 * I + i + 1) / 2;
      for (int m = 32 * k + j; m < 32 * I; ++m) acc = fma(li[m], X[m * LP + 32 * k + j], acc);
      P[idx] = acc;
    }
    __syncthreads();
    for (int idx = tid; idx < I * 1024; idx += blockDim.x) {
      const int k = idx / 1024, i = (idx / 32) % 32, j = idx % 32;
      double acc = 0.0;
      for (int q = 0; q <= i; ++q) acc = fma(X[(32 * I + i) * LP + 32 * I + q], P[k * 1024 + q * 32 + j], acc);
      X[(32 * I + i) * LP + 32 * k + j] = -acc;
    }
    __syncthreads();
  }
  for (int idx = tid; idx < nb * nb; idx += blockDim.x) {
    const int i = idx % nb, m = idx / nb;
    if (m <= i) a[(o + i) + (long long)(o + m) * lda] = X[i * LP + m];
  }
}

// dst = lower triangle of src (strict upper of dst zeroed) or, back, only the
// lower triangle of dst overwritten.
__global__ void tril_copy_kernel(const double* src, long long lds, double* dst, long long ldd, int n, int zero_upper) {
  const long long total = (long long)n * n;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int r = static_cast<int>(idx % n), c = static_cast<int>(idx / n);
    if (r >= c)
      dst[r + c * ldd] = src[r + c * lds];
    else if (zero_upper)
      dst[r + c * ldd] = 0.0;
  }
}

}  // namespace

size_t trtri_work_elems(int n) { return 2 * (size_t)n * n + 64; }

cudaError_t trtri_lower(cudaStream_t st, double* a_in, int n, long long lda_in, double* work, int* bad,
                        int sm_count) {
  if (n <= 0) return cudaSuccess;
  // operate on a zero-upper copy: the GEMM levels stream the triangular
  // blocks densely (the caller's strict upper triangle stays untouched)
  double* a = work;
  const long long lda = n;
  work += (size_t)n * n;
  tril_copy_kernel<<<592, 256, 0, st>>>(a_in, lda_in, a, lda, n, 1); count_launches(1);
  const int leaves = (n + LEAF - 1) / LEAF;
  const size_t smem = ((size_t)LEAF * (LEAF + 1) + (size_t)LEAF * (LEAF + 1) / 2) * sizeof(double);
  cudaError_t e = cudaFuncSetAttribute(trtri_leaf_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  trtri_leaf_kernel<<<leaves, LEAF_THREADS, smem, st>>>(a, n, lda, bad); count_launches(1);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  // levels: pairs of inverted b-blocks become inverted 2b-blocks; the full
  // pairs of a level are independent and run as ONE batched launch per
  // product (the small levels are latency-bound: 8 + 4 launches of 12-19 us
  // at N_mu 1024 become 2 + 2), a ragged last pair separately
  for (int b = LEAF; b < n; b *= 2) {
    const long long step = 2LL * b * (lda + 1);  // pair to pair along the diagonal
    int full = 0;
    while ((full + 1) * 2 * b <= n) ++full;      // pairs with b2 == b
    if (full > 0) {
      double* x11 = a;
      double* l21 = a + b;
      double* x22 = a + b + (long long)b * lda;
      // T_z = L21_z X11_z (b x b), X11 lower: B(n, k) = X11(k, n) is zero for k < n
      e = dgemm_batched(st, full, b, b, b, l21, lda, step, Lay::MN, x11, lda, step, Lay::K, work, b, (long long)b * b,
                        1.0, 0.0, true);
      if (e != cudaSuccess) return e;
      // X21_z = -X22_z T_z
      e = dgemm_batched(st, full, b, b, b, x22, lda, step, Lay::MN, work, b, (long long)b * b, Lay::K, l21, lda, step,
                        -1.0, 0.0, false);
      if (e != cudaSuccess) return e;
    }
    const int r0 = full * 2 * b;
    if (r0 + b < n) {  // the ragged pair (b2 < b)
      const int r1 = r0 + b, b2 = n - r1;
      double* x11 = a + r0 + (long long)r0 * lda;
      double* l21 = a + r1 + (long long)r0 * lda;
      double* x22 = a + r1 + (long long)r1 * lda;
      e = dgemm(st, b2, b, b, l21, lda, Lay::MN, x11, lda, Lay::K, work, b2, 1.0, 0.0, nullptr, false, sm_count,
                nullptr, 0, true);
      if (e != cudaSuccess) return e;
      e = dgemm(st, b2, b, b2, x22, lda, Lay::MN, work, b2, Lay::K, l21, lda, -1.0, 0.0, nullptr, false, sm_count,
                nullptr, 0);
      if (e != cudaSuccess) return e;
    }
  }
  tril_copy_kernel<<<592, 256, 0, st>>>(a, lda, a_in, lda_in, n, 0); count_launches(1);
  return cudaGetLastError();
}

}  // namespace lrgw_dev
