// sigma.cu — the Hadamard-form static-COHSEX self-energy diagonals
// (reference gw.hpp:93-137, detail::hadamard_diag / sigma_hadamard):
//
//   d[n] = Psi(:, n)^T (H o M) Psi(:, n),   M = Psi_o Psi_o^T,
//
// at the ISDF points (Psi = rows of the orbitals at the vn or nn points). The
// mask M and the product (H o M) Psi are DMMA GEMMs (gemm.cu); the Hadamard
// with H is applied in place on the mask (one streaming pass over an N_mu^2
// block), and the per-band column dot is one warp per band with a fixed
// lane-strided order and a shuffle tree (deterministic, no atomics).
#include "kernels.h"

namespace lrgw_dev {

namespace {

__global__ void hadamard_inplace_kernel(int n, const double* __restrict__ h, long long ldh, double* m,
                                        long long ldm) {
  const long long total = (long long)n * n;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int r = static_cast<int>(idx % n), c = static_cast<int>(idx / n);
    m[r + c * ldm] *= h[r + c * ldh];
  }
}

// out[j] = alpha * sum_i a(i, j) b(i, j); one warp per column.
__global__ void col_dot_kernel(int rows, int cols, const double* __restrict__ a, long long lda,
                               const double* __restrict__ b, long long ldb, double alpha, double* out) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= cols) return;
  const double* ac = a + (long long)warp * lda;
  const double* bc = b + (long long)warp * ldb;
  double s = 0.0;
  for (int i = lane; i < rows; i += 32) s = fma(ac[i], bc[i], s);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) out[warp] = alpha * s;
}

}  // namespace

cudaError_t hadamard_inplace(cudaStream_t st, int n, const double* h, long long ldh, double* m, long long ldm) {
  if (n <= 0) return cudaSuccess;
  const long long total = (long long)n * n;
  const int blocks = static_cast<int>(std::min<long long>((total + 255) / 256, 148 * 8));
  hadamard_inplace_kernel<<<blocks, 256, 0, st>>>(n, h, ldh, m, ldm);
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t col_dot(cudaStream_t st, int rows, int cols, const double* a, long long lda, const double* b,
                    long long ldb, double alpha, double* out) {
  if (cols <= 0) return cudaSuccess;
  col_dot_kernel<<<(cols + 7) / 8, 256, 0, st>>>(rows, cols, a, lda, b, ldb, alpha, out);
  count_launches(1);
  return cudaGetLastError();
}

}  // namespace lrgw_dev
