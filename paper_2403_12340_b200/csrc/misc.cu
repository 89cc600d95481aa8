// misc.cu — small elementwise / reduction kernels used around the hot path.
#include <cfloat>
#include <climits>
#include "kernels.h"

namespace lrgw_dev {

namespace {

__global__ void scale_copy_kernel(const double* src, double* dst, size_t n, double alpha) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = alpha * src[i];
}

__global__ void fill_kernel(double* dst, size_t n, double v) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = v;
}

__global__ void add_diag_kernel(double* a, int n, long long lda, double v) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    a[i + i * lda] += v;
}

__global__ void axpby_kernel(int rows, int cols, double alpha, const double* x, long long ldx,
                             double beta, double* y, long long ldy) {
  const long long total = (long long)rows * cols;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int r = static_cast<int>(idx % rows), c = static_cast<int>(idx / rows);
    double* yy = y + r + c * ldy;
    *yy = alpha * x[r + c * ldx] + (beta == 0.0 ? 0.0 : beta * *yy);
  }
}

// Deterministic two-level reductions: fixed grid, per-block partials, one
// final block (no atomics on doubles).
__global__ void max_abs_kernel(const double* x, size_t n, double* partial) {
  __shared__ double s[256];
  double m = 0.0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    m = fmax(m, fabs(x[i]));
  s[threadIdx.x] = m;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) s[threadIdx.x] = fmax(s[threadIdx.x], s[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = s[0];
}

__global__ void sum_sq_diff_kernel(const double* a, const double* b, size_t n, double* partial) {
  __shared__ double s[256];
  double acc = 0.0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const double d = b ? a[i] - b[i] : a[i];
    acc = fma(d, d, acc);
  }
  s[threadIdx.x] = acc;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) s[threadIdx.x] += s[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = s[0];
}

__global__ void finish_kernel(const double* partial, int n, double* out, int is_max) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r = is_max ? fmax(r, partial[i]) : r + partial[i];
    *out = r;
  }
}

__global__ void zero_strict_upper_kernel(double* a, int n, long long lda) {
  const long long total = (long long)n * n;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int i = static_cast<int>(idx % n), j = static_cast<int>(idx / n);
    if (i < j) a[i + j * lda] = 0.0;
  }
}

constexpr int kRedBlocks = 296;

// out (cols x rows, ld ldo) = in^T (rows x cols, ld ldi), 32 x 32 smem tiles.
__global__ void transpose_kernel(const double* in, long long ldi, int rows, int cols, double* out, long long ldo) {
  __shared__ double tile[32][33];
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;  // bx: column block of in, by: row block of in
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    const int r = by + threadIdx.x, c = bx + j;
    if (r < rows && c < cols) tile[j][threadIdx.x] = in[r + (long long)c * ldi];
  }
  __syncthreads();
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    const int r = bx + threadIdx.x, c = by + j;  // out(r, c) = in(c, r)
    if (r < cols && c < rows) out[r + (long long)c * ldo] = tile[threadIdx.x][j];
  }
}

// pair matrix M (N_r x n1 n2, column i + n1 j = a(:, i) .* b(:, j)); isdf.hpp:51-66
__global__ void pair_matrix_kernel(const double* a, long long lda, int n1, const double* b, long long ldb, int n2,
                                   int n_r, double* m, long long ldm) {
  const long long total = (long long)n_r * n1 * n2;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int r = static_cast<int>(idx % n_r);
    const long long col = idx / n_r;
    const int i = static_cast<int>(col % n1), j = static_cast<int>(col / n1);
    m[r + col * ldm] = a[r + i * lda] * b[r + j * ldb];
  }
}

}  // namespace

cudaError_t transpose(cudaStream_t st, const double* in, long long ldi, int rows, int cols, double* out,
                      long long ldo) {
  if (rows <= 0 || cols <= 0) return cudaSuccess;
  transpose_kernel<<<dim3((cols + 31) / 32, (rows + 31) / 32), dim3(32, 8), 0, st>>>(in, ldi, rows, cols, out, ldo);
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t pair_matrix(cudaStream_t st, const double* a, long long lda, int n1, const double* b, long long ldb,
                        int n2, int n_r, double* m, long long ldm) {
  if ((long long)n_r * n1 * n2 == 0) return cudaSuccess;
  pair_matrix_kernel<<<1184, 256, 0, st>>>(a, lda, n1, b, ldb, n2, n_r, m, ldm); count_launches(1);
  return cudaGetLastError();
}

cudaError_t scale_copy(cudaStream_t st, const double* src, double* dst, size_t n, double alpha) {
  if (n == 0) return cudaSuccess;
  scale_copy_kernel<<<1184, 256, 0, st>>>(src, dst, n, alpha); count_launches(1);
  return cudaGetLastError();
}

cudaError_t fill(cudaStream_t st, double* dst, size_t n, double v) {
  if (n == 0) return cudaSuccess;
  fill_kernel<<<1184, 256, 0, st>>>(dst, n, v); count_launches(1);
  return cudaGetLastError();
}

cudaError_t add_diag(cudaStream_t st, double* a, int n, long long lda, double v) {
  if (n <= 0) return cudaSuccess;
  add_diag_kernel<<<(n + 255) / 256, 256, 0, st>>>(a, n, lda, v); count_launches(1);
  return cudaGetLastError();
}

cudaError_t axpby(cudaStream_t st, int rows, int cols, double alpha, const double* x, long long ldx,
                  double beta, double* y, long long ldy) {
  if (rows <= 0 || cols <= 0) return cudaSuccess;
  axpby_kernel<<<1184, 256, 0, st>>>(rows, cols, alpha, x, ldx, beta, y, ldy); count_launches(1);
  return cudaGetLastError();
}

cudaError_t zero_strict_upper(cudaStream_t st, double* a, int n, long long lda) {
  if (n <= 1) return cudaSuccess;
  zero_strict_upper_kernel<<<592, 256, 0, st>>>(a, n, lda); count_launches(1);
  return cudaGetLastError();
}

// d_out must hold kRedBlocks + 1 doubles; the result lands in d_out[kRedBlocks].
cudaError_t max_abs(cudaStream_t st, const double* x, size_t n, double* d_out) {
  max_abs_kernel<<<kRedBlocks, 256, 0, st>>>(x, n, d_out); count_launches(1);
  finish_kernel<<<1, 32, 0, st>>>(d_out, kRedBlocks, d_out + kRedBlocks, 1); count_launches(1);
  return cudaGetLastError();
}

// First index i with chol(i, i)^2 < 1e-14 max|A| (the LU singularity rule of
// linalg.hpp:128, 137 on a Cholesky factor), or -1, into *out. One CTA.
__global__ void tiny_pivot_kernel(const double* chol, int n, long long ld, const double* max_abs_a, int* out) {
  __shared__ int best;
  if (threadIdx.x == 0) best = INT_MAX;
  __syncthreads();
  const double mx = *max_abs_a;
  const double tiny = 1e-14 * (mx > 0.0 ? mx : 1.0);
  int mine = INT_MAX;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double d = chol[(long long)i * (ld + 1)];
    if (d * d < tiny) {
      mine = i;
      break;
    }
  }
  if (mine != INT_MAX) atomicMin(&best, mine);
  __syncthreads();
  if (threadIdx.x == 0) *out = best == INT_MAX ? -1 : best;
}

// Diagonal of a triangular factor: out = {min |d_i|, max |d_i|, all(d_i^2 >=
// 1e-14 max d^2) ? 1 : 0}. One CTA (the fused fit's singularity rule, decided
// on the device so the fit never waits on the host).
__global__ void diag_stats_kernel(const double* a, int n, long long ld, double* out) {
  __shared__ double smin[256], smax[256];
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  double mn = HUGE_VAL, mx = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double d = fabs(a[(long long)i * (ld + 1)]);
    if (!(d <= DBL_MAX)) bad = 1;  // NaN / Inf
    mn = fmin(mn, d);
    mx = fmax(mx, d);
  }
  smin[threadIdx.x] = mn;
  smax[threadIdx.x] = mx;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      smin[threadIdx.x] = fmin(smin[threadIdx.x], smin[threadIdx.x + o]);
      smax[threadIdx.x] = fmax(smax[threadIdx.x], smax[threadIdx.x + o]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double gmax = smax[0] * smax[0];
    const double tiny = 1e-14 * (gmax > 0.0 ? gmax : 1.0);
    out[0] = smin[0];
    out[1] = smax[0];
    out[2] = (!bad && smin[0] * smin[0] >= tiny) ? 1.0 : 0.0;
  }
}

cudaError_t diag_stats(cudaStream_t st, const double* a, int n, long long ld, double* out) {
  diag_stats_kernel<<<1, 256, 0, st>>>(a, n, ld, out); count_launches(1);
  return cudaGetLastError();
}

cudaError_t tiny_pivot_dev(cudaStream_t st, const double* chol, int n, long long ld, const double* max_abs_a,
                           int* out) {
  tiny_pivot_kernel<<<1, 256, 0, st>>>(chol, n, ld, max_abs_a, out); count_launches(1);
  return cudaGetLastError();
}

// sum (a - b)^2 (b may be null) -> d_out2[kRedBlocks]
cudaError_t frob_diff(cudaStream_t st, const double* a, const double* b, size_t n, double* d_out2) {
  sum_sq_diff_kernel<<<kRedBlocks, 256, 0, st>>>(a, b, n, d_out2); count_launches(1);
  finish_kernel<<<1, 32, 0, st>>>(d_out2, kRedBlocks, d_out2 + kRedBlocks, 0); count_launches(1);
  return cudaGetLastError();
}

}  // namespace lrgw_dev
