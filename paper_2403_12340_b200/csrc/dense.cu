// dense.cu — the reference's dense utility layer (matrix.hpp products,
// linalg.hpp qrcp / lu_* / sym_eig, dft.hpp, the guarded pair matrix of
// isdf.hpp:49-88) on the device, behind host-buffer C-ABI calls for the C++
// drop-in headers. Products run on the path's DMMA engines, the
// factorisations are cuSOLVER leaves with the reference's singularity rule,
// QRCP takes its pivots from the path's greedy selection (K1: the greedy
// pivoted Cholesky on A^T A has QRCP's pivot sequence, swap-mirrored ties
// included) and its Q / R from geqrf / orgqr of the pivoted columns, and the
// unitary DFT is a cuFFT Z2Z leaf scaled by 1 / sqrt(N_r).
#include <cufft.h>
#include <cusolverDn.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "internal.h"
#include "select.h"

using namespace lrgw_impl;

namespace {

void lu_checked(lrgw_ctx c, double* lu, int n, int* ipiv_dev, double max_abs_in) {
  int lwork = 0;
  cks(cusolverDnDgetrf_bufferSize(c->solver, n, n, lu, n, &lwork), "getrf_bufferSize");
  DBuf work = dalloc(c, (size_t)std::max(lwork, 1));
  DBuf info = ialloc(c, 1);
  cks(cusolverDnDgetrf(c->solver, n, n, lu, n, work.d(), ipiv_dev, info.i()), "getrf");
  std::vector<double> diag(n);
  ck(cudaMemcpy2DAsync(diag.data(), sizeof(double), lu, (size_t)(n + 1) * sizeof(double), sizeof(double), n,
                       cudaMemcpyDeviceToHost, c->stream),
     "D2H diag");
  ck(cudaStreamSynchronize(c->stream), "sync");
  // linalg.hpp:128, 137: singular when |pivot| < 1e-14 max|A|
  const double tiny = 1e-14 * (max_abs_in > 0.0 ? max_abs_in : 1.0);
  for (int i = 0; i < n; ++i)
    if (!(std::abs(diag[i]) >= tiny)) fail(LRGW_ERR_SINGULAR, "lu_factor: matrix is singular", i);
}

double host_max_abs(const double* a, size_t n) {
  double m = 0.0;
  for (size_t i = 0; i < n; ++i) m = std::max(m, std::abs(a[i]));
  return m;
}

}  // namespace

extern "C" {

int lrgw_matmul(lrgw_ctx c, char ta, char tb, int m, int n, int k, const double* a, long long lda, const double* b,
                long long ldb, double* cm, long long ldc) {
  return guarded(c, [&] {
    if (m < 0 || n < 0 || k < 0) fail(LRGW_ERR_INVALID_INPUT, "matmul: negative dimension");
    if (m == 0 || n == 0) return;
    const bool at = ta == 'T' || ta == 't', bt = tb == 'T' || tb == 't';
    const long long ar = at ? k : m, ac = at ? m : k, br = bt ? n : k, bc = bt ? k : n;
    if (lda < std::max(1LL, ar) || ldb < std::max(1LL, br) || ldc < m) fail(LRGW_ERR_INVALID_INPUT, "matmul: bad leading dimension");
    DBuf da = dalloc(c, (size_t)lda * ac), db = dalloc(c, (size_t)ldb * bc), dc = dalloc(c, (size_t)ldc * n);
    if (k == 0) {
      ck(fill(c->stream, dc.d(), (size_t)ldc * n, 0.0), "fill");
    } else {
      ck(cudaMemcpyAsync(da.p, a, sizeof(double) * lda * ac, cudaMemcpyHostToDevice, c->stream), "H2D");
      ck(cudaMemcpyAsync(db.p, b, sizeof(double) * ldb * bc, cudaMemcpyHostToDevice, c->stream), "H2D");
      Work w = make_work(c, (size_t)8 * m * n);
      gemm(c, m, n, k, da.d(), lda, at ? Lay::K : Lay::MN, db.d(), ldb, bt ? Lay::MN : Lay::K, dc.d(), ldc, 1.0, 0.0,
           nullptr, false, &w);
    }
    download(c, cm, dc.p, sizeof(double) * ldc * n);
  });
}

// linalg.hpp:117-150 — LuFactors{lu, piv (0-based row swapped with at step i), max|A|}
int lrgw_lu_factor(lrgw_ctx c, const double* a, int n, double* lu, int32_t* piv, double* max_abs_out) {
  return guarded(c, [&] {
    if (n < 1) fail(LRGW_ERR_INVALID_INPUT, "lu_factor: not square");
    const size_t nn = (size_t)n * n;
    const double mx = host_max_abs(a, nn);
    if (max_abs_out) *max_abs_out = mx;
    DBuf d = upload(c, a, nn);
    DBuf ip = ialloc(c, n);
    lu_checked(c, d.d(), n, ip.i(), mx);
    download(c, lu, d.p, nn * sizeof(double));
    download(c, piv, ip.p, (size_t)n * sizeof(int));
    for (int i = 0; i < n; ++i) piv[i] -= 1;  // cuSOLVER's ipiv is 1-based
  });
}

// linalg.hpp:152-175 — X = A^-1 B from the factors of lrgw_lu_factor.
int lrgw_lu_solve_factored(lrgw_ctx c, const double* lu, const int32_t* piv, int n, const double* b, int nrhs,
                           double* x) {
  return guarded(c, [&] {
    if (n < 1 || nrhs < 0) fail(LRGW_ERR_INVALID_INPUT, "lu_solve: rhs row mismatch");
    if (nrhs == 0) return;
    std::vector<int> ip(piv, piv + n);
    for (int& v : ip) v += 1;
    DBuf d = upload(c, lu, (size_t)n * n), rhs = upload(c, b, (size_t)n * nrhs);
    DBuf dp = upload_i(c, ip.data(), n), info = ialloc(c, 1);
    cks(cusolverDnDgetrs(c->solver, CUBLAS_OP_N, n, nrhs, d.d(), n, dp.i(), rhs.d(), n, info.i()), "getrs");
    download(c, x, rhs.p, (size_t)n * nrhs * sizeof(double));
  });
}

// linalg.hpp:190-345 — ascending eigenvalues, orthonormal eigenvectors in the columns of q.
int lrgw_sym_eig(lrgw_ctx c, const double* a, int n, double* values, double* q) {
  return guarded(c, [&] {
    if (n < 1) fail(LRGW_ERR_INVALID_INPUT, "sym_eig: not square");
    const size_t nn = (size_t)n * n;
    DBuf d = upload(c, a, nn), w = dalloc(c, n), info = ialloc(c, 1);
    int lwork = 0;
    cks(cusolverDnDsyevd_bufferSize(c->solver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, d.d(), n, w.d(),
                                    &lwork),
        "syevd_bufferSize");
    DBuf work = dalloc(c, (size_t)std::max(lwork, 1));
    cks(cusolverDnDsyevd(c->solver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, d.d(), n, w.d(), work.d(),
                         lwork, info.i()),
        "syevd");
    int h = 0;
    download(c, &h, info.p, sizeof(int));
    if (h != 0) fail(LRGW_ERR_NUMERIC, "sym_eig: no convergence");
    download(c, values, w.p, (size_t)n * sizeof(double));
    if (q) download(c, q, d.p, nn * sizeof(double));
  });
}

// linalg.hpp:17-111 — QrcpResult{q (m x k), r (k x n), perm (n)}, k = min(m, n).
int lrgw_qrcp(lrgw_ctx c, const double* a, int m, int n, int32_t* perm, double* q, double* r) {
  return guarded(c, [&] {
    if (m < 1 || n < 1) fail(LRGW_ERR_INVALID_INPUT, "qrcp: empty matrix");
    const int k = std::min(m, n);
    const size_t mn = (size_t)m * n;
    DBuf da = upload(c, a, mn);
    // pivot order: greedy pivoted Cholesky on A^T A (rows of A^T, b = ones)
    DBuf at = dalloc(c, mn), ones = dalloc(c, n);
    ck(transpose(c->stream, da.d(), m, m, n, at.d(), n), "transpose");
    ck(fill(c->stream, ones.d(), n, 1.0), "fill");
    SelectKeep keep;
    select_impl(c, at.d(), n, m, ones.d(), n, 1, n, k, nullptr, &keep);
    // the full swap-mirrored permutation (selection order, then the rest)
    const std::vector<int>& order = keep.order;
    // the reference's perm (linalg.hpp:48-53): replay the k position swaps
    std::vector<int> pm(n);
    for (int i = 0; i < n; ++i) pm[i] = i;
    for (int s = 0; s < k; ++s) {
      const int p = (int)(std::find(pm.begin() + s, pm.end(), order[s]) - pm.begin());
      std::swap(pm[s], pm[p]);
    }
    for (int i = 0; i < n; ++i) perm[i] = pm[i];
    // Q R of the pivoted columns (Householder leaves)
    DBuf ap = dalloc(c, mn), dperm = upload_i(c, pm.data(), n);
    ck(gather_cols(c->stream, da.d(), m, m, dperm.i(), n, ap.d(), m), "gather_cols");
    DBuf tau = dalloc(c, k), info = ialloc(c, 1);
    int lw1 = 0, lw2 = 0;
    cks(cusolverDnDgeqrf_bufferSize(c->solver, m, n, ap.d(), m, &lw1), "geqrf_bufferSize");
    DBuf work = dalloc(c, (size_t)std::max(lw1, 1));
    cks(cusolverDnDgeqrf(c->solver, m, n, ap.d(), m, tau.d(), work.d(), lw1, info.i()), "geqrf");
    std::vector<double> hr(mn);
    download(c, hr.data(), ap.p, mn * sizeof(double));
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < k; ++i) r[i + (size_t)j * k] = i <= j ? hr[i + (size_t)j * m] : 0.0;
    cks(cusolverDnDorgqr_bufferSize(c->solver, m, k, k, ap.d(), m, tau.d(), &lw2), "orgqr_bufferSize");
    DBuf work2 = dalloc(c, (size_t)std::max(lw2, 1));
    cks(cusolverDnDorgqr(c->solver, m, k, k, ap.d(), m, tau.d(), work2.d(), lw2, info.i()), "orgqr");
    download(c, q, ap.p, (size_t)m * k * sizeof(double));
  });
}

// dft.hpp:37-68 — unitary 3-D DFT of an interleaved complex grid vector
// (forward e^{-2 pi i k.r / n}, inverse e^{+...}, 1/sqrt(N_r) each way).
int lrgw_dft(lrgw_ctx c, const int* dims, const double* x, int inverse, double* y) {
  return guarded(c, [&] {
    if (!dims) fail(LRGW_ERR_INVALID_INPUT, "dft: null dims");
    for (int i = 0; i < 3; ++i)
      if (dims[i] < 1) fail(LRGW_ERR_INVALID_INPUT, "dft: size mismatch");
    const size_t n_r = (size_t)dims[0] * dims[1] * dims[2];
    DBuf d = upload(c, x, 2 * n_r);
    cufftHandle plan;
    ckf(cufftPlan3d(&plan, dims[2], dims[1], dims[0], CUFFT_Z2Z), "cufftPlan3d");
    ckf(cufftSetStream(plan, c->stream), "cufftSetStream");
    const cufftResult rr = cufftExecZ2Z(plan, reinterpret_cast<cufftDoubleComplex*>(d.d()),
                                        reinterpret_cast<cufftDoubleComplex*>(d.d()),
                                        inverse ? CUFFT_INVERSE : CUFFT_FORWARD);
    ck(cudaStreamSynchronize(c->stream), "sync");
    cufftDestroy(plan);
    ckf(rr, "cufftExecZ2Z");
    ck(scale_copy(c->stream, d.d(), d.d(), 2 * n_r, 1.0 / std::sqrt((double)n_r)), "scale");
    download(c, y, d.p, 2 * n_r * sizeof(double));
  });
}

// isdf.hpp:49-88 — M (N_r x N1 N2, column i + N1 j = a(:, i) .* b(:, j)) or its
// transpose; refused beyond the reference's 2^26-entry guard.
int lrgw_pair_matrix(lrgw_ctx c, const double* a, const double* b, int n_r, int n1, int n2, int transposed,
                     double* out) {
  return guarded(c, [&] {
    if (n_r < 1 || n1 < 1 || n2 < 1) fail(LRGW_ERR_INVALID_INPUT, "pair_matrix: row mismatch");
    const long long cols = (long long)n1 * n2;
    if ((long long)n_r * cols > (1LL << 26))
      fail(LRGW_ERR_GUARD_EXCEEDED, transposed ? "pair_matrix_transposed: materialization guard exceeded"
                                               : "pair_matrix: materialization guard exceeded");
    DBuf da = upload(c, a, (size_t)n_r * n1), db = upload(c, b, (size_t)n_r * n2), dm = dalloc(c, (size_t)n_r * cols);
    ck(pair_matrix(c->stream, da.d(), n_r, n1, db.d(), n_r, n2, n_r, dm.d(), n_r), "pair_matrix");
    if (transposed) {
      DBuf dt = dalloc(c, (size_t)n_r * cols);
      ck(transpose(c->stream, dm.d(), n_r, n_r, (int)cols, dt.d(), cols), "transpose");
      download(c, out, dt.p, (size_t)n_r * cols * sizeof(double));
    } else {
      download(c, out, dm.p, (size_t)n_r * cols * sizeof(double));
    }
  });
}

// apply_coulomb (model.hpp:208-223) with the operator's own kernel array
// (CoulombOperator::kernel, length N_r): Re(F^-1 diag(kernel) F x).
int lrgw_apply_coulomb_kernel(lrgw_ctx c, const int* dims, const double* kernel, const double* x, int m, double* y) {
  return guarded(c, [&] {
    if (!dims || !kernel) fail(LRGW_ERR_INVALID_INPUT, "apply_coulomb: null argument");
    for (int i = 0; i < 3; ++i)
      if (dims[i] < 2) fail(LRGW_ERR_INVALID_INPUT, "Grid: all dims must be >= 2");
    if (m <= 0) return;
    const size_t n_r = (size_t)dims[0] * dims[1] * dims[2];
    DBuf dx = upload(c, x, n_r * m), dy = dalloc(c, n_r * m), dk = upload(c, kernel, n_r);
    const long long nh = half_len(dims);
    DBuf xh = dalloc(c, (size_t)2 * nh * m);
    fft_forward(c, dims, dx.d(), n_r, m, xh.d());
    ck(coulomb_scale_half_custom(c->stream, dims[0], dims[1], dims[2], dk.d(), xh.d(), m), "scale");
    fft_inverse(c, dims, xh.d(), m, dy.d(), n_r);
    download(c, y, dy.p, n_r * m * sizeof(double));
  });
}

}  // extern "C"
