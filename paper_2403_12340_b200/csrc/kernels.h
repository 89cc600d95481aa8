// kernels.h — internal device-side entry points of liblrgw_cuda (not the C-ABI;
// see include/lrgw_cuda.h for that). All matrices column-major FP64.
#pragma once

#include <algorithm>
#include <cstddef>
#include <cuda_runtime.h>

namespace lrgw_dev {

// Kernel launches issued by this library (all launcher sites bump it).
long long launch_count();
void count_launches(int n);

enum class Lay { MN, K };  // operand stored MN-contiguous (col-major) or K-contiguous

// C = alpha * A diag(scale) B^T + beta * C with A: M x K, B: N x K (see gemm.cuh).
// lower: only lower-triangle tiles (M == N); the strict upper triangle of the
// result is unspecified (callers mirror the lower one). `work` enables split-K.
// tri_b: B(n, k) == 0 for k < n (skip those k); colmap: output column n goes
// to column colmap[n] of C (device array).
cudaError_t dgemm(cudaStream_t st, int M, int N, int K, const double* A, long long lda, Lay la,
                  const double* B, long long ldb, Lay lb, double* C, long long ldc, double alpha,
                  double beta, const double* scale, bool lower, int sm_count, double* work,
                  size_t work_elems, bool tri_b = false, const int* colmap = nullptr,
                  const int* n_dev = nullptr, const double* cin = nullptr, long long ldcin = 0,
                  const int* cin_map = nullptr);

// `batch` independent products C_z = alpha A_z B_z^T + beta C_z with A_z = A + z bsa
// (likewise B, C), one launch (64 x 64 tiles): the small GEMMs of a recursion level.
cudaError_t dgemm_batched(cudaStream_t st, int batch, int M, int N, int K, const double* A, long long lda,
                          long long bsa, Lay la, const double* B, long long ldb, long long bsb, Lay lb, double* C,
                          long long ldc, long long bsc, double alpha, double beta, bool tri_b);

// TMA-fed engine (gemm4.cuh / gemm_tma.cu) for MN-contiguous operands:
// cudaErrorNotSupported when a shape / alignment is not covered (callers fall
// back to the cp.async engines). Enabled with LRGW_TMA=1.
bool tma_gemm_enabled();
bool tma_tall_enabled();  // tall-skinny widths 33..112 on the TMA engine (LRGW_TMA_TALL=0: off)
// map: a CUtensorMap (cuda.h) of a column-major rows x cols matrix, boxes {16 rows, bk cols}, 128 B swizzle
bool tma_encode_mn(void* map, const double* ptr, long long rows, long long cols, long long ld, int bk);
cudaError_t dgemm_tma(cudaStream_t st, int M, int N, int K, const double* A, long long lda, const double* B,
                      long long ldb, double* C, long long ldc, double alpha, double beta, bool tri_b,
                      const int* colmap, const int* n_dev);
// K-contiguous operands (A(m, k) at m lda + k): lower tiles, k-scale, split-K
// partials (k_chunk a multiple of 16; the caller reduces with dgemm_tma_k_tile(M)).
int dgemm_tma_k_tile(int m);
int dgemm_tma_k_per_sm(int m);  // resident CTAs per SM of that configuration
cudaError_t dgemm_tma_k(cudaStream_t st, int M, int N, int K, const double* A, long long lda, const double* B,
                        long long ldb, double* C, long long ldc, double alpha, double beta, const double* scale,
                        bool lower, int splits, int k_chunk, double* partial);
cudaError_t hadamard_tma(cudaStream_t st, int M, int N, const double* a1, long long lda1, const double* b1,
                         long long ldb1, int k1, const double* a2, long long lda2, const double* b2, long long ldb2,
                         int k2, double* C, long long ldc, double alpha, double beta);

// C = alpha * (A1 B1^T) o (A2 B2^T) + beta * C; A1: M x K1, B1: N x K1, A2: M x K2,
// B2: N x K2, all MN-contiguous (isdf.hpp:132 fit GEMM pair + Hadamard).
cudaError_t hadamard_gemm(cudaStream_t st, int M, int N, const double* a1, long long lda1,
                          const double* b1, long long ldb1, int k1, const double* a2,
                          long long lda2, const double* b2, long long ldb2, int k2, double* C,
                          long long ldc, double alpha, double beta);

// C = A B^T (A: M x K, B: N x K, both MN-contiguous; N <= 128) with the
// selection's residual downdate fused: d[m] -= sum_n C(m, n)^2 where
// pos[m] >= kend. cudaErrorNotSupported: shape / alignment not covered.
cudaError_t dgemm_tall_downdate(cudaStream_t st, int M, int N, int K, const double* A, long long lda,
                                const double* B, long long ldb, double* C, long long ldc, double* d,
                                const int* pos, int kend);

// The selection's block panel in one launch (panel.cu): W = (A1 B1^T) o (A2 B2^T)
// - L LR^T (M x N), C = W X^T (X: N x N, X(n, j) = x[n + j ldx]) and
// d[m] -= sum_n C(m, n)^2 where pos[m] >= kend. cudaErrorNotSupported when the
// shape / alignment is not covered (callers run the three-launch path).
bool select_panel_enabled(int n1, int n2);
// The panel on the TMA engine (panel4.cu): X given with its columns permuted
// inside 16-groups (select_cand_greedy's xperm); N <= 112.
bool select_panel_tma_enabled();
cudaError_t select_panel_tma(cudaStream_t st, int M, int N, const double* a1, long long lda1, const double* b1,
                             long long ldb1, int k1, const double* a2, long long lda2, const double* b2,
                             long long ldb2, int k2, const double* l, long long ldl, const double* lrow,
                             long long ldlr, int k, const double* xperm, long long ldx, double* c, long long ldc,
                             double* d, const int* pos, int kend);
// Device-driven form (k_dev != nullptr): k = *k_dev, N = *n_dev (<= the N
// given, which sizes the tile), c is the factor's column 0 (the block writes
// columns k .. k + N) and kend = k + N.
cudaError_t select_panel(cudaStream_t st, int M, int N, const double* a1, long long lda1, const double* b1,
                         long long ldb1, int k1, const double* a2, long long lda2, const double* b2, long long ldb2,
                         int k2, const double* l, long long ldl, const double* lrow, long long ldlr, int k,
                         const double* x, long long ldx, double* c, long long ldc, double* d, const int* pos,
                         int kend, const int* k_dev = nullptr, const int* n_dev = nullptr);

// a(j,i) = a(i,j) for i > j (average = 0) or both = (a(i,j) + a(j,i))/2.
cudaError_t mirror_lower(cudaStream_t st, double* a, int n, long long lda, bool average);

// dst(r, c) = src(rows[r], c), rows on device.
cudaError_t gather_rows(cudaStream_t st, const double* src, long long lds, int cols, const int* rows,
                        int n_rows, double* dst, long long ldd);

// rows `rows` of a (n1 cols), b (n2 cols) and l (nl cols) into da, db, dl (ld ldd), one launch.
// Device-side counts (optional): nl = *nl_dev, n_rows = *nrows_dev, rows += *row_off_dev.
cudaError_t gather_rows3(cudaStream_t st, const double* a, long long lda, int n1, const double* b, long long ldb,
                         int n2, const double* l, long long ldl, int nl, const int* rows, int n_rows, double* da,
                         double* db, double* dl, long long ldd, const int* nl_dev = nullptr,
                         const int* nrows_dev = nullptr, const int* row_off_dev = nullptr);

// dst(:, c) = src(:, cols[c]), cols on device.
cudaError_t gather_cols(cudaStream_t st, const double* src, long long lds, int rows, const int* cols, int n,
                        double* dst, long long ldd);

// K7 probe passes over Theta (skinny.cu), m in {1, 2, 4, 8, 16}.
bool skinny_supported(int m);
cudaError_t skinny_tn(cudaStream_t st, const double* theta, long long ldt, int n_r, int n_mu, const double* x,
                      long long ldx, int m, double* u, long long ldu, double* work, size_t work_elems, int sm_count);
cudaError_t skinny_nn(cudaStream_t st, const double* theta, long long ldt, int n_r, int n_mu, const double* w,
                      long long ldw, int m, double* z, long long ldz, int sm_count);

// K3 quadrature (quadrature.cu).
// Workspace (doubles) of quad_nodes: per-segment 64 x 64 partials + the plan tables.
size_t quad_partial_elems(int n_mu, int n_nodes, int sm_count);
cudaError_t quad_nodes(cudaStream_t st, int n_mu, int n_v, int n_c, const double* pv, long long ldv,
                       const double* pc, long long ldc, int n_nodes, const double* dv,
                       const double* dc, const double* gw, int sm_count, double* partial,
                       double* running, double beta, double pref, double* t, long long ldt,
                       cudaEvent_t k_begin = nullptr, cudaEvent_t k_end = nullptr);

// The node kernel on the TMA feed (quad4.cu); cudaErrorNotSupported when the
// panels do not qualify for a tensor map. LRGW_QUAD_TMA=0 keeps the cp.async kernel.
bool quad_tma_enabled();
cudaError_t quad_nodes_tma(cudaStream_t st, int n_mu, int n_v, int n_c, const double* pv, long long ldv,
                           const double* pc, long long ldc, int n_nodes, long long units, const double* dv,
                           const double* dc, const double* gw, const int* seg_base, int ctas,
                           double* partial);

// The batched 3-D D2Z of m columns (fft.cu; cuFFT's layout and sign):
// cudaErrorNotSupported for axes that do not factor into 2, 3, 5 or an odd
// dims[0] / dims[1] (callers use the cuFFT leaf). LRGW_FFT_OWN=0: always cuFFT.
bool fft_own_enabled();
cudaError_t fft_d2z_3d(cudaStream_t st, const int* dims, const double* x, long long ldx, int m, double* xhat,
                       int sm_count);

// Coulomb (coulomb.cu): G-space half-spectrum weights c(G) = w_G v(G) / N_r
// (w_G = 2 off the self-conjugate i1 planes, 1 on them) laid out to match a
// D2Z output column of 2*n3*n2*(n1/2+1) interleaved reals.
cudaError_t coulomb_half_weights(cudaStream_t st, int n1, int n2, int n3, double c1, double c2,
                                 double c3, int zero_kernel, double* w);
// The same scale with a caller-supplied full-grid kernel v (its G / -G average).
cudaError_t coulomb_scale_half_custom(cudaStream_t st, int n1, int n2, int n3, const double* v, double* xhat,
                                      int cols);
// y(r) = x_hat(G) * v(G) / N_r over the half spectrum (in place, complex).
cudaError_t coulomb_scale_half(cudaStream_t st, int n1, int n2, int n3, double c1, double c2,
                               double c3, int zero_kernel, double* xhat, int cols);


// scalar helpers (misc.cu)
cudaError_t scale_copy(cudaStream_t st, const double* src, double* dst, size_t n, double alpha);
cudaError_t fill(cudaStream_t st, double* dst, size_t n, double v);
// M (n_r x n1 n2): column i + n1 j = a(:, i) .* b(:, j) (the reference's pair matrix)
cudaError_t pair_matrix(cudaStream_t st, const double* a, long long lda, int n1, const double* b, long long ldb,
                        int n2, int n_r, double* m, long long ldm);
cudaError_t zero_strict_upper(cudaStream_t st, double* a, int n, long long lda);
// out (cols x rows) = in^T (rows x cols), column-major.
cudaError_t transpose(cudaStream_t st, const double* in, long long ldi, int rows, int cols, double* out,
                      long long ldo);

// In-place inverse of the lower triangle of a (n x n, ld lda) — trtri.cu.
// work: trtri_work_elems(n) doubles; *bad (device, preset to INT_MAX) gets
// (first zero pivot + 1) if the factor is singular.
size_t trtri_work_elems(int n);
cudaError_t trtri_lower(cudaStream_t st, double* a, int n, long long lda, double* work, int* bad, int sm_count);
cudaError_t add_diag(cudaStream_t st, double* a, int n, long long lda, double v);
cudaError_t axpby(cudaStream_t st, int rows, int cols, double alpha, const double* x, long long ldx,
                  double beta, double* y, long long ldy);
cudaError_t max_abs(cudaStream_t st, const double* x, size_t n, double* d_out);
// first i with chol(i, i)^2 < 1e-14 max(*max_abs_a, 1 if 0) (or NaN), else -1 -> *out
cudaError_t diag_stats(cudaStream_t st, const double* a, int n, long long ld, double* out);
cudaError_t tiny_pivot_dev(cudaStream_t st, const double* chol, int n, long long ld, const double* max_abs_a,
                           int* out);
// sigma.cu: m = h o m (n x n); out[j] = alpha * a(:, j) . b(:, j).
cudaError_t hadamard_inplace(cudaStream_t st, int n, const double* h, long long ldh, double* m, long long ldm);
cudaError_t col_dot(cudaStream_t st, int rows, int cols, const double* a, long long lda, const double* b,
                    long long ldb, double alpha, double* out);
cudaError_t frob_diff(cudaStream_t st, const double* a, const double* b, size_t n, double* d_out2);

}  // namespace lrgw_dev
