/* lrgw_cuda.h — C-ABI of liblrgw_cuda.so, the B200 (sm_100a) implementation of
 * the low-rank epsilon^-1 hot path of arXiv 2403.12340 (reference: the
 * header-only C++ library `lrgw`, /root/reference/proj/include/lrgw).
 *
 * Plain C: pointers, sizes, int status codes; no C++ or torch types. Every
 * matrix is column-major float64 with an explicit leading dimension.
 * The reference's C++ API (include/lrgw/*.hpp in this repo) is a thin layer
 * over these entry points; INTEGRATION.md shows how a caller binds them.
 *
 * Status codes map 1:1 onto the reference exception taxonomy
 * (errors.hpp:10-36, contour.hpp:92-96). A failing call leaves a message in
 * lrgw_ctx_last_error(); LRGW_ERR_SINGULAR also sets lrgw_ctx_last_pivot().
 * Calls are synchronous at the ABI (results are complete on return) unless
 * the name carries `_async`. A context is single-threaded; concurrent
 * contexts are allowed.
 */
#ifndef LRGW_CUDA_H_
#define LRGW_CUDA_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LRGW_ABI_VERSION 2

enum lrgw_status {
  LRGW_OK = 0,
  LRGW_ERR_INVALID_INPUT = 1,        /* invalid_input   (errors.hpp:10-12) */
  LRGW_ERR_GUARD_EXCEEDED = 2,       /* guard_exceeded  (errors.hpp:21-23) */
  LRGW_ERR_NUMERIC = 3,              /* numeric_error   (errors.hpp:26-28) */
  LRGW_ERR_SINGULAR = 4,             /* singular_matrix (errors.hpp:31-36) */
  LRGW_ERR_CONTOUR_CONVERGENCE = 5,  /* contour_convergence_error (contour.hpp:92-96) */
  LRGW_ERR_IO = 6,                   /* io_error        (errors.hpp:15-17) */
  LRGW_ERR_CUDA = 7,                 /* device / library failure (no reference analogue) */
  LRGW_ERR_UNSUPPORTED = 8,          /* reported as invalid_input by the C++ layer */
  LRGW_ERR_INTERNAL = 9
};

/* PointSelector (isdf.hpp:28) */
enum lrgw_point_selector { LRGW_QRCP_DIRECT = 0, LRGW_QRCP_SKETCHED = 1 };

/* Build stages timed by lrgw_build (device time, CUDA events on the context
 * stream, consecutive intervals). */
enum lrgw_stage {
  LRGW_STAGE_SELECT = 0,    /* K1 ISDF point selection                         */
  LRGW_STAGE_FIT_LHS = 1,   /* K2a lhs (explicit fit only; empty when fused)   */
  LRGW_STAGE_FIT_SOLVE = 2, /* L_P gather + recursive DMMA triangular inverse  */
  LRGW_STAGE_FIT_GEMM = 3,  /* K2b Theta = L L_P^-1                            */
  LRGW_STAGE_CONTOUR = 4,   /* K3 Cauchy quadrature of the core T (+ tables)   */
  LRGW_STAGE_FFT = 5,       /* cuFFT leaf: batched D2Z of Theta                */
  LRGW_STAGE_PVP = 6,       /* K5 Theta^T V Theta G-space SYRK                 */
  LRGW_STAGE_SMW = 7,       /* K6 SMW core K (cuSOLVER potrf leaves + DMMA)    */
  LRGW_STAGE_TOTAL = 8,
  LRGW_STAGE_QUAD_KERNEL = 9, /* the K3 kernel alone (last quadrature launch)  */
  LRGW_STAGE_CUSOLVER = 10,   /* the cuSOLVER potrf leaves inside SMW (summed)  */
  LRGW_STAGE_CUFFT = 11,      /* the cuFFT D2Z leaf of FFT (= FFT; listed apart) */
  LRGW_NUM_STAGES = 12
};

typedef struct lrgw_ctx_s* lrgw_ctx;
typedef struct lrgw_eps_s* lrgw_eps; /* device-resident factored eps^-1 (smw.hpp:77-82) */

int lrgw_abi_version(void);

/* ---- context ------------------------------------------------------------- */
int lrgw_ctx_create(int device, lrgw_ctx* out);
int lrgw_ctx_destroy(lrgw_ctx ctx);
int lrgw_ctx_set_stream(lrgw_ctx ctx, void* cuda_stream); /* NULL = context-owned stream */
void* lrgw_ctx_stream(lrgw_ctx ctx);
int lrgw_ctx_synchronize(lrgw_ctx ctx);
const char* lrgw_ctx_last_error(lrgw_ctx ctx);
int lrgw_ctx_last_pivot(lrgw_ctx ctx);
/* Per-stage device milliseconds of the last lrgw_build (LRGW_NUM_STAGES). */
int lrgw_ctx_stage_ms(lrgw_ctx ctx, double* ms, int n);
/* Kernel launches issued by this context since creation (own kernels only). */
long long lrgw_ctx_kernel_launches(lrgw_ctx ctx);
/* Candidate-set size of the batched greedy point selection (default 64). */
int lrgw_ctx_set_select_batch(lrgw_ctx ctx, int s);
/* on != 0: lrgw_build keeps Theta factored as L L_P^-1 (the selection factor
 * and its point block) instead of forming it — the N_r x N_mu^2 fit GEMM
 * leaves the build; the handle applies eps^-1 unchanged and forms Theta, K,
 * T, Theta^T V Theta on first demand (lrgw_eps_get / info / device_ptrs,
 * the screened projections). Default off. */
int lrgw_ctx_set_theta_implicit(lrgw_ctx ctx, int on);

/* ---- host-scalar contour geometry ----------------------------------------- */
int lrgw_num_aux(double k_mu, int n1, int n2, int* out);                 /* isdf.hpp:42-46 */
int lrgw_elliptic_k(double k, double* out);                              /* elliptic.hpp:28-33 */
int lrgw_jacobi_sn_cn_dn(double u, double k, double* out3);              /* elliptic.hpp:48-85 */
int lrgw_jacobi_complex(double x, double y, double k, double* out6);     /* elliptic.hpp:97-118 */
/* spec7 = {q, Q, r, R, L, e_shift, bypass}                                  contour.hpp:35-71 */
int lrgw_elliptic_params(const double* energies, int n_e, int n_v, int n_c, double delta_rel,
                         int max_nodes, double* spec7);
int lrgw_cauchy_error_bound(const double* spec7, int n_lambda, double* out); /* contour.hpp:75-80 */

/* ---- host-buffer API: drop-in bodies of the reference free functions ------ */
/* select_interpolation_points (isdf.hpp:95-112); pts sorted ascending. */
int lrgw_select_interpolation_points(lrgw_ctx ctx, const double* psi_a, const double* psi_b,
                                     int n_r, int n1, int n2, int n_mu, int method, int32_t* pts);
/* fit_auxiliary_basis (isdf.hpp:118-163): theta is n_r x n_mu. */
int lrgw_fit_auxiliary_basis(lrgw_ctx ctx, const double* psi_a, const double* psi_b, int n_r,
                             int n1, int n2, const int32_t* pts, int n_mu, double* theta);
/* coupled_coefficients_direct (contour.hpp:114-137). */
int lrgw_coupled_coefficients_direct(lrgw_ctx ctx, const double* psi_v_pts,
                                     const double* psi_c_pts, int n_mu, int n_v, int n_c,
                                     const double* energies, int n_e, double* t);
/* detail::sum_node_terms (contour.hpp:185-222): acc = sum_k w_k term_k. */
int lrgw_sum_node_terms(lrgw_ctx ctx, const double* psi_v_pts, const double* psi_c_pts, int n_mu,
                        int n_v, int n_c, const double* energies, int n_e, const double* spec7,
                        const double* nodes, const double* weights, int n_nodes, double* acc);
/* Fixed closed trapezoid of n_lambda intervals (n_lambda + 1 nodes), times the
 * prefactor and symmetrised — the BASELINE configs' quadrature. */
int lrgw_coupled_coefficients_fixed(lrgw_ctx ctx, const double* psi_v_pts,
                                    const double* psi_c_pts, int n_mu, int n_v, int n_c,
                                    const double* energies, int n_e, int n_lambda, double* t);
/* coupled_coefficients_contour (contour.hpp:298-329). On
 * LRGW_ERR_CONTOUR_CONVERGENCE `t`, nodes_used and est_rel hold the best estimate. */
int lrgw_coupled_coefficients_contour(lrgw_ctx ctx, const double* psi_v_pts,
                                      const double* psi_c_pts, int n_mu, int n_v, int n_c,
                                      const double* energies, int n_e, double delta_rel,
                                      int max_nodes, double* t, int* nodes_used, double* est_rel);
/* contour_refinement_levels (contour.hpp:282-294): up to max_levels estimates. */
int lrgw_contour_refinement_levels(lrgw_ctx ctx, const double* psi_v_pts,
                                   const double* psi_c_pts, int n_mu, int n_v, int n_c,
                                   const double* energies, int n_e, int max_level_nodes,
                                   int max_levels, double* out, int* counts, int* n_levels);
/* build_coulomb kernel (model.hpp:165-195), length n_r. */
int lrgw_coulomb_kernel(const int* dims, const double* cell, double* kernel);
/* apply_coulomb (model.hpp:208-223); zero_kernel selects zero_coulomb (198-204). */
int lrgw_apply_coulomb(lrgw_ctx ctx, const int* dims, const double* cell, int zero_kernel,
                       const double* x, int m, double* y);
/* assemble_K (smw.hpp:42-73). */
int lrgw_assemble_K(lrgw_ctx ctx, const double* t, const double* p, int n_r, int n_mu,
                    const int* dims, const double* cell, int zero_kernel, double* k);
/* build_epsilon_inverse (smw.hpp:84-94): uploads P, keeps P and K on device. */
int lrgw_build_epsilon_inverse(lrgw_ctx ctx, const double* t, const double* p, int n_r, int n_mu,
                               const int* dims, const double* cell, int zero_kernel,
                               lrgw_eps* out);
/* An eps handle from host P and a caller-supplied K (e.g. the K = 0 identity). */
int lrgw_eps_from_parts(lrgw_ctx ctx, const double* p, const double* k, int n_r, int n_mu,
                        const int* dims, const double* cell, int zero_kernel, lrgw_eps* out);
/* epsilon_inverse_apply (smw.hpp:97-103): Y = X + V P (K (P^T X)), X n_r x m. */
int lrgw_epsilon_inverse_apply(lrgw_ctx ctx, lrgw_eps e, const double* x, int m, double* y);
/* Host copies of the factors (any pointer may be NULL). vp = V P is formed on demand. */
int lrgw_eps_get(lrgw_ctx ctx, lrgw_eps e, double* k, double* p, double* vp, double* t,
                 int32_t* pts);
int lrgw_eps_shape(lrgw_eps e, int* n_r, int* n_mu);
int lrgw_eps_destroy(lrgw_eps e);

/* ---- device-pointer API (the hot path; all pointers in device memory) ----- */
typedef struct {
  int n_r, n_v, n_c;
  int dims[3];
  double cell[3];
  double k_mu;       /* N_mu = clamp(llround(k_mu sqrt(N_v N_c)), 1, N_r) (isdf.hpp:42-46, 180) */
  int n_lambda;      /* > 0: fixed trapezoid of n_lambda intervals; 0: adaptive (delta_rel) */
  double delta_rel;  /* adaptive stopping rule (contour.hpp:313-320) */
  int max_nodes;     /* adaptive node cap (contour.hpp:31) */
  int zero_kernel;   /* 1: V = 0 (zero_coulomb) */
  int n_e;           /* length of `energies` (>= n_v + n_c; contour.hpp:35-44) */
} lrgw_build_params;

/* The factored eps^-1 build, stages 1-5, from device-resident orbitals
 * phi_v (n_r x n_v, ld ldv) and phi_c (n_r x n_c, ld ldc) and host energies
 * (ascending, n_v + n_c). Stage device times: lrgw_ctx_stage_ms. */
int lrgw_build(lrgw_ctx ctx, const lrgw_build_params* prm, const double* phi_v, long long ldv,
               const double* phi_c, long long ldc, const double* energies, lrgw_eps* out);
/* Build diagnostics and device pointers of a factored inverse. Pointers are
 * owned by the handle (pvp and the selection / fit fields only for handles
 * made by lrgw_build; otherwise NULL / -1). */
typedef struct {
  int n_r, n_mu;
  double* theta;        /* n_r x n_mu, sorted-point column order       */
  double* k;            /* n_mu x n_mu SMW core                        */
  double* t;            /* n_mu x n_mu quadrature core T               */
  double* pvp;          /* n_mu x n_mu Theta^T V Theta                 */
  double min_margin;    /* smallest relative top-2 residual margin (d1 - d2) / d1 over the greedy steps */
  int min_margin_step;  /* the step it occurred at                     */
  int fit_path;         /* 0: fused Theta = L L_P^-1; 1: explicit Gram LU (isdf.hpp:143); 2: implicit (kept factored) */
  double lp_diag_ratio; /* (max|L_P,ii| / min|L_P,ii|)^2, a lower bound on cond(G(P,P)) */
  int select_blocks;    /* candidate blocks of the selection            */
} lrgw_eps_info;
int lrgw_eps_info_get(lrgw_eps e, lrgw_eps_info* out);
/* Device pointers owned by the handle (n_r x n_mu Theta, n_mu^2 K and T). */
int lrgw_eps_device_ptrs(lrgw_eps e, double** theta, double** k, double** t);
/* eps^-1 applied to a device block: y = x + V Theta (K (Theta^T x)). */
int lrgw_eps_apply_dev(lrgw_ctx ctx, lrgw_eps e, const double* x, long long ldx, int m, double* y,
                       long long ldy);

/* Projected screened interactions (reference gw.hpp:73-88
 * project_screened_interactions) from a factored inverse e and the vn / nn
 * interpolation vectors P_vn (N_r x n_vn) and P_nn (N_r x n_nn), column
 * major:
 *   B_x = P_x^T V P_vc,  W_x = B_x K B_x^T (x = vn, nn),  V_vn = P_vn^T V P_vn
 * (each symmetric). Host arrays; outputs n_vn^2, n_nn^2, n_vn^2. The vn / nn
 * decompositions themselves are lrgw_select_interpolation_points +
 * lrgw_fit_auxiliary_basis on the pair factors (Phi_v, Psi) / (Psi, Psi)
 * (isdf.hpp:166-183). */
int lrgw_project_screened_interactions(lrgw_ctx ctx, lrgw_eps e, const double* p_vn, int n_vn,
                                       const double* p_nn, int n_nn, double* w_vn, double* w_nn,
                                       double* v_vn);
/* The same on device arrays (P_x with leading dims ld_x; outputs n x n, ld n). */
int lrgw_dev_project_screened(lrgw_ctx ctx, lrgw_eps e, const double* p_vn, long long ld_vn, int n_vn,
                              const double* p_nn, long long ld_nn, int n_nn, double* w_vn, double* w_nn,
                              double* v_vn);

/* Static-COHSEX self-energy diagonals of the low-rank pipeline (reference
 * gw.hpp:93-137 detail::sigma_hadamard + gw.hpp:143-153
 * self_energies_lowrank): with Psi = orbitals (n_r x (n_v + n_c), column
 * major), Psi_vn / Psi_nn its rows at the vn / nn points,
 *   sigma_sex_x = -diag(Psi_vn^T (W_vn o Psi_o Psi_o^T) Psi_vn)
 *   sigma_x     = -diag(Psi_vn^T (V_vn o Psi_o Psi_o^T) Psi_vn)
 *   sigma_coh   = 1/2 diag(Psi_nn^T (W_nn o Psi_nn Psi_nn^T) Psi_nn)
 * (Psi_o = the occupied columns of Psi_vn) and sigma_total their sum
 * (SelfEnergies::finalize, gw.hpp:31-41: LRGW_ERR_NUMERIC on a non-finite
 * band). Host arrays; outputs of length n_v + n_c (any may be null). */
int lrgw_self_energies_lowrank(lrgw_ctx ctx, const double* psi, int n_r, int n_v, int n_c,
                               const int32_t* pts_vn, int n_vn, const int32_t* pts_nn, int n_nn,
                               const double* w_vn, const double* w_nn, const double* v_vn,
                               double* sigma_sex_x, double* sigma_x, double* sigma_coh,
                               double* sigma_total);
/* The same on device arrays (psi with leading dim ldp; W / V blocks n x n,
 * ld n; point arrays on the host; device outputs, no finiteness check). */
int lrgw_dev_self_energies(lrgw_ctx ctx, const double* psi, long long ldp, int n_r, int n_v, int n_c,
                           const int32_t* pts_vn, int n_vn, const int32_t* pts_nn, int n_nn,
                           const double* w_vn, const double* w_nn, const double* v_vn,
                           double* sigma_sex_x, double* sigma_x, double* sigma_coh);

/* WFN1 orbital files (reference model.hpp:236-339, save_system /
 * load_system): "WFN1", uint32 LE header length, JSON header
 * {cell, dims, nc, nr, nv}, f64 LE psi (column major), energies, vxc.
 * Failures return LRGW_ERR_IO with the reference's io_error message in
 * lrgw_last_error() (thread-local; the context-free calls' error text). */
const char* lrgw_last_error(void);
int lrgw_wfn1_info(const char* path, int* dims3, double* cell3, int* n_v, int* n_c);
/* Host load: psi (n_r x (n_v + n_c)), energies, vxc (n_v + n_c); any may be null. */
int lrgw_wfn1_load(const char* path, double* psi, double* energies, double* vxc);
/* Device load: psi streamed straight into HBM (leading dim ld >= n_r) in
 * column blocks through pinned double buffers; energies / vxc to the host. */
int lrgw_wfn1_load_device(lrgw_ctx ctx, const char* path, double* psi, long long ld, double* energies,
                          double* vxc);
int lrgw_wfn1_save(const char* path, const int* dims3, const double* cell3, int n_v, int n_c,
                   const double* psi, const double* energies, const double* vxc);

/* Stage-level device entry points (multi-rank orchestration composes these). */
int lrgw_dev_select(lrgw_ctx ctx, const double* a, long long lda, int n1, const double* b,
                    long long ldb, int n2, int n_r, int n_mu, int32_t* pts_host,
                    double* min_margin);
int lrgw_dev_fit(lrgw_ctx ctx, const double* a, long long lda, int n1, const double* b,
                 long long ldb, int n2, int n_r, const int32_t* pts_host, int n_mu,
                 double* theta, long long ldt);
/* Fit for a row panel [row0, row0 + rows) of Theta given the full point-row
 * factors a_mu (n_mu x n1) and b_mu (n_mu x n2): rank-local, no exchange. */
int lrgw_dev_fit_panel(lrgw_ctx ctx, const double* a, long long lda, int n1, const double* b,
                       long long ldb, int n2, int rows, const double* a_mu, const double* b_mu,
                       const double* g_inv, int n_mu, double* theta, long long ldt);
/* Partial node sum over nodes [node0, node0 + count) of an n_lambda-interval
 * trapezoid, unscaled (acc = sum w_k term_k, lower triangle mirrored). */
int lrgw_dev_contour_partial(lrgw_ctx ctx, const double* pv, long long ldv, const double* pc,
                             long long ldpc, int n_mu, int n_v, int n_c, const double* energies,
                             int n_e, int n_lambda, int node0, int count, double* acc);
int lrgw_dev_contour_fixed(lrgw_ctx ctx, const double* pv, long long ldv, const double* pc,
                           long long ldpc, int n_mu, int n_v, int n_c, const double* energies,
                           int n_e, int n_lambda, double* t, long long ldt);
int lrgw_dev_pvp(lrgw_ctx ctx, const int* dims, const double* cell, int zero_kernel,
                 const double* theta, long long ldt, int n_mu, double* pvp);
int lrgw_dev_smw_core(lrgw_ctx ctx, const double* t, const double* pvp, int n_mu, double* k);
int lrgw_dev_coulomb_apply(lrgw_ctx ctx, const int* dims, const double* cell, int zero_kernel,
                           const double* x, long long ldx, int m, double* y, long long ldy);
/* Plain FP64 GEMM through the path's DMMA engine: C = alpha op(A) op(B) + beta C,
 * trans = 'N' | 'T' (BLAS semantics). Exposed for tests and benchmarking. */
int lrgw_dev_dgemm(lrgw_ctx ctx, char trans_a, char trans_b, int m, int n, int k, double alpha,
                   const double* a, long long lda, const double* b, long long ldb, double beta,
                   double* c, long long ldc);
/* The ISDF Gram-pair Hadamard product through the path's engine (isdf.hpp:132):
 * C = (A1 B1^T) o (A2 B2^T), A1: m x k1, B1: n x k1, A2: m x k2, B2: n x k2, all
 * column-major. Exposed for tests and benchmarking. */
int lrgw_dev_hadamard(lrgw_ctx ctx, int m, int n, const double* a1, long long lda1, const double* b1,
                      long long ldb1, int k1, const double* a2, long long lda2, const double* b2, long long ldb2,
                      int k2, double* c, long long ldc);

/* In-place inverse of the lower triangle of a device matrix (n x n, column
 * major, ld lda); the strict upper triangle is left untouched. Singular ->
 * LRGW_ERR_SINGULAR with the pivot index. Exposed for tests. */
int lrgw_dev_trtri_lower(lrgw_ctx ctx, double* a, int n, long long lda);

/* Top s1 rows by (d desc, position asc) among rows with pos[r] >= k — the
 * candidate set of one selection block (device arrays; host outputs, rows of
 * missing entries are -1). Exposed for tests. */
int lrgw_dev_select_topk(lrgw_ctx ctx, const double* d, const int32_t* pos, int n_r, int k, int s1,
                         int32_t* rows_host, double* vals_host, int32_t* pos_host);

/* Certified greedy of one selection block (the controller-warp kernel of
 * lrgw_select_interpolation_points) on the s candidates' Schur block wcc
 * (device, s x s, ld s): top = the s+1 entries of lrgw_dev_select_topk (host
 * values / positions / rows); pos / perm (device, n_r each) are the position
 * bookkeeping, updated in place. Outputs: x (device, s x s, ld s) = L_sel^-1
 * (b x b lower, pivot order), the b accepted pivot rows (host), their
 * margins (host, optional) and b (host). Reference: linalg.hpp:26-111 steps
 * k .. k+b-1. Used by the multi-rank build (paper_2403_12340_b200/dist.py). */
/* Theta row panel from the selection factor: theta(:, colmap[q]) =
 * sum_{p >= q} L(:, p) X(p, q) with L the panel's pivoted-Cholesky factor
 * (rows x n_mu, pivot order), X = L_P^-1 (device, lower, ld ldx) and colmap
 * (host) the sorted-point rank of pivot q — the fused fit of lrgw_build
 * (isdf.hpp:132-170 Theta = Z C^T (C C^T)^-1 in factored form) for one
 * rank's panel. */
int lrgw_dev_theta_from_factor(lrgw_ctx ctx, const double* l, long long ldl, int rows, int n_mu,
                               const double* x, long long ldx, const int32_t* colmap_host,
                               double* theta, long long ldt);

/* One selection block's panel update on a rank's rows [r0, r0 + rows):
 *   W = (A A_sel^T) o (B B_sel^T) - L[:, :k] L_sel^T     (rows x nb)
 *   L[:, k:k+nb] = W X^T,  d -= rowsum(L[:, k:k+nb]^2) where pos >= k + nb
 * with piv = [A_sel | B_sel | L_sel] (device, nb x (n1 + n2 + k), column
 * major, ld ldpiv) the accepted pivots' rows, X = L_sel^-1 (device, ld ldx)
 * from lrgw_dev_cand_greedy, L (device, ld rows) and d, pos (device, the
 * panel's residual diagonal and positions). The tail of one block of
 * lrgw_select_interpolation_points (linalg.hpp:60-100 for steps k..k+nb-1). */
int lrgw_dev_select_panel_update(lrgw_ctx ctx, const double* a, long long lda, int n1, const double* b,
                                 long long ldb, int n2, int rows, double* l, long long ldl, int k, int nb,
                                 const double* piv, long long ldpiv, const double* x, long long ldx,
                                 const int32_t* pos, double* d);

/* out = X^T diag(w) X (m x m, symmetric) for X (device, kdim x m, column
 * major, ld ldx) and w (device, kdim) — the weighted G-space SYRK of
 * Theta^T V Theta (smw.hpp:61-62) on one rank's G-slab, with X the slab's
 * spectrum viewed as interleaved reals and w the Hermitian-weighted v(G)/N_r
 * repeated for the real and imaginary parts. Lower-triangle DMMA tiles +
 * mirror. */
int lrgw_dev_gram_weighted(lrgw_ctx ctx, const double* x, long long ldx, int kdim, int m, const double* w,
                           double* out, long long ldo);

int lrgw_dev_cand_greedy(lrgw_ctx ctx, int n_r, int s, int steps, int k, const double* top_vals,
                         const int32_t* top_pos, const int32_t* top_rows, const double* wcc, int32_t* pos,
                         int32_t* perm, double* x, int32_t* piv_rows_host, double* margins_host,
                         int32_t* b_host);


/* ---- dense utility layer of the reference API (host buffers) --------------
 * The drop-in headers' matrix.hpp / linalg.hpp / dft.hpp / isdf.hpp helpers
 * over the device: DMMA products, cuSOLVER factorisations with the
 * reference's singularity rule, QRCP pivots from the path's greedy selection. */
/* C = op(A) op(B), op = 'N' | 'T' (matrix.hpp:71-120 matmul / matmul_tn / matmul_nt). */
int lrgw_matmul(lrgw_ctx ctx, char trans_a, char trans_b, int m, int n, int k, const double* a, long long lda,
                const double* b, long long ldb, double* c, long long ldc);
/* linalg.hpp:117-150: partial-pivot LU; piv[i] = row swapped with row i at step i;
 * LRGW_ERR_SINGULAR (pivot index) when |u_ii| < 1e-14 max|A|. */
int lrgw_lu_factor(lrgw_ctx ctx, const double* a, int n, double* lu, int32_t* piv, double* max_abs);
/* linalg.hpp:152-175: X = A^-1 B from the factors (B n x nrhs). */
int lrgw_lu_solve_factored(lrgw_ctx ctx, const double* lu, const int32_t* piv, int n, const double* b, int nrhs,
                           double* x);
/* linalg.hpp:190-345: ascending eigenvalues; eigenvectors in the columns of q (may be NULL). */
int lrgw_sym_eig(lrgw_ctx ctx, const double* a, int n, double* values, double* q);
/* linalg.hpp:17-111: A P = Q R; perm (n) = columns in selection order, q (m x k), r (k x n), k = min(m, n). */
int lrgw_qrcp(lrgw_ctx ctx, const double* a, int m, int n, int32_t* perm, double* q, double* r);
/* dft.hpp:37-68: unitary 3-D DFT of an interleaved complex grid vector (x, y: 2 n_r doubles). */
int lrgw_dft(lrgw_ctx ctx, const int* dims, const double* x, int inverse, double* y);
/* apply_coulomb with the operator's own kernel array (CoulombOperator::kernel, N_r values). */
int lrgw_apply_coulomb_kernel(lrgw_ctx ctx, const int* dims, const double* kernel, const double* x, int m, double* y);
/* isdf.hpp:49-88: the pair matrix (N_r x N1 N2) or its transpose, 2^26-entry guard. */
int lrgw_pair_matrix(lrgw_ctx ctx, const double* a, const double* b, int n_r, int n1, int n2, int transposed,
                     double* out);

/* ---- multi-rank build (one process per GPU) -------------------
 * A communicator carries the build's few exchanges between the ranks of one
 * box: NCCL over NVLink / NVSwitch (device buffers, the context's stream), or
 * a caller-supplied host transport (any runtime that can move host bytes:
 * MPI, torch.distributed gloo, ...; device payloads are staged through
 * pinned host buffers). Grid rows are split into contiguous z-plane panels:
 * rank p owns rows [row0, row0 + rows) of lrgw_z_panel. */
typedef struct lrgw_comm_s* lrgw_comm;

/* Host transport callbacks (return 0 on success); rank order everywhere. */
typedef struct {
  void* user;
  /* in-place element-wise sum of `count` doubles over all ranks */
  int (*allreduce_sum_f64)(void* user, double* buf, long long count);
  /* recv (world * bytes) = every rank's `bytes` of send, rank order */
  int (*allgather)(void* user, const void* send, void* recv, long long bytes);
  /* send block q (send_bytes[q], packed in rank order) goes to rank q; recv
   * block p (recv_bytes[p], packed in rank order) comes from rank p */
  int (*alltoallv)(void* user, const void* send, const long long* send_bytes, void* recv,
                   const long long* recv_bytes);
} lrgw_host_transport;

/* 1 when libnccl.so.2 can be loaded (dlopen; no link-time dependency). */
int lrgw_nccl_available(void);
/* rank 0 makes the id (128 bytes) and shares it with the other ranks. */
int lrgw_nccl_unique_id(unsigned char id[128]);
int lrgw_comm_create_nccl(lrgw_ctx ctx, int rank, int world, const unsigned char id[128], lrgw_comm* out);
int lrgw_comm_create_host(int rank, int world, const lrgw_host_transport* transport, lrgw_comm* out);
int lrgw_comm_destroy(lrgw_comm comm);
int lrgw_comm_info(lrgw_comm comm, int* rank, int* world);
/* This rank's grid-row panel: whole z-planes [z0, z1) of the n3 planes,
 * z_p = floor(n3 p / world) (requires n3 >= world). */
int lrgw_z_panel(const int* dims, int world, int rank, int* row0, int* rows);

/* The factored eps^-1 build (stages 1-5) across the ranks of `comm`, each
 * rank passing its OWN panel of the orbitals (rows x n_v and rows x n_c
 * device arrays, rows from lrgw_z_panel) and the full energies:
 *   1 selection: per candidate block the local top-(s+1) by (residual,
 *     position) is all-gathered and merged on the device; the candidates'
 *     rows [Phi_v | Phi_c | L] are owner-contributed (one all-reduce); the
 *     certified greedy runs replicated (identical on every rank); each rank
 *     updates its panel of the factor L and of the residual diagonal
 *   2 fit: Theta panel = L panel L_P^-1 (L_P owner-contributed)
 *   3 quadrature nodes split across ranks, all-reduce of the partial core
 *   4-5 slab 3-D FFT of the Theta panel (2-D transforms of the owned planes,
 *     one all-to-all to y-pencils, 1-D transforms along z), the G-slab
 *     Theta^T V Theta SYRK, all-reduce; SMW core replicated.
 * The handle keeps the rank's Theta panel (lrgw_eps_info: theta is rows x
 * n_mu) and replicated K, T, Theta^T V Theta and points. world == 1 is the
 * one-GPU build. Stage device times: lrgw_ctx_stage_ms (this rank). */
int lrgw_build_sharded(lrgw_ctx ctx, lrgw_comm comm, const lrgw_build_params* prm, const double* phi_v,
                       long long ldv, const double* phi_c, long long ldc, const double* energies,
                       lrgw_eps* out);
/* y = eps^-1 x on this rank's panel rows (device x, y: rows x m): u =
 * all-reduce(Theta_p^T x_p), z_p = Theta_p (K u), V z from the all-gathered
 * z, y_p = x_p + (V z)_p (smw.hpp:97-103). */
int lrgw_eps_apply_sharded(lrgw_ctx ctx, lrgw_comm comm, lrgw_eps e, const double* x, long long ldx, int m,
                           double* y, long long ldy);

#ifdef __cplusplus
}
#endif

#endif /* LRGW_CUDA_H_ */
