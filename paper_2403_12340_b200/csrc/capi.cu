// capi.cu — the C-ABI of liblrgw_cuda.so (include/lrgw_cuda.h).
//
// Host orchestration of the B200 hot path: context (stream, cuSOLVER handle,
// cuFFT plan cache), device scratch through the stream-ordered allocator,
// stage timing with CUDA events, and the mapping of every failure onto the
// reference exception taxonomy (errors.hpp:10-36). Stage math lives in the
// kernels (gemm.cu, quadrature.cu, select.cu, coulomb.cu, misc.cu); cuFFT
// and cuSOLVER are used only as leaf calls (3-D FFT, N_mu x N_mu factors).
#include <cufft.h>
#include <cusolverDn.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <set>
#include <unordered_map>
#include <string>
#include <tuple>
#include <vector>

#include "elliptic.h"
#include "kernels.h"
#include "lrgw_cuda.h"
#include "select.h"
#include "wfn1.h"

namespace lrgw_dev {
static std::atomic<long long> g_launches{0};
long long launch_count() { return g_launches.load(); }
void count_launches(int n) { g_launches += n; }
}  // namespace lrgw_dev

using namespace lrgw_dev;

#include "internal.h"

using namespace lrgw_impl;


namespace lrgw_impl {

void release_cached(lrgw_ctx c) {  // caller holds mem_mu
  if (c->mem_free.empty()) return;
  cudaStreamSynchronize(c->stream);
  for (auto& kv : c->mem_free) cudaFree(kv.second);
  c->mem_free.clear();
  c->mem_cached = 0;
}

// Stream-ordered allocation from the context cache: a cached block of at least
// the (rounded) size and at most 1/4 larger is reused; otherwise the driver
// allocates, after dropping the cache if memory is short.
void* ctx_alloc(lrgw_ctx c, size_t bytes) {
  const size_t gran = bytes < (1u << 20) ? 512 : (2u << 20);
  const size_t want = (bytes + gran - 1) / gran * gran;
  std::lock_guard<std::mutex> lk(c->mem_mu);
  auto it = c->mem_free.lower_bound(want);
  if (it != c->mem_free.end() && it->first <= want + want / 4) {
    void* p = it->second;
    c->mem_live[p] = it->first;
    c->mem_cached -= it->first;
    c->mem_free.erase(it);
    return p;
  }
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, want);
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    release_cached(c);
    e = cudaMalloc(&p, want);
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    fail(LRGW_ERR_CUDA, std::string("device allocation of ") + std::to_string(bytes) + " bytes: " +
                            cudaGetErrorString(e));
  }
  c->mem_live[p] = want;
  return p;
}

// Return a block to the cache. Work already queued on the context stream may
// still use it; every later user is ordered behind that work on the same stream.
void ctx_free(lrgw_ctx c, void* p) {
  if (!p) return;
  std::lock_guard<std::mutex> lk(c->mem_mu);
  auto it = c->mem_live.find(p);
  if (it == c->mem_live.end()) return;
  c->mem_free.emplace(it->second, p);
  c->mem_cached += it->second;
  c->mem_live.erase(it);
}



DBuf upload(lrgw_ctx c, const double* h, size_t n) {
  DBuf b = dalloc(c, n);
  if (n) ck(cudaMemcpyAsync(b.p, h, n * sizeof(double), cudaMemcpyHostToDevice, c->stream), "H2D");
  return b;
}

DBuf upload_i(lrgw_ctx c, const int32_t* h, size_t n) {
  DBuf b = ialloc(c, n);
  if (n) ck(cudaMemcpyAsync(b.p, h, n * sizeof(int), cudaMemcpyHostToDevice, c->stream), "H2D");
  return b;
}

void download(lrgw_ctx c, void* h, const void* d, size_t bytes) {
  if (bytes) ck(cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, c->stream), "D2H");
  ck(cudaStreamSynchronize(c->stream), "sync");
}

void use_device(lrgw_ctx c) { ck(cudaSetDevice(c->device), "cudaSetDevice"); }

lrgw_eps_s* new_eps(lrgw_ctx c) {
  auto* e = new lrgw_eps_s;
  e->ctx = c;
  std::lock_guard<std::mutex> lk(c->mem_mu);
  c->live_eps.insert(e);
  return e;
}

// Stage boundary i of the build (no-op outside lrgw_build).
// Stage boundary of lrgw_build: CUDA event for the stage timings plus an NVTX
// range per stage (profilers attribute kernels to stages; a no-op otherwise).
void mark(lrgw_ctx c, int i) {
  static const char* const names[LRGW_STAGE_TOTAL] = {"select", "fit_lhs", "fit_solve", "fit_gemm",
                                                        "contour", "fft", "pvp", "smw"};
  if (!c->timing) return;
  ck(cudaEventRecord(c->ev[i], c->stream), "cudaEventRecord");
  if (i > 0) nvtxRangePop();
  if (i < LRGW_STAGE_TOTAL) nvtxRangePushA(names[i]);
}

lrgw_host::Spec spec_from7(const double* s7) {
  lrgw_host::Spec s;
  s.q = s7[0];
  s.big_q = s7[1];
  s.r = s7[2];
  s.big_r = s7[3];
  s.l = s7[4];
  s.e_shift = s7[5];
  s.bypass = s7[6] != 0.0;
  return s;
}

void spec_to7(const lrgw_host::Spec& s, double* o) {
  o[0] = s.q;
  o[1] = s.big_q;
  o[2] = s.r;
  o[3] = s.big_r;
  o[4] = s.l;
  o[5] = s.e_shift;
  o[6] = s.bypass ? 1.0 : 0.0;
}

void check_grid(const int* dims, const double* cell) {
  for (int i = 0; i < 3; ++i) {
    if (dims[i] < 2) fail(LRGW_ERR_INVALID_INPUT, "Grid: all dims must be >= 2");
    if (!(cell[i] > 0.0)) fail(LRGW_ERR_INVALID_INPUT, "Grid: cell lengths must be > 0");
  }
}

// ---------------------------------------------------------------------------
// cuFFT plans (leaf): batched 3-D D2Z / Z2D over columns, dims {n3, n2, n1}
// row-major = the grid's linear index i1 + n1 (i2 + n2 i3) (grid.hpp:11).
// ---------------------------------------------------------------------------
cufftHandle get_plan(lrgw_ctx c, const int* dims, int batch, long long rdist, long long cdist,
                     bool forward) {
  const auto key = std::make_tuple(dims[0], dims[1], dims[2], batch, rdist, cdist, forward ? 1 : 0);
  auto it = c->plans.find(key);
  if (it != c->plans.end()) return it->second;
  cufftHandle plan;
  long long n[3] = {dims[2], dims[1], dims[0]};
  long long rembed[3] = {dims[2], dims[1], dims[0]};
  long long cembed[3] = {dims[2], dims[1], dims[0] / 2 + 1};
  ckf(cufftCreate(&plan), "cufftCreate");
  size_t work = 0;
  if (forward)
    ckf(cufftMakePlanMany64(plan, 3, n, rembed, 1, rdist, cembed, 1, cdist, CUFFT_D2Z, batch, &work),
        "cufftMakePlanMany64(D2Z)");
  else
    ckf(cufftMakePlanMany64(plan, 3, n, cembed, 1, cdist, rembed, 1, rdist, CUFFT_Z2D, batch, &work),
        "cufftMakePlanMany64(Z2D)");
  ckf(cufftSetStream(plan, c->stream), "cufftSetStream");
  c->plans[key] = plan;
  return plan;
}

long long half_len(const int* dims) { return (long long)(dims[0] / 2 + 1) * dims[1] * dims[2]; }

// xhat (complex, half spectrum, column stride half_len) = D2Z(x)
// Columns per cuFFT execution: bounds the plan's work area (a single plan
// over all 8192 Theta columns of Si512 would ask cuFFT for a Theta-sized
// work buffer next to the 58 GB Theta and its 59 GB spectrum).
int fft_batch() {
  static const int v = getenv("LRGW_FFT_BATCH") ? std::max(1, atoi(getenv("LRGW_FFT_BATCH"))) : 1024;
  return v;
}

void fft_forward(lrgw_ctx c, const int* dims, const double* x, long long ldx, int m, double* xhat) {
  const long long nh = half_len(dims);
  if (fft_own_enabled()) {  // the two-pass shared-memory D2Z (fft.cu) where the axes allow it
    const cudaError_t e = fft_d2z_3d(c->stream, dims, x, ldx, m, xhat, c->sm_count);
    if (e != cudaErrorNotSupported) {
      ck(e, "fft_d2z_3d");
      return;
    }
    cudaGetLastError();
  }
  const int fb = fft_batch();
  for (int j0 = 0; j0 < m; j0 += fb) {
    const int b = std::min(fb, m - j0);
    cufftHandle plan = get_plan(c, dims, b, ldx, nh, true);
    ckf(cufftExecD2Z(plan, const_cast<double*>(x) + (size_t)j0 * ldx,
                     reinterpret_cast<cufftDoubleComplex*>(xhat + (size_t)j0 * 2 * nh)),
        "cufftExecD2Z");
  }
}

void fft_inverse(lrgw_ctx c, const int* dims, double* xhat, int m, double* y, long long ldy) {
  const long long nh = half_len(dims);
  const int fb = fft_batch();
  for (int j0 = 0; j0 < m; j0 += fb) {
    const int b = std::min(fb, m - j0);
    cufftHandle plan = get_plan(c, dims, b, ldy, nh, false);
    ckf(cufftExecZ2D(plan, reinterpret_cast<cufftDoubleComplex*>(xhat + (size_t)j0 * 2 * nh), y + (size_t)j0 * ldy),
        "cufftExecZ2D");
  }
}

// y = V x = Re(F^-1 diag(v) F x) (model.hpp:208-223)
void coulomb_apply(lrgw_ctx c, const int* dims, const double* cell, int zero, const double* x,
                   long long ldx, int m, double* y, long long ldy) {
  if (m <= 0) return;
  const long long nh = half_len(dims);
  DBuf xh = dalloc(c, (size_t)2 * nh * m);
  fft_forward(c, dims, x, ldx, m, xh.d());
  ck(coulomb_scale_half(c->stream, dims[0], dims[1], dims[2], cell[0], cell[1], cell[2], zero, xh.d(), m),
     "coulomb_scale_half");
  fft_inverse(c, dims, xh.d(), m, y, ldy);
}


Work make_work(lrgw_ctx c, size_t elems) {
  Work w;
  w.buf = dalloc(c, elems);
  w.elems = elems;
  return w;
}

void gemm(lrgw_ctx c, int M, int N, int K, const double* A, long long lda, Lay la, const double* B,
          long long ldb, Lay lb, double* C, long long ldc, double alpha, double beta,
          const double* scale, bool lower, Work* w) {
  ck(dgemm(c->stream, M, N, K, A, lda, la, B, ldb, lb, C, ldc, alpha, beta, scale, lower, c->sm_count,
           w ? w->buf.d() : nullptr, w ? w->elems : 0),
     "dgemm");
}

// pvp = Theta^T V Theta via the half-spectrum G-space SYRK (smw.hpp:61-62):
// one batched D2Z of Theta (cuFFT leaf), then a lower-triangle DMMA GEMM over
// K = 2 * half_len interleaved reals with w_G v(G)/N_r fused as the scale.
void pvp_impl(lrgw_ctx c, const int* dims, const double* cell, int zero, const double* theta,
              long long ldt, int n_mu, double* pvp) {
  const long long nh = half_len(dims);
  DBuf xh = dalloc(c, (size_t)2 * nh * n_mu);
  fft_forward(c, dims, theta, ldt, n_mu, xh.d());
  mark(c, 6);
  DBuf wts = dalloc(c, (size_t)2 * nh);
  ck(coulomb_half_weights(c->stream, dims[0], dims[1], dims[2], cell[0], cell[1], cell[2], zero, wts.d()),
     "coulomb_half_weights");
  Work w = make_work(c, (size_t)16 * n_mu * n_mu);
  gemm(c, n_mu, n_mu, (int)(2 * nh), xh.d(), 2 * nh, Lay::K, xh.d(), 2 * nh, Lay::K, pvp, n_mu, 1.0, 0.0,
       wts.d(), true, &w);
  ck(mirror_lower(c->stream, pvp, n_mu, n_mu, false), "mirror");
}

// Projected screened interactions (gw.hpp:73-88) from the factored inverse:
//   B_x = P_x^T V P_vc,  W_x = B_x K B_x^T  (x = vn, nn),  V_vn = P_vn^T V P_vn.
// Every N_r contraction runs in G space over the half spectrum, like pvp_impl:
// one D2Z per operand (P_vc's spectrum shared by both B), then DMMA GEMMs
// with w_G v(G)/N_r fused as the k-scale — B_x is a cross GEMM, V_vn a
// lower-tile SYRK. The N_mu-sized products are lower-tile GEMMs, mirrored
// (exactly symmetric, the reference's symmetrize).
void project_impl(lrgw_ctx c, const lrgw_eps_s* e, const double* p_vn, long long ld_vn, int n_vn,
                  const double* p_nn, long long ld_nn, int n_nn, double* w_vn, double* w_nn, double* v_vn) {
  const int n_mu = e->n_mu;
  const long long nh = half_len(e->dims);
  DBuf xvc = dalloc(c, (size_t)2 * nh * n_mu);
  fft_forward(c, e->dims, e->theta, e->n_r, n_mu, xvc.d());
  DBuf wts = dalloc(c, (size_t)2 * nh);
  ck(coulomb_half_weights(c->stream, e->dims[0], e->dims[1], e->dims[2], e->cell[0], e->cell[1], e->cell[2],
                          e->zero, wts.d()),
     "coulomb_half_weights");
  const int nmax = std::max({n_vn, n_nn, n_mu});
  Work w = make_work(c, (size_t)16 * nmax * nmax);
  DBuf b = dalloc(c, (size_t)nmax * n_mu), bk = dalloc(c, (size_t)nmax * n_mu);
  auto one = [&](const double* px, long long ldx, int nx, double* wx, double* vx) {
    if (nx <= 0) return;
    DBuf xh = dalloc(c, (size_t)2 * nh * nx);
    fft_forward(c, e->dims, px, ldx, nx, xh.d());
    // B = P_x^T V P_vc (nx x n_mu): k = interleaved half-spectrum reals
    gemm(c, nx, n_mu, (int)(2 * nh), xh.d(), 2 * nh, Lay::K, xvc.d(), 2 * nh, Lay::K, b.d(), nx, 1.0, 0.0,
         wts.d(), false, &w);
    // B K (K symmetric), then W = (B K) B^T on lower tiles
    gemm(c, nx, n_mu, n_mu, b.d(), nx, Lay::MN, e->k, n_mu, Lay::MN, bk.d(), nx, 1.0, 0.0);
    gemm(c, nx, nx, n_mu, bk.d(), nx, Lay::MN, b.d(), nx, Lay::MN, wx, nx, 1.0, 0.0, nullptr, true, &w);
    ck(mirror_lower(c->stream, wx, nx, nx, false), "mirror");
    if (vx) {
      gemm(c, nx, nx, (int)(2 * nh), xh.d(), 2 * nh, Lay::K, xh.d(), 2 * nh, Lay::K, vx, nx, 1.0, 0.0, wts.d(),
           true, &w);
      ck(mirror_lower(c->stream, vx, nx, nx, false), "mirror");
    }
  };
  one(p_vn, ld_vn, n_vn, w_vn, v_vn);
  one(p_nn, ld_nn, n_nn, w_nn, nullptr);
}

// Static-COHSEX self-energy diagonals (gw.hpp:93-137, sigma_hadamard) on
// the device: Psi rows at the vn / nn points (gather), the occupied and
// all-band masks as lower-tile DMMA SYRKs, H o M in place, (H o M) Psi as a
// DMMA GEMM and the per-band column dot with the sign / 1/2 folded in:
//   sex_x = -diag(Psi_vn^T (W_vn o M_occ) Psi_vn), x = -diag(... V_vn ...),
//   coh = 1/2 diag(Psi_nn^T (W_nn o M_all) Psi_nn).
void sigma_impl(lrgw_ctx c, const double* psi, long long ldp, int n_v, int nb, const int32_t* pts_vn,
                int n_vn, const int32_t* pts_nn, int n_nn, const double* w_vn, const double* v_vn,
                const double* w_nn, double* sex_x, double* sx, double* coh) {
  const int nmax = std::max(n_vn, n_nn);
  Work w = make_work(c, (size_t)16 * std::max(nmax, 1) * std::max(nmax, 1));
  DBuf mask = dalloc(c, (size_t)nmax * nmax), hm = dalloc(c, (size_t)nmax * nmax);
  auto one_set = [&](const int32_t* pts, int n, int n_occ, const double* h1, double* out1, double a1,
                     const double* h2, double* out2, double a2) {
    DBuf dp = upload_i(c, pts, n);
    DBuf ps = dalloc(c, (size_t)n * nb), hp = dalloc(c, (size_t)n * nb);
    ck(gather_rows(c->stream, psi, ldp, nb, dp.i(), n, ps.d(), n), "gather");
    // M = Psi_o Psi_o^T (n x n, lower tiles + mirror)
    if (n_occ > 0) {
      gemm(c, n, n, n_occ, ps.d(), n, Lay::MN, ps.d(), n, Lay::MN, mask.d(), n, 1.0, 0.0, nullptr, true, &w);
      ck(mirror_lower(c->stream, mask.d(), n, n, false), "mirror");
    } else {
      ck(fill(c->stream, mask.d(), (size_t)n * n, 0.0), "fill");
    }
    auto diag = [&](const double* h, double* out, double alpha) {
      ck(cudaMemcpyAsync(hm.d(), mask.d(), sizeof(double) * n * n, cudaMemcpyDeviceToDevice, c->stream), "D2D");
      ck(hadamard_inplace(c->stream, n, h, n, hm.d(), n), "hadamard");
      // hp = (H o M) Psi: B(band, nu) = Psi(nu, band) is K-contiguous
      gemm(c, n, nb, n, hm.d(), n, Lay::MN, ps.d(), n, Lay::K, hp.d(), n, 1.0, 0.0);
      ck(col_dot(c->stream, n, nb, ps.d(), n, hp.d(), n, alpha, out), "col_dot");
    };
    diag(h1, out1, a1);
    if (h2) diag(h2, out2, a2);
  };
  if (n_vn > 0) {
    one_set(pts_vn, n_vn, n_v, w_vn, sex_x, -1.0, v_vn, sx, -1.0);
  } else {
    ck(fill(c->stream, sex_x, nb, 0.0), "fill");
    ck(fill(c->stream, sx, nb, 0.0), "fill");
  }
  if (n_nn > 0) {
    one_set(pts_nn, n_nn, nb, w_nn, coh, 0.5, nullptr, nullptr, 0.0);
  } else {
    ck(fill(c->stream, coh, nb, 0.0), "fill");
  }
}

void check_points(const int32_t* pts, int n, int n_r, const char* what) {
  if (n > 0 && !pts) fail(LRGW_ERR_INVALID_INPUT, std::string(what) + ": null point array");
  for (int i = 0; i < n; ++i)
    if (pts[i] < 0 || pts[i] >= n_r) fail(LRGW_ERR_INVALID_INPUT, std::string(what) + ": point index out of range");
}

// ---------------------------------------------------------------------------
// Dense N_mu x N_mu leaf factorisations (cuSOLVER).
// ---------------------------------------------------------------------------
double dev_max_abs(lrgw_ctx c, const double* x, size_t n) {
  DBuf r = dalloc(c, 512);
  ck(max_abs(c->stream, x, n, r.d()), "max_abs");
  double h = 0;
  download(c, &h, r.d() + 296, sizeof(double));
  return h;
}

// In-place Cholesky of an SPD matrix (lower). Returns info (0 = ok).
int potrf_lower(lrgw_ctx c, double* a, int n) {
  int lwork = 0;
  cks(cusolverDnDpotrf_bufferSize(c->solver, CUBLAS_FILL_MODE_LOWER, n, a, n, &lwork), "potrf_bufferSize");
  DBuf work = dalloc(c, (size_t)std::max(lwork, 1));
  DBuf info = ialloc(c, 1);
  if (c->timing) ck(cudaEventRecord(c->ev_lib[0], c->stream), "cudaEventRecord");
  cks(cusolverDnDpotrf(c->solver, CUBLAS_FILL_MODE_LOWER, n, a, n, work.d(), lwork, info.i()), "potrf");
  if (c->timing) ck(cudaEventRecord(c->ev_lib[1], c->stream), "cudaEventRecord");
  int h = 0;
  download(c, &h, info.p, sizeof(int));
  float ms = 0.0f;
  if (c->timing && cudaEventElapsedTime(&ms, c->ev_lib[0], c->ev_lib[1]) == cudaSuccess) c->lib_ms += ms;
  return h;
}

void potri_lower(lrgw_ctx c, double* a, int n) {
  int lwork = 0;
  cks(cusolverDnDpotri_bufferSize(c->solver, CUBLAS_FILL_MODE_LOWER, n, a, n, &lwork), "potri_bufferSize");
  DBuf work = dalloc(c, (size_t)std::max(lwork, 1));
  DBuf info = ialloc(c, 1);
  cks(cusolverDnDpotri(c->solver, CUBLAS_FILL_MODE_LOWER, n, a, n, work.d(), lwork, info.i()), "potri");
  int h = 0;
  download(c, &h, info.p, sizeof(int));
  if (h != 0) fail(LRGW_ERR_SINGULAR, "potri: singular factor", h - 1);
  ck(mirror_lower(c->stream, a, n, n, false), "mirror");
}

// Smallest |L_kk|^2 of a Cholesky factor against the LU threshold
// 1e-14 * max|A| (linalg.hpp:128, 137). Returns the offending index or -1.
int tiny_pivot(lrgw_ctx c, const double* chol, int n, double max_abs_a) {
  std::vector<double> diag(n);
  // n is N_mu (<= a few thousand): one D2H of the factor's diagonal via a strided copy
  ck(cudaMemcpy2DAsync(diag.data(), sizeof(double), chol, (size_t)(n + 1) * sizeof(double), sizeof(double),
                       n, cudaMemcpyDeviceToHost, c->stream),
     "D2H diag");
  ck(cudaStreamSynchronize(c->stream), "sync");
  const double tiny = 1e-14 * (max_abs_a > 0.0 ? max_abs_a : 1.0);
  for (int i = 0; i < n; ++i)
    if (diag[i] * diag[i] < tiny) return i;
  return -1;
}

// Inverse of the symmetric ISDF Gram via LU with the reference singularity
// rule (linalg.hpp:123-150); on a tiny pivot, the truncated-eigenvalue
// pseudo-inverse of isdf.hpp:144-161. ginv is overwritten (n x n).
void gram_inverse(lrgw_ctx c, const double* gram, int n, double* ginv) {
  const double mx = dev_max_abs(c, gram, (size_t)n * n);
  const double tiny = 1e-14 * (mx > 0.0 ? mx : 1.0);
  DBuf lu = dalloc(c, (size_t)n * n);
  ck(cudaMemcpyAsync(lu.p, gram, sizeof(double) * n * n, cudaMemcpyDeviceToDevice, c->stream), "D2D");
  int lwork = 0;
  cks(cusolverDnDgetrf_bufferSize(c->solver, n, n, lu.d(), n, &lwork), "getrf_bufferSize");
  DBuf work = dalloc(c, (size_t)std::max(lwork, 1));
  DBuf ipiv = ialloc(c, n);
  DBuf info = ialloc(c, 1);
  cks(cusolverDnDgetrf(c->solver, n, n, lu.d(), n, work.d(), ipiv.i(), info.i()), "getrf");
  std::vector<double> diag(n);
  ck(cudaMemcpy2DAsync(diag.data(), sizeof(double), lu.d(), (size_t)(n + 1) * sizeof(double), sizeof(double), n,
                       cudaMemcpyDeviceToHost, c->stream),
     "D2H diag");
  ck(cudaStreamSynchronize(c->stream), "sync");
  bool singular = false;
  for (int i = 0; i < n; ++i)
    if (!(std::abs(diag[i]) >= tiny)) singular = true;
  if (!singular) {
    ck(fill(c->stream, ginv, (size_t)n * n, 0.0), "fill");
    ck(add_diag(c->stream, ginv, n, n, 1.0), "add_diag");
    cks(cusolverDnDgetrs(c->solver, CUBLAS_OP_N, n, n, lu.d(), n, ipiv.i(), ginv, n, info.i()), "getrs");
    ck(mirror_lower(c->stream, ginv, n, n, true), "symmetrize");
    return;
  }
  // pseudo-inverse fallback (isdf.hpp:144-161)
  DBuf q = dalloc(c, (size_t)n * n);
  ck(cudaMemcpyAsync(q.p, gram, sizeof(double) * n * n, cudaMemcpyDeviceToDevice, c->stream), "D2D");
  DBuf w = dalloc(c, n);
  int lw2 = 0;
  cks(cusolverDnDsyevd_bufferSize(c->solver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, q.d(), n, w.d(),
                                  &lw2),
      "syevd_bufferSize");
  DBuf work2 = dalloc(c, (size_t)std::max(lw2, 1));
  cks(cusolverDnDsyevd(c->solver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, q.d(), n, w.d(), work2.d(),
                       lw2, info.i()),
      "syevd");
  std::vector<double> hw(n);
  int hinfo = 0;
  ck(cudaMemcpyAsync(&hinfo, info.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream), "D2H");
  download(c, hw.data(), w.p, sizeof(double) * n);
  if (hinfo != 0) fail(LRGW_ERR_NUMERIC, "fit_auxiliary_basis: eigensolver failed");
  double lam_max = 0.0;
  for (double v : hw) lam_max = std::max(lam_max, std::abs(v));
  if (lam_max <= 0.0) fail(LRGW_ERR_NUMERIC, "fit_auxiliary_basis: degenerate Gram matrix");
  std::vector<double> inv(n, 0.0);
  int kept = 0;
  for (int i = 0; i < n; ++i)
    if (std::abs(hw[i]) > 1e-12 * lam_max) {
      inv[i] = 1.0 / hw[i];
      ++kept;
    }
  if (kept == 0) fail(LRGW_ERR_NUMERIC, "fit_auxiliary_basis: degenerate Gram matrix");
  DBuf dinv = upload(c, inv.data(), n);
  // pinv = Q diag(inv) Q^T  (A = Q: MN, B = Q: MN, scale on k)
  gemm(c, n, n, n, q.d(), n, Lay::MN, q.d(), n, Lay::MN, ginv, n, 1.0, 0.0, dinv.d());
}

// In-place inverse of a lower-triangular factor (cuSOLVER trtri, leaf).
void trtri_lower(lrgw_ctx c, double* a, int n) {
  DBuf work = dalloc(c, trtri_work_elems(n));
  DBuf bad = ialloc(c, 1);
  const int big = 0x7fffffff;
  ck(cudaMemcpyAsync(bad.p, &big, sizeof(int), cudaMemcpyHostToDevice, c->stream), "H2D");
  ck(lrgw_dev::trtri_lower(c->stream, a, n, n, work.d(), bad.i(), c->sm_count), "trtri");
  int h = 0;
  download(c, &h, bad.p, sizeof(int));
  if (h != big) fail(LRGW_ERR_SINGULAR, "trtri: singular factor", h - 1);
}

// K = (T^-1/2 - P^T V P)^-1 (smw.hpp:42-73). T must be negative definite
// (the reference's sym_eig check, smw.hpp:47-51): -T = R R^T (Cholesky leaf;
// failure -> numeric_error, a pivot below the LU threshold -> singular). Then
//   T^-1/2 - P = -R^-T M R^-1,  M = I/2 + R^T P R  (SPD, >= I/2)
//   K = -R M^-1 R^T = -Z Z^T,   Z = R Q^-T,  M = Q Q^T
// i.e. two Cholesky factorisations and one triangular inverse (cuSOLVER
// leaves) plus four N_mu^3 DMMA GEMMs; K is symmetric by construction.
// Every check (the two potrf infos, the two tiny-pivot scans, the trtri flag)
// lands in one device status block read once at the end — one host sync
// instead of seven — and is evaluated in the order the steps run, so the
// first failing step names the error as before.
//
// Split in two so the build can overlap the first factorisation (it needs T
// only) with the Coulomb stage on a side stream: smw_factor_t enqueues
// R = chol(-T) and its checks on `st`; smw_finish the rest on the context
// stream (the caller orders the two).
enum { SMW_INFO_T, SMW_TINY_T, SMW_INFO_M, SMW_TINY_M, SMW_TRTRI_BAD, SMW_NSTAT };

struct SmwState {
  DBuf stat, mxb, r, pwork;  // held until the side stream is joined
  bool leaf_timed = false;
  cudaStream_t pending = nullptr;  // side stream not yet joined (error paths drain it)
  ~SmwState() {
    if (pending) cudaStreamSynchronize(pending);
  }
};

// Device status of the fused fit, read back with the SMW status (one host
// wait per build after the selection): diag = {min |L_ii|, max |L_ii|, ok}
// of L_P, bad = trtri's first zero pivot + 1 (0x7f7f7f7f: none).
struct FusedFit {
  DBuf diag, bad;
  double h[3] = {0.0, 0.0, 0.0};
  int hbad = 0;
  bool ok() const { return h[2] == 1.0 && hbad == 0x7f7f7f7f; }
  // (max |L_ii| / min |L_ii|)^2 is a lower bound on cond(G(P, P)) = cond(L_P)^2
  double ratio() const { return h[0] > 0.0 ? (h[1] / h[0]) * (h[1] / h[0]) : HUGE_VAL; }
};

void smw_factor_t(lrgw_ctx c, cudaStream_t st, const double* t, int n, SmwState& s) {
  const size_t nn = (size_t)n * n;
  s.stat = ialloc(c, SMW_NSTAT);
  s.mxb = dalloc(c, 2 * 512);
  s.r = dalloc(c, nn);
  int* sd = s.stat.i();
  ck(cudaMemsetAsync(sd, 0x7f, SMW_NSTAT * sizeof(int), st), "memset");
  int lwork = 0;
  cks(cusolverDnDpotrf_bufferSize(c->solver, CUBLAS_FILL_MODE_LOWER, n, s.r.d(), n, &lwork), "potrf_bufferSize");
  s.pwork = dalloc(c, (size_t)std::max(lwork, 1));
  ck(max_abs(st, t, nn, s.mxb.d()), "max_abs");
  ck(scale_copy(st, t, s.r.d(), nn, -1.0), "scale_copy");
  if (st != c->stream) cks(cusolverDnSetStream(c->solver, st), "cusolverDnSetStream");
  if (c->timing) ck(cudaEventRecord(c->ev_lib[0], st), "cudaEventRecord");
  const cusolverStatus_t ps = cusolverDnDpotrf(c->solver, CUBLAS_FILL_MODE_LOWER, n, s.r.d(), n, s.pwork.d(), lwork,
                                               sd + SMW_INFO_T);
  if (c->timing) ck(cudaEventRecord(c->ev_lib[1], st), "cudaEventRecord");
  if (st != c->stream) cks(cusolverDnSetStream(c->solver, c->stream), "cusolverDnSetStream");
  cks(ps, "potrf");
  s.leaf_timed = c->timing;
  ck(tiny_pivot_dev(st, s.r.d(), n, n, s.mxb.d() + 296, sd + SMW_TINY_T), "tiny_pivot");
  ck(zero_strict_upper(st, s.r.d(), n, n), "zero_upper");
  if (st != c->stream) s.pending = st;
}

// The context stream waits for the side stream's factorisation.
void smw_join(lrgw_ctx c, SmwState& s) {
  if (!s.pending) return;
  ck(cudaEventRecord(c->ev_join, s.pending), "cudaEventRecord");
  ck(cudaStreamWaitEvent(c->stream, c->ev_join, 0), "cudaStreamWaitEvent");
  s.pending = nullptr;
}

// false (and no SMW check raised): the fused fit's status in ff failed —
// Theta, and so pvp and K, must be rebuilt on the explicit path.
bool smw_finish(lrgw_ctx c, SmwState& s, const double* pvp, int n, double* k, FusedFit* ff = nullptr) {
  const size_t nn = (size_t)n * n;
  int* sd = s.stat.i();
  double* r = s.r.d();
  int lwork = 0;
  cks(cusolverDnDpotrf_bufferSize(c->solver, CUBLAS_FILL_MODE_LOWER, n, r, n, &lwork), "potrf_bufferSize");
  DBuf pwork = dalloc(c, (size_t)std::max(lwork, 1));
  Work w = make_work(c, 8 * nn);
  // Y = P R   (R lower: R(k, j) = 0 for k < j)
  DBuf y = dalloc(c, nn);
  ck(dgemm(c->stream, n, n, n, pvp, n, Lay::MN, r, n, Lay::K, y.d(), n, 1.0, 0.0, nullptr, false, c->sm_count,
           nullptr, 0, true, nullptr),
     "dgemm(PR)");
  // M = R^T Y + I/2 (lower tiles, mirrored)
  DBuf m = dalloc(c, nn);
  gemm(c, n, n, n, r, n, Lay::K, y.d(), n, Lay::K, m.d(), n, 1.0, 0.0, nullptr, true, &w);
  ck(mirror_lower(c->stream, m.d(), n, n, false), "mirror");
  ck(add_diag(c->stream, m.d(), n, n, 0.5), "add_diag");
  ck(max_abs(c->stream, m.d(), nn, s.mxb.d() + 512), "max_abs");
  if (c->timing) ck(cudaEventRecord(c->ev_lib[2], c->stream), "cudaEventRecord");
  cks(cusolverDnDpotrf(c->solver, CUBLAS_FILL_MODE_LOWER, n, m.d(), n, pwork.d(), lwork, sd + SMW_INFO_M), "potrf");
  if (c->timing) ck(cudaEventRecord(c->ev_lib[3], c->stream), "cudaEventRecord");
  ck(tiny_pivot_dev(c->stream, m.d(), n, n, s.mxb.d() + 512 + 296, sd + SMW_TINY_M), "tiny_pivot");
  ck(zero_strict_upper(c->stream, m.d(), n, n), "zero_upper");
  // Q^-1 (recursive DMMA trtri; a zero pivot -> TRTRI_BAD = its index + 1)
  {
    DBuf twork = dalloc(c, trtri_work_elems(n));
    ck(lrgw_dev::trtri_lower(c->stream, m.d(), n, n, twork.d(), sd + SMW_TRTRI_BAD, c->sm_count), "trtri");
  }
  // Z = R Q^-T ; K = -Z Z^T (lower tiles, mirrored)
  gemm(c, n, n, n, r, n, Lay::MN, m.d(), n, Lay::MN, y.d(), n, 1.0, 0.0);
  gemm(c, n, n, n, y.d(), n, Lay::MN, y.d(), n, Lay::MN, k, n, -1.0, 0.0, nullptr, true, &w);
  ck(mirror_lower(c->stream, k, n, n, false), "mirror");
  int h[SMW_NSTAT];
  if (ff) {
    ck(cudaMemcpyAsync(ff->h, ff->diag.p, sizeof(ff->h), cudaMemcpyDeviceToHost, c->stream), "D2H");
    ck(cudaMemcpyAsync(&ff->hbad, ff->bad.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream), "D2H");
  }
  download(c, h, sd, sizeof(h));
  if (c->timing) {
    float ms = 0.0f;
    double lib = 0.0;
    if (s.leaf_timed && cudaEventElapsedTime(&ms, c->ev_lib[0], c->ev_lib[1]) == cudaSuccess) lib += ms;
    if (cudaEventElapsedTime(&ms, c->ev_lib[2], c->ev_lib[3]) == cudaSuccess) lib += ms;
    c->lib_ms += lib;
  }
  if (ff && !ff->ok()) return false;
  const int unset = 0x7f7f7f7f;
  if (h[SMW_INFO_T] != 0)
    fail(LRGW_ERR_NUMERIC, "assemble_K: T is not negative definite (gapless or rank-deficient input)");
  if (h[SMW_TINY_T] >= 0) fail(LRGW_ERR_SINGULAR, "assemble_K: T singular", h[SMW_TINY_T]);
  if (h[SMW_INFO_M] != 0) fail(LRGW_ERR_SINGULAR, "assemble_K: middle matrix singular", 0);
  if (h[SMW_TINY_M] >= 0) fail(LRGW_ERR_SINGULAR, "assemble_K: middle matrix singular", h[SMW_TINY_M]);
  if (h[SMW_TRTRI_BAD] != unset) fail(LRGW_ERR_SINGULAR, "trtri: singular factor", h[SMW_TRTRI_BAD] - 1);
  return true;
}

cudaStream_t side_stream(lrgw_ctx c) {
  if (!c->side) {
    ck(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking), "cudaStreamCreate");
    ck(cudaEventCreateWithFlags(&c->ev_side, cudaEventDisableTiming), "event");
    ck(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming), "event");
  }
  return c->side;
}

void smw_core(lrgw_ctx c, const double* t, const double* pvp, int n, double* k) {
  SmwState s;
  smw_factor_t(c, c->stream, t, n, s);
  smw_finish(c, s, pvp, n, k);
}

// ---------------------------------------------------------------------------
// Stage 1: ISDF point selection (isdf.hpp:95-112) — see select.cu.
// ---------------------------------------------------------------------------
// Host mirror of select.cu's candidate entry (d, position, grid row).

// keep (optional): the pivoted-Cholesky factor L (n_r x steps, pivot order)
// and the pivot sequence, reused by the fused fit of lrgw_build.
bool fused_downdate_enabled() {
  static const bool on = !(getenv("LRGW_FUSED_DOWNDATE") && atoi(getenv("LRGW_FUSED_DOWNDATE")) == 0);
  return on;
}

bool select_trace() {
  static const bool on = getenv("LRGW_SELECT_TRACE") != nullptr;
  return on;
}


// Opt-in (LRGW_SELECT_DEVLOOP=1): measured no faster than the host loop —
// Si64 select 10.28 vs 10.12 ms, C60 42.5 vs 41.7 ms (profiles/r02/
// sweep_devloop.txt): the per-block read-back of nb costs less than the
// device loop's speculative last block and split-K W[C, C] update.
bool select_device_loop_enabled() {
  static const bool on = getenv("LRGW_SELECT_DEVLOOP") && atoi(getenv("LRGW_SELECT_DEVLOOP")) == 1;
  return on;
}

// The device loop's pinned read-back slots and event ring live in the context
// (cudaHostAlloc / cudaFreeHost synchronise the device: never per call).
int* select_pinned(lrgw_ctx c, size_t n) {
  if (c->sel_pinned_n < n) {
    if (c->sel_pinned) cudaFreeHost(c->sel_pinned);
    c->sel_pinned = nullptr;
    c->sel_pinned_n = 0;
    ck(cudaHostAlloc(reinterpret_cast<void**>(&c->sel_pinned), n * sizeof(int), cudaHostAllocDefault),
       "cudaHostAlloc");
    c->sel_pinned_n = n;
  }
  return c->sel_pinned;
}

// The per-block read of the accepted count b: the greedy writes b into a
// host-mapped pinned slot before its triangular-inverse tail and the host
// spins on it, so the panel's launches are queued while the greedy is still
// running (a cudaMemcpy + stream sync left the device idle ~30 us per block:
// D2H, the host wake-up and the first launch after it).
int* select_flag_arm(lrgw_ctx c) {
  if (!c->sel_flag) {
    ck(cudaHostAlloc(reinterpret_cast<void**>(&c->sel_flag), 64, cudaHostAllocMapped | cudaHostAllocPortable),
       "cudaHostAlloc");
    ck(cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->sel_flag_dev), c->sel_flag, 0),
       "cudaHostGetDevicePointer");
  }
  *reinterpret_cast<volatile int*>(c->sel_flag) = -1;
  return c->sel_flag_dev;
}

int select_wait_b(lrgw_ctx c, const int* b_dev) {
  volatile int* f = c->sel_flag;
  for (unsigned it = 1;; ++it) {
    const int v = *f;
    if (v >= 0) return v;
    if ((it & 1023u) == 0) {
      const cudaError_t q = cudaStreamQuery(c->stream);
      if (q == cudaErrorNotReady) continue;
      if (q != cudaSuccess) ck(q, "select greedy");
      // the stream drained without the slot changing: read b the slow way
      if (*f >= 0) return *f;
      int nb = 0;
      download(c, &nb, b_dev, sizeof(int));
      return nb;
    }
  }
}

cudaEvent_t select_event(lrgw_ctx c, int j) {
  constexpr int R = sizeof(c->sel_ev) / sizeof(c->sel_ev[0]);
  cudaEvent_t& e = c->sel_ev[j % R];
  if (!e) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
  return e;
}

std::vector<int32_t> select_impl(lrgw_ctx c, const double* a, long long lda, int n1, const double* b,
                                 long long ldb, int n2, int n_r, int n_mu, double* min_margin,
                                 SelectKeep* keep) {
  if (n_mu > n_r) fail(LRGW_ERR_INVALID_INPUT, "select_interpolation_points: N_mu > N_r");
  if (n_mu < 1) fail(LRGW_ERR_INVALID_INPUT, "select_interpolation_points: N_mu < 1");
  if (n1 < 1 || n2 < 1) fail(LRGW_ERR_INVALID_INPUT, "select_interpolation_points: empty orbital set");
  if (select_ent_bytes() != sizeof(HostEnt)) fail(LRGW_ERR_INTERNAL, "select: entry layout mismatch");
  const long long m = (long long)n1 * n2;
  const int kmax = (int)std::min<long long>(m, n_r);
  const int steps = std::min(n_mu, kmax);
  const int s = std::max(1, std::min({c->select_batch, select_max_candidates(), n_r}));
  const int lds = s + (s & 1);  // even leading dims: 16-byte operand loads

  DBuf d = dalloc(c, n_r), pos = ialloc(c, n_r), perm = ialloc(c, n_r);
  // (lrgw_build sizes L like the half spectrum that later takes its block from
  // the cache: one Theta-sized block cycles L -> spectrum -> L across builds)
  DBuf L = dalloc(c, std::max((size_t)n_r * std::max(steps, 1), keep ? keep->min_l_elems : 0));
  DBuf wsel;  // W columns of the accepted pivots (only the three-launch fallback materialises them)
  DBuf xperm;  // X with permuted column groups for the TMA panel (panel4.cu)
  DBuf amu = dalloc(c, (size_t)lds * n1), bmu = dalloc(c, (size_t)lds * n2);
  DBuf lrow = dalloc(c, (size_t)lds * std::max(steps, 1));       // L rows of candidates / pivots
  DBuf wcc = dalloc(c, (size_t)s * s), xcol = dalloc(c, (size_t)s * s);
  DBuf bout_d = ialloc(c, 4);
  int* bout = bout_d.i();
  DBuf top(c, (size_t)(s + 1) * sizeof(HostEnt));
  DBuf tmp(c, select_topk_tmp_bytes(n_r, s + 1));
  DBuf cand = ialloc(c, s);
  DBuf order = ialloc(c, std::max(steps, 1)), margin = dalloc(c, std::max(steps, 1));
  Work w = make_work(c, (size_t)8 * s * s);

  ck(select_init(c->stream, a, lda, n1, b, ldb, n2, n_r, d.d(), pos.i(), perm.i()), "select_init");
  ck(select_topk_reset(c->stream, tmp.p), "select_topk_reset");
  int k = 0;
  // Device-driven block loop (the fused-panel path, where the per-block host
  // round trip is a visible share of the stage): every kernel of block j reads
  // the pivots-so-far k from kb2[j & 1] and the accepted count from bout[0];
  // the greedy writes k + nb to kb2[(j + 1) & 1]. The host never waits on the
  // block it just enqueued: it reads k back (pinned, two blocks behind) only
  // to decide when to stop; blocks enqueued past the end find k >= steps and
  // do nothing.
  const int cap = select_accept_cap(s, n_r);
  const bool dev_loop = select_device_loop_enabled() && fused_downdate_enabled() && select_panel_enabled(n1, n2) &&
                        (long long)n_r >= (long long)steps + s + 1 && n_r % 2 == 0 && lda % 2 == 0 &&
                        ldb % 2 == 0 && (reinterpret_cast<uintptr_t>(a) & 15) == 0 &&
                        (reinterpret_cast<uintptr_t>(b) & 15) == 0 && cap > 16 && s % 2 == 0;
  if (dev_loop) {
    DBuf kb2 = ialloc(c, 2), wpart = dalloc(c, select_wcc_work_elems());
    ck(cudaMemsetAsync(kb2.p, 0, 2 * sizeof(int), c->stream), "memset");
    int* hk = select_pinned(c, (size_t)steps + 8);
    int j = 0, known = 0;
    while (known < steps) {
      int* kin = kb2.i() + (j & 1);
      int* kout = kb2.i() + ((j + 1) & 1);
      ck(select_topk(c->stream, d.d(), pos.i(), n_r, 0, s + 1, tmp.p, top.p, kin), "select_topk");
      ck(select_cand_rows(c->stream, top.p, s, cand.i()), "cand_rows");
      ck(gather_rows3(c->stream, a, lda, n1, b, ldb, n2, L.d(), n_r, 0, cand.i(), s, amu.d(), bmu.d(), lrow.d(), lds,
                      kin),
         "gather");
      ck(hadamard_gemm(c->stream, s, s, amu.d(), lds, amu.d(), lds, n1, bmu.d(), lds, bmu.d(), lds, n2, wcc.d(), s,
                       1.0, 0.0),
         "hadamard_gemm(W_CC)");
      ck(select_wcc_lsub(c->stream, lrow.d(), lds, s, kin, wcc.d(), wpart.d()), "wcc_lsub");
      ck(select_cand_greedy(c->stream, n_r, s, steps, 0, top.p, wcc.d(), pos.i(), perm.i(), xcol.d(), order.i(),
                            min_margin ? margin.d() : nullptr, bout, cap, select_accept_round(), kin, kout),
         "cand_greedy");
      ck(gather_rows3(c->stream, a, lda, n1, b, ldb, n2, L.d(), n_r, 0, order.i(), 0, amu.d(), bmu.d(), lrow.d(), lds,
                      kin, bout, kin),
         "gather");
      ck(select_panel(c->stream, n_r, cap, a, lda, amu.d(), lds, n1, b, ldb, bmu.d(), lds, n2, L.d(), n_r, lrow.d(),
                      lds, 0, xcol.d(), s, L.d(), n_r, d.d(), pos.i(), 0, kin, bout),
         "select_panel");
      ck(cudaMemcpyAsync(hk + j, kout, sizeof(int), cudaMemcpyDeviceToHost, c->stream), "D2H");
      ck(cudaEventRecord(select_event(c, j), c->stream), "cudaEventRecord");
      ++j;
      if (j >= 2) {
        ck(cudaEventSynchronize(select_event(c, j - 2)), "cudaEventSynchronize");
        const int prev = j >= 3 ? hk[j - 3] : 0;
        known = hk[j - 2];
        if (known <= prev && known < steps) fail(LRGW_ERR_INTERNAL, "select: no progress (non-finite residuals?)");
      }
      if (j > steps + 4) fail(LRGW_ERR_INTERNAL, "select: block loop did not terminate");
    }
    ck(cudaStreamSynchronize(c->stream), "sync");
    int prev = 0;
    for (int q = 0; q < j; ++q) {
      if (hk[q] > prev) {
        if (select_trace()) fprintf(stderr, "select block k=%d se=%d b=%d (device loop)\n", prev, s, hk[q] - prev);
        if (keep) ++keep->blocks;
        prev = hk[q];
      }
    }
    k = steps;
  }
  while (k < steps) {
    const int se = std::min(s, n_r - k);
    // Candidate set C (top s by residual, position) and its Schur block
    //   W[C, C] = (A_C A_C^T) o (B_C B_C^T) - L[C, :k] L[C, :k]^T
    // (s x s: only the candidates' rows ever enter the greedy).
    ck(select_topk(c->stream, d.d(), pos.i(), n_r, k, se + 1, tmp.p, top.p), "select_topk");
    ck(select_cand_rows(c->stream, top.p, se, cand.i()), "cand_rows");
    ck(gather_rows3(c->stream, a, lda, n1, b, ldb, n2, L.d(), n_r, k, cand.i(), se, amu.d(), bmu.d(), lrow.d(), lds),
       "gather");
    ck(hadamard_gemm(c->stream, se, se, amu.d(), lds, amu.d(), lds, n1, bmu.d(), lds, bmu.d(), lds, n2, wcc.d(), se,
                     1.0, 0.0),
       "hadamard_gemm(W_CC)");
    if (k > 0)
      gemm(c, se, se, k, lrow.d(), lds, Lay::MN, lrow.d(), lds, Lay::MN, wcc.d(), se, -1.0, 1.0, nullptr, false, &w);
    const bool use_panel = fused_downdate_enabled() && select_panel_enabled(n1, n2);
    const bool use_p4 = use_panel && select_panel_tma_enabled();
    if (use_p4 && !xperm.p) xperm = dalloc(c, (size_t)s * s);
    ck(select_cand_greedy(c->stream, n_r, se, steps, k, top.p, wcc.d(), pos.i(), perm.i(), xcol.d(), order.i(),
                          min_margin ? margin.d() : nullptr, bout, select_accept_cap(se, n_r, use_p4),
                          select_accept_round(), nullptr, nullptr, use_p4 ? xperm.d() : nullptr,
                          select_flag_arm(c)),
       "cand_greedy");
    const int nb = select_wait_b(c, bout);  // the one host wait per block
    if (nb <= 0) fail(LRGW_ERR_INTERNAL, "select: no progress (non-finite residuals?)");
    if (select_trace()) fprintf(stderr, "select block k=%d se=%d b=%d\n", k, se, nb);
    // Full-length W columns of the nb accepted pivots only (grid rows
    // order[k .. k+nb)), then L[:, k:k+nb] = W_sel X^T with X = L_sel^-1.
    const int* srow = order.i() + k;
    const int ldb_ = nb + (nb & 1);
    ck(gather_rows3(c->stream, a, lda, n1, b, ldb, n2, L.d(), n_r, k, srow, nb, amu.d(), bmu.d(), lrow.d(), ldb_),
       "gather");
    // one launch (panel4.cu on the TMA engine, else panel.cu): W_sel,
    // L[:, k:k+nb] = W_sel X^T and the downdate
    cudaError_t pe = cudaErrorNotSupported;
    if (use_p4)
      pe = select_panel_tma(c->stream, n_r, nb, a, lda, amu.d(), ldb_, n1, b, ldb, bmu.d(), ldb_, n2, L.d(), n_r,
                            lrow.d(), ldb_, k, xperm.d(), se, L.d() + (size_t)k * n_r, n_r, d.d(), pos.i(), k + nb);
    if (pe == cudaErrorNotSupported && use_panel) {
      cudaGetLastError();
      pe = select_panel(c->stream, n_r, nb, a, lda, amu.d(), ldb_, n1, b, ldb, bmu.d(), ldb_, n2, L.d(), n_r,
                        lrow.d(), ldb_, k, xcol.d(), se, L.d() + (size_t)k * n_r, n_r, d.d(), pos.i(), k + nb);
    }
    if (pe != cudaErrorNotSupported) {
      ck(pe, "select_panel");
      k += nb;
      if (keep) ++keep->blocks;
      continue;
    }
    cudaGetLastError();
    if (!wsel.p) wsel = dalloc(c, (size_t)n_r * s);
    ck(hadamard_gemm(c->stream, n_r, nb, a, lda, amu.d(), ldb_, n1, b, ldb, bmu.d(), ldb_, n2, wsel.d(), n_r, 1.0,
                     0.0),
       "hadamard_gemm");
    if (k > 0) gemm(c, n_r, nb, k, L.d(), n_r, Lay::MN, lrow.d(), ldb_, Lay::MN, wsel.d(), n_r, -1.0, 1.0);
    // L[:, k:k+nb] = W_sel X^T with d -= rowsum(L_blk^2) fused in the epilogue (rows not yet taken)
    cudaError_t fe = fused_downdate_enabled()
                         ? dgemm_tall_downdate(c->stream, n_r, nb, nb, wsel.d(), n_r, xcol.d(), se,
                                               L.d() + (size_t)k * n_r, n_r, d.d(), pos.i(), k + nb)
                         : cudaErrorNotSupported;
    if (fe == cudaErrorNotSupported) {
      cudaGetLastError();
      gemm(c, n_r, nb, nb, wsel.d(), n_r, Lay::MN, xcol.d(), se, Lay::MN, L.d() + (size_t)k * n_r, n_r, 1.0, 0.0);
      ck(select_downdate(c->stream, L.d(), n_r, k, nb, pos.i(), d.d()), "downdate");
    } else {
      ck(fe, "dgemm_tall_downdate");
    }
    k += nb;
    if (keep) ++keep->blocks;
  }
  // one read-back (pinned) of the points, the pivot order and the margins
  const size_t n_ord = keep ? (size_t)steps : 0, n_mg = min_margin ? (size_t)std::max(steps, 1) : 0;
  const size_t o_ord = (size_t)n_mu, o_mg = (o_ord + n_ord + 1) / 2 * 2;  // margins 8-byte aligned
  int* hp = select_pinned(c, o_mg + 2 * n_mg + 2);
  ck(cudaMemcpyAsync(hp, perm.p, sizeof(int) * n_mu, cudaMemcpyDeviceToHost, c->stream), "D2H");
  if (n_ord) ck(cudaMemcpyAsync(hp + o_ord, order.p, sizeof(int) * n_ord, cudaMemcpyDeviceToHost, c->stream), "D2H");
  if (n_mg) ck(cudaMemcpyAsync(hp + o_mg, margin.p, sizeof(double) * n_mg, cudaMemcpyDeviceToHost, c->stream), "D2H");
  ck(cudaStreamSynchronize(c->stream), "sync");
  std::vector<int32_t> pts(hp, hp + n_mu);
  std::sort(pts.begin(), pts.end());
  if (keep) {
    keep->steps = steps;
    keep->order.assign(hp + o_ord, hp + o_ord + n_ord);
    keep->L = std::move(L);
  }
  if (min_margin) {
    const double* hm = reinterpret_cast<const double*>(hp + o_mg);
    std::vector<double> mg(hm, hm + n_mg);
    double mn = 1.0;
    int at = -1;
    for (int i = 0; i < steps; ++i)
      if (mg[i] < mn) {
        mn = mg[i];
        at = i;
      }
    *min_margin = mn;
    if (keep) keep->min_margin_step = at;
  }
  return pts;
}

// The reference's seeded stream (rng.hpp:13-48: PCG32 oneseq, Box-Muller with
// the cached second variate) for the sketch of qrcp_sketched.
struct Pcg32 {
  uint64_t s = 0;
  bool have = false;
  double spare = 0.0;
  explicit Pcg32(uint64_t seed) {
    next();
    s += 0x853c49e6748fea9bULL ^ seed;
    next();
  }
  uint32_t next() {
    const uint64_t old = s;
    s = old * 6364136223846793005ULL + 1442695040888963407ULL;
    const uint32_t x = static_cast<uint32_t>(((old >> 18u) ^ old) >> 27u);
    const uint32_t rot = static_cast<uint32_t>(old >> 59u);
    return (x >> rot) | (x << ((32u - rot) & 31u));
  }
  double uniform() { return (static_cast<double>(next()) + 1.0) / 4294967296.0; }
  double gaussian() {
    if (have) {
      have = false;
      return spare;
    }
    const double u1 = uniform(), u2 = uniform();
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double a = 6.283185307179586476925286766559 * u2;
    spare = r * std::sin(a);
    have = true;
    return r * std::cos(a);
  }
};

// PointSelector::qrcp_sketched (isdf.hpp:95-112): the pair rows compressed by
// the reference's fixed Gaussian sketch G (2 N_mu x N1 N2, Rng(0x15df)) when
// 2 N_mu < N1 N2, then greedy QRCP on the sketch's columns. The sketch is
// formed on the device as F = M G^T (M the N_r x N1 N2 pair matrix, one DMMA
// GEMM; the reference's guard on materialising M applies), and the QRCP
// pivots of Z_s = F^T are the greedy pivoted-Cholesky pivots of F F^T —
// select_impl with a = F and b = 1 ((F F^T) o (1 1^T) = F F^T).
std::vector<int32_t> select_sketched(lrgw_ctx c, const double* a, long long lda, int n1, const double* b,
                                     long long ldb, int n2, int n_r, int n_mu) {
  const long long m = (long long)n1 * n2;
  if ((long long)n_r * m > (1LL << 26))
    fail(LRGW_ERR_GUARD_EXCEEDED, "pair_matrix_transposed: materialization guard exceeded");
  if (2LL * n_mu >= m) return select_impl(c, a, lda, n1, b, ldb, n2, n_r, n_mu, nullptr);
  const int ns = 2 * n_mu;
  std::vector<double> g((size_t)ns * m);
  Pcg32 rng(0x15dfu);
  for (double& x : g) x = rng.gaussian();  // Matrix::gaussian: column-major fill (matrix.hpp:29-33)
  DBuf dg = upload(c, g.data(), g.size());
  DBuf pm = dalloc(c, (size_t)n_r * m);
  ck(pair_matrix(c->stream, a, lda, n1, b, ldb, n2, n_r, pm.d(), n_r), "pair_matrix");
  DBuf f = dalloc(c, (size_t)n_r * ns), ones = dalloc(c, (size_t)n_r);
  Work w = make_work(c, (size_t)4 * n_r * ns);
  gemm(c, n_r, ns, (int)m, pm.d(), n_r, Lay::MN, dg.d(), ns, Lay::MN, f.d(), n_r, 1.0, 0.0, nullptr, false, &w);
  ck(fill(c->stream, ones.d(), (size_t)n_r, 1.0), "fill");
  return select_impl(c, f.d(), n_r, ns, ones.d(), n_r, 1, n_r, n_mu, nullptr);
}

// ---------------------------------------------------------------------------
// Stage 2: Theta = lhs G^-1 with lhs = (A A_mu^T) o (B B_mu^T) (isdf.hpp:118-163).
// ---------------------------------------------------------------------------
void check_points(const int32_t* pts, int n_mu, int n_r) {
  if (n_mu < 1) fail(LRGW_ERR_INVALID_INPUT, "fit_auxiliary_basis: empty point set");
  for (int i = 0; i < n_mu; ++i) {
    if (pts[i] < 0 || pts[i] >= n_r) fail(LRGW_ERR_INVALID_INPUT, "rows_at: index out of range");
    if (i > 0 && pts[i] <= pts[i - 1])
      fail(LRGW_ERR_INVALID_INPUT, "fit_auxiliary_basis: points must be distinct and sorted");
  }
}

void fit_impl(lrgw_ctx c, const double* a, long long lda, int n1, const double* b, long long ldb, int n2,
              int n_r, const int32_t* pts, int n_mu, double* theta, long long ldt) {
  check_points(pts, n_mu, n_r);
  DBuf dp = upload_i(c, pts, n_mu);
  DBuf amu = dalloc(c, (size_t)n_mu * n1), bmu = dalloc(c, (size_t)n_mu * n2);
  ck(gather_rows(c->stream, a, lda, n1, dp.i(), n_mu, amu.d(), n_mu), "gather");
  ck(gather_rows(c->stream, b, ldb, n2, dp.i(), n_mu, bmu.d(), n_mu), "gather");
  DBuf lhs = dalloc(c, (size_t)n_r * n_mu);
  ck(hadamard_gemm(c->stream, n_r, n_mu, a, lda, amu.d(), n_mu, n1, b, ldb, bmu.d(), n_mu, n2, lhs.d(), n_r, 1.0,
                   0.0),
     "hadamard_gemm");
  DBuf gram = dalloc(c, (size_t)n_mu * n_mu);
  ck(gather_rows(c->stream, lhs.d(), n_r, n_mu, dp.i(), n_mu, gram.d(), n_mu), "gather");
  ck(mirror_lower(c->stream, gram.d(), n_mu, n_mu, true), "symmetrize");
  DBuf ginv = dalloc(c, (size_t)n_mu * n_mu);
  mark(c, 2);
  gram_inverse(c, gram.d(), n_mu, ginv.d());
  mark(c, 3);
  gemm(c, n_r, n_mu, n_mu, lhs.d(), n_r, Lay::MN, ginv.d(), n_mu, Lay::MN, theta, ldt, 1.0, 0.0);
}

// Fused fit from the selection's Cholesky factor: with the greedy pivots
// p_0..p_{N_mu-1}, G(:, P) = L L_P^T and G(P, P) = L_P L_P^T where
// L_P = L[P, :] is lower triangular, so
//   Theta = (Z C^T)(C C^T)^-1 = G(:, P) G(P, P)^-1 = L L_P^-1
// (isdf.hpp:130-143 in exact arithmetic). One triangular inverse of L_P
// (cuSOLVER trtri, leaf) and one DMMA GEMM that skips the zero upper triangle
// of L_P^-1 and scatters the pivot-ordered columns into sorted-point order.
// Returns false (caller falls back to the explicit path) when L_P has a pivot
// below the LU singularity threshold of linalg.hpp:128, 137.
// Theta = L L_P^-1 from the selection's factor, enqueued without a host wait:
// the singularity rule of the LU the reference solves (1e-14 max G(p, p) on
// L_ii^2, linalg.hpp:128) and trtri's zero-pivot flag land in ff and are
// checked when the SMW status is read (smw_finish); a failed check rebuilds
// Theta on the explicit path there. false: not applicable (steps != N_mu).
bool fused_fit(lrgw_ctx c, const SelectKeep& keep, int n_r, const std::vector<int32_t>& pts_sorted, int n_mu,
               double* theta, long long ldt, FusedFit& ff) {
  if (keep.steps != n_mu) return false;
  const std::vector<int>& order = keep.order;
  // output column of pivot-ordered column q: its rank among the sorted points
  std::vector<int> colmap(n_mu);
  for (int q = 0; q < n_mu; ++q)
    colmap[q] = (int)(std::lower_bound(pts_sorted.begin(), pts_sorted.end(), order[q]) - pts_sorted.begin());
  DBuf dorder = upload_i(c, order.data(), n_mu);
  DBuf dmap = upload_i(c, colmap.data(), n_mu);
  ff.diag = dalloc(c, 4);
  ff.bad = ialloc(c, 1);
  DBuf lp = dalloc(c, (size_t)n_mu * n_mu);
  ck(gather_rows(c->stream, keep.L.d(), n_r, n_mu, dorder.i(), n_mu, lp.d(), n_mu), "gather");
  // zero the (numerically tiny) strict upper triangle and check the diagonal
  ck(zero_strict_upper(c->stream, lp.d(), n_mu, n_mu), "zero_upper");
  ck(diag_stats(c->stream, lp.d(), n_mu, n_mu, ff.diag.d()), "diag_stats");
  // X = L_P^-1 in place (trtri.cu: recursive 2 x 2 blocking on the DMMA engine)
  {
    DBuf work = dalloc(c, trtri_work_elems(n_mu));
    ck(cudaMemsetAsync(ff.bad.p, 0x7f, sizeof(int), c->stream), "memset");  // 0x7f7f7f7f: no zero pivot
    ck(lrgw_dev::trtri_lower(c->stream, lp.d(), n_mu, n_mu, work.d(), ff.bad.i(), c->sm_count), "trtri");
  }
  mark(c, 3);  // FIT_SOLVE = gather L_P + trtri; FIT_GEMM = L L_P^-1 below
  // B(n, k) = X(k, n) stored n-contiguous (X^T): both operands MN-contiguous
  // for the paired-fragment engine
  DBuf xt = dalloc(c, (size_t)n_mu * n_mu);
  ck(transpose(c->stream, lp.d(), n_mu, n_mu, n_mu, xt.d(), n_mu), "transpose");
  ck(dgemm(c->stream, n_r, n_mu, n_mu, keep.L.d(), n_r, Lay::MN, xt.d(), n_mu, Lay::MN, theta, ldt, 1.0, 0.0,
           nullptr, false, c->sm_count, nullptr, 0, true, dmap.i()),
     "dgemm(theta)");
  return true;
}

// ---------------------------------------------------------------------------
// Stage 3: quadrature (K3, quadrature.cu).
// ---------------------------------------------------------------------------

NodeSet trapezoid(const lrgw_host::Spec& s, int n_intervals) {
  NodeSet ns;
  const double h = 2.0 * s.big_r / n_intervals;
  for (int k = 0; k <= n_intervals; ++k) {
    ns.nodes.push_back(-s.big_r + k * h);
    ns.weights.push_back((k == 0 || k == n_intervals) ? 0.5 * h : h);
  }
  return ns;
}

// out (n_mu^2, mirrored) = pref * (beta * running + sum_k w_k term_k); running updated if given.
void quad_run(lrgw_ctx c, const double* pv, long long ldv, const double* pc, long long ldpc, int n_mu, int n_v,
              int n_c, const std::vector<double>& dv, const std::vector<double>& dc, const std::vector<double>& gw,
              int n_nodes, double* running, double beta, double pref, double* out, long long ldo) {
  if (n_nodes <= 0) {
    ck(fill(c->stream, out, (size_t)n_mu * n_mu, 0.0), "fill");
    return;
  }
  DBuf ddv = upload(c, dv.data(), dv.size()), ddc = upload(c, dc.data(), dc.size());
  DBuf dgw = upload(c, gw.data(), gw.size());
  DBuf partial = dalloc(c, quad_partial_elems(n_mu, n_nodes, c->sm_count));
  ck(quad_nodes(c->stream, n_mu, n_v, n_c, pv, ldv, pc, ldpc, n_nodes, ddv.d(), ddc.d(), dgw.d(), c->sm_count,
                partial.d(), running, beta, pref, out, ldo, c->timing ? c->ev_quad[0] : nullptr,
                c->timing ? c->ev_quad[1] : nullptr),
     "quad_nodes");
  if (c->timing) c->quad_timed = true;
}

void node_tables_or_fail(const lrgw_host::Spec& s, const double* e, int n_v, int n_c, const NodeSet& ns,
                         std::vector<double>* dv, std::vector<double>* dc, std::vector<double>* gw) {
  const int st = lrgw_host::node_tables(s, e, n_v, n_c, ns.nodes.data(), ns.weights.data(),
                                        (int)ns.nodes.size(), dv, dc, gw);
  if (st == lrgw_host::kNumeric) fail(LRGW_ERR_NUMERIC, "jacobi_complex: argument too close to a pole");
  if (st != lrgw_host::kOk) fail(st, "contour node geometry");
}

void check_coupled(int n_mu, int n_v, int n_c, int n_e) {
  if (n_mu < 1 || n_v < 1 || n_c < 1) fail(LRGW_ERR_INVALID_INPUT, "coupled_coefficients: empty input");
  if (n_v + n_c > n_e) fail(LRGW_ERR_INVALID_INPUT, "coupled_coefficients: not enough energies");
}

// T = sum_i (v_i v_i^T) o (Pc diag(1/(e_i - e_c)) Pc^T), symmetrised
// (contour.hpp:114-137) through the K3 kernel with one-hot valence diagonals.
void direct_impl(lrgw_ctx c, const double* pv, long long ldv, const double* pc, long long ldpc, int n_mu, int n_v,
                 int n_c, const double* e, double* t, long long ldt) {
  std::vector<double> dv((size_t)2 * n_v * n_v, 0.0), dc((size_t)2 * n_v * n_c, 0.0), gw((size_t)2 * n_v, 0.0);
  for (int i = 0; i < n_v; ++i) {
    dv[2 * ((size_t)i * n_v + i)] = 1.0;
    for (int j = 0; j < n_c; ++j) dc[2 * ((size_t)i * n_c + j)] = 1.0 / (e[i] - e[n_v + j]);
    gw[2 * i + 1] = 1.0;  // term = g_im * Re(Jv o Jc) with real J's
  }
  quad_run(c, pv, ldv, pc, ldpc, n_mu, n_v, n_c, dv, dc, gw, n_v, nullptr, 0.0, 1.0, t, ldt);
}

void fixed_impl(lrgw_ctx c, const double* pv, long long ldv, const double* pc, long long ldpc, int n_mu, int n_v,
                int n_c, const double* e, int n_e, int n_lambda, double* t, long long ldt) {
  if (n_lambda < 1) fail(LRGW_ERR_INVALID_INPUT, "contour quadrature: N_lambda < 1");
  lrgw_host::Spec s;
  host_status(lrgw_host::elliptic_params(e, n_e, n_v, n_c, 1e-7, 1025, &s), "elliptic_params");
  if (s.bypass) {  // single energy denominator: the mandated direct sum (driver.hpp:239-240)
    direct_impl(c, pv, ldv, pc, ldpc, n_mu, n_v, n_c, e, t, ldt);
    return;
  }
  NodeSet ns = trapezoid(s, n_lambda);
  std::vector<double> dv, dc, gw;
  node_tables_or_fail(s, e, n_v, n_c, ns, &dv, &dc, &gw);
  quad_run(c, pv, ldv, pc, ldpc, n_mu, n_v, n_c, dv, dc, gw, (int)ns.nodes.size(), nullptr, 0.0,
           lrgw_host::prefactor(s), t, ldt);
}

// Nested 2^m+1 levels (contour.hpp:235-279); visit(n_nodes, T_dev) -> continue?
template <class Visit>
void levels_impl(lrgw_ctx c, const double* pv, long long ldv, const double* pc, long long ldpc, int n_mu, int n_v,
                 int n_c, const double* e, const lrgw_host::Spec& s, int max_level_nodes, Visit&& visit) {
  if (s.bypass) fail(LRGW_ERR_INVALID_INPUT, "contour quadrature: spec is bypass-flagged; use the direct sum");
  if ((1 << 4) + 1 > max_level_nodes) fail(LRGW_ERR_INVALID_INPUT, "contour quadrature: node cap below one level");
  const double pref = lrgw_host::prefactor(s);
  DBuf running = dalloc(c, (size_t)n_mu * n_mu);
  DBuf tl = dalloc(c, (size_t)n_mu * n_mu);
  bool first = true;
  for (int m = 4;; ++m) {
    const int n_nodes = (1 << m) + 1;
    if (n_nodes > max_level_nodes) break;
    const double h = 2.0 * s.big_r / (n_nodes - 1);
    NodeSet ns;
    if (first) {
      for (int k = 0; k < n_nodes; ++k) {
        ns.nodes.push_back(-s.big_r + k * h);
        ns.weights.push_back((k == 0 || k == n_nodes - 1) ? 0.5 * h : h);
      }
    } else {
      for (int k = 1; k < n_nodes; k += 2) {
        ns.nodes.push_back(-s.big_r + k * h);
        ns.weights.push_back(h);
      }
    }
    std::vector<double> dv, dc, gw;
    node_tables_or_fail(s, e, n_v, n_c, ns, &dv, &dc, &gw);
    quad_run(c, pv, ldv, pc, ldpc, n_mu, n_v, n_c, dv, dc, gw, (int)ns.nodes.size(), running.d(),
             first ? 0.0 : 0.5, pref, tl.d(), n_mu);
    first = false;
    if (!visit(n_nodes, tl.d())) break;
  }
}


void adaptive_impl(lrgw_ctx c, const double* pv, long long ldv, const double* pc, long long ldpc, int n_mu, int n_v,
                   int n_c, const double* energies, const lrgw_host::Spec& spec, double* t) {
  const size_t nn = (size_t)n_mu * n_mu;
  DBuf prev = dalloc(c, nn), red = dalloc(c, 512);
  bool have = false, conv = false;
  levels_impl(c, pv, ldv, pc, ldpc, n_mu, n_v, n_c, energies, spec, spec.max_nodes, [&](int, double* tl) {
    ck(cudaMemcpyAsync(t, tl, nn * sizeof(double), cudaMemcpyDeviceToDevice, c->stream), "D2D");
    if (!have) {
      have = true;
      ck(cudaMemcpyAsync(prev.p, tl, nn * sizeof(double), cudaMemcpyDeviceToDevice, c->stream), "D2D");
      return true;
    }
    double h[2];
    ck(frob_diff(c->stream, tl, prev.d(), nn, red.d()), "frob");
    ck(cudaMemcpyAsync(&h[0], red.d() + 296, sizeof(double), cudaMemcpyDeviceToHost, c->stream), "D2H");
    ck(frob_diff(c->stream, tl, nullptr, nn, red.d()), "frob");
    download(c, &h[1], red.d() + 296, sizeof(double));
    ck(cudaMemcpyAsync(prev.p, tl, nn * sizeof(double), cudaMemcpyDeviceToDevice, c->stream), "D2D");
    if (std::sqrt(h[0]) / std::max(std::sqrt(h[1]), 1e-300) <= spec.delta_rel) {
      conv = true;
      return false;
    }
    return true;
  });
  if (!conv) fail(LRGW_ERR_CONTOUR_CONVERGENCE, "coupled_coefficients_contour: did not reach delta_rel within max_nodes");
}

}  // namespace

// ===========================================================================
// C-ABI
// ===========================================================================
extern "C" {

int lrgw_abi_version(void) { return LRGW_ABI_VERSION; }

int lrgw_ctx_create(int device, lrgw_ctx* out) {
  if (!out) return LRGW_ERR_INVALID_INPUT;
  *out = nullptr;
  auto* c = new (std::nothrow) lrgw_ctx_s;
  if (!c) return LRGW_ERR_INTERNAL;
  c->device = device;
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete c;
    return LRGW_ERR_CUDA;
  }
  c->stream = c->own_stream;
  cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device);
  if (cusolverDnCreate(&c->solver) != CUSOLVER_STATUS_SUCCESS) {
    cudaStreamDestroy(c->own_stream);
    delete c;
    return LRGW_ERR_CUDA;
  }
  cusolverDnSetStream(c->solver, c->stream);
  // keep freed pool memory cached across calls (stream-ordered allocator)
  c->launches0 = launch_count();
  *out = c;
  return LRGW_OK;
}

int lrgw_ctx_destroy(lrgw_ctx c) {
  if (!c) return LRGW_OK;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  {
    std::lock_guard<std::mutex> lk(c->mem_mu);
    for (lrgw_eps_s* e : c->live_eps) {  // orphan the handles, free their buffers
      for (double* p : {e->theta, e->k, e->t, e->pvp, e->lp, e->lpinv}) {
        auto it = c->mem_live.find(p);
        if (it != c->mem_live.end()) {
          cudaFree(p);
          c->mem_live.erase(it);
        }
      }
      e->theta = e->k = e->t = e->pvp = e->lp = e->lpinv = nullptr;
      e->ctx = nullptr;
    }
    c->live_eps.clear();
    release_cached(c);
  }
  for (auto& kv : c->plans) cufftDestroy(kv.second);
  for (auto& kv : c->plans_many) cufftDestroy(kv.second);
  if (c->solver) cusolverDnDestroy(c->solver);
  if (c->sel_pinned) cudaFreeHost(c->sel_pinned);
  if (c->sel_flag) cudaFreeHost(c->sel_flag);
  for (auto e : c->sel_ev)
    if (e) cudaEventDestroy(e);
  if (c->side) {
    cudaStreamSynchronize(c->side);
    cudaStreamDestroy(c->side);
    cudaEventDestroy(c->ev_side);
    cudaEventDestroy(c->ev_join);
  }
  if (c->own_stream) cudaStreamDestroy(c->own_stream);
  for (auto& x : c->ev)
    if (x) cudaEventDestroy(x);
  for (auto& x : c->ev_quad)
    if (x) cudaEventDestroy(x);
  for (auto& x : c->ev_lib)
    if (x) cudaEventDestroy(x);
  delete c;
  return LRGW_OK;
}

int lrgw_ctx_set_stream(lrgw_ctx c, void* stream) {
  return guarded(c, [&] {
    ck(cudaStreamSynchronize(c->stream), "sync");
    c->stream = stream ? static_cast<cudaStream_t>(stream) : c->own_stream;
    cusolverDnSetStream(c->solver, c->stream);
    for (auto& kv : c->plans) cufftSetStream(kv.second, c->stream);
  });
}

void* lrgw_ctx_stream(lrgw_ctx c) { return c ? static_cast<void*>(c->stream) : nullptr; }

int lrgw_ctx_synchronize(lrgw_ctx c) {
  return guarded(c, [&] { ck(cudaStreamSynchronize(c->stream), "sync"); });
}

const char* lrgw_ctx_last_error(lrgw_ctx c) { return c ? c->err.c_str() : "null context"; }
int lrgw_ctx_last_pivot(lrgw_ctx c) { return c ? c->pivot : -1; }

int lrgw_ctx_stage_ms(lrgw_ctx c, double* ms, int n) {
  if (!c || !ms) return LRGW_ERR_INVALID_INPUT;
  for (int i = 0; i < n && i < LRGW_NUM_STAGES; ++i) ms[i] = c->stage_ms[i];
  return LRGW_OK;
}

long long lrgw_ctx_kernel_launches(lrgw_ctx c) { return c ? launch_count() - c->launches0 : 0; }

int lrgw_ctx_set_theta_implicit(lrgw_ctx c, int on) {
  if (!c) return LRGW_ERR_INVALID_INPUT;
  c->theta_implicit = on != 0;
  return LRGW_OK;
}

int lrgw_ctx_set_select_batch(lrgw_ctx c, int s) {
  if (!c || s < 1 || s > select_max_candidates()) return LRGW_ERR_INVALID_INPUT;
  c->select_batch = s;
  return LRGW_OK;
}

// ---- host scalars ---------------------------------------------------------
int lrgw_num_aux(double k_mu, int n1, int n2, int* out) {
  if (!(k_mu > 0.0) || !out) return LRGW_ERR_INVALID_INPUT;
  *out = static_cast<int>(std::llround(k_mu * std::sqrt(static_cast<double>(n1) * n2)));
  return LRGW_OK;
}

int lrgw_elliptic_k(double k, double* out) { return lrgw_host::elliptic_k(k, out); }

int lrgw_jacobi_sn_cn_dn(double u, double k, double* o) {
  return lrgw_host::jacobi_sn_cn_dn(u, k, o, o + 1, o + 2);
}

int lrgw_jacobi_complex(double x, double y, double k, double* o) {
  std::complex<double> sn, cn, dn;
  const int st = lrgw_host::jacobi_complex(x, y, k, &sn, &cn, &dn);
  if (st != lrgw_host::kOk) return st;
  o[0] = sn.real();
  o[1] = sn.imag();
  o[2] = cn.real();
  o[3] = cn.imag();
  o[4] = dn.real();
  o[5] = dn.imag();
  return LRGW_OK;
}

int lrgw_elliptic_params(const double* e, int n_e, int n_v, int n_c, double delta_rel, int max_nodes,
                         double* spec7) {
  lrgw_host::Spec s;
  const int st = lrgw_host::elliptic_params(e, n_e, n_v, n_c, delta_rel, max_nodes, &s);
  if (st == lrgw_host::kOk) spec_to7(s, spec7);
  return st;
}

int lrgw_cauchy_error_bound(const double* spec7, int n_lambda, double* out) {
  return lrgw_host::cauchy_error_bound(spec_from7(spec7), n_lambda, out);
}

int lrgw_coulomb_kernel(const int* dims, const double* cell, double* kernel) {
  return guarded_host([&] {
    check_grid(dims, cell);
    const double two_pi = 6.283185307179586476925286766559;
    const int n1 = dims[0], n2 = dims[1], n3 = dims[2];
    for (long long idx = 0; idx < (long long)n1 * n2 * n3; ++idx) {
      const int i1 = (int)(idx % n1), i2 = (int)((idx / n1) % n2), i3 = (int)(idx / ((long long)n1 * n2));
      const int f1 = i1 <= n1 / 2 ? i1 : i1 - n1, f2 = i2 <= n2 / 2 ? i2 : i2 - n2, f3 = i3 <= n3 / 2 ? i3 : i3 - n3;
      const double g1 = two_pi * f1 / cell[0], g2 = two_pi * f2 / cell[1], g3 = two_pi * f3 / cell[2];
      const double g = g1 * g1 + g2 * g2 + g3 * g3;
      kernel[idx] = g > 0.0 ? 12.566370614359172953850573533118 / g : 0.0;
    }
  });
}

// ---- host-buffer API --------------------------------------------------------
int lrgw_select_interpolation_points(lrgw_ctx c, const double* psi_a, const double* psi_b, int n_r, int n1,
                                     int n2, int n_mu, int method, int32_t* pts) {
  return guarded(c, [&] {
    if (method != LRGW_QRCP_DIRECT && method != LRGW_QRCP_SKETCHED)
      fail(LRGW_ERR_INVALID_INPUT, "select_interpolation_points: unknown point selector");
    if (n_mu > n_r) fail(LRGW_ERR_INVALID_INPUT, "select_interpolation_points: N_mu > N_r");
    if (n_mu < 1) fail(LRGW_ERR_INVALID_INPUT, "select_interpolation_points: N_mu < 1");
    DBuf a = upload(c, psi_a, (size_t)n_r * n1), b = upload(c, psi_b, (size_t)n_r * n2);
    std::vector<int32_t> p = method == LRGW_QRCP_SKETCHED
                                 ? select_sketched(c, a.d(), n_r, n1, b.d(), n_r, n2, n_r, n_mu)
                                 : select_impl(c, a.d(), n_r, n1, b.d(), n_r, n2, n_r, n_mu, nullptr);
    std::copy(p.begin(), p.end(), pts);
  });
}

int lrgw_fit_auxiliary_basis(lrgw_ctx c, const double* psi_a, const double* psi_b, int n_r, int n1, int n2,
                             const int32_t* pts, int n_mu, double* theta) {
  return guarded(c, [&] {
    check_points(pts, n_mu, n_r);
    DBuf a = upload(c, psi_a, (size_t)n_r * n1), b = upload(c, psi_b, (size_t)n_r * n2);
    DBuf th = dalloc(c, (size_t)n_r * n_mu);
    fit_impl(c, a.d(), n_r, n1, b.d(), n_r, n2, n_r, pts, n_mu, th.d(), n_r);
    download(c, theta, th.p, sizeof(double) * n_r * n_mu);
  });
}

int lrgw_coupled_coefficients_direct(lrgw_ctx c, const double* pv, const double* pc, int n_mu, int n_v, int n_c,
                                     const double* e, int n_e, double* t) {
  return guarded(c, [&] {
    check_coupled(n_mu, n_v, n_c, n_e);
    DBuf dv = upload(c, pv, (size_t)n_mu * n_v), dc = upload(c, pc, (size_t)n_mu * n_c);
    DBuf dt = dalloc(c, (size_t)n_mu * n_mu);
    direct_impl(c, dv.d(), n_mu, dc.d(), n_mu, n_mu, n_v, n_c, e, dt.d(), n_mu);
    download(c, t, dt.p, sizeof(double) * n_mu * n_mu);
  });
}

int lrgw_sum_node_terms(lrgw_ctx c, const double* pv, const double* pc, int n_mu, int n_v, int n_c, const double* e,
                        int n_e, const double* spec7, const double* nodes, const double* weights, int n_nodes,
                        double* acc) {
  return guarded(c, [&] {
    check_coupled(n_mu, n_v, n_c, n_e);
    lrgw_host::Spec s = spec_from7(spec7);
    NodeSet ns;
    ns.nodes.assign(nodes, nodes + n_nodes);
    ns.weights.assign(weights, weights + n_nodes);
    std::vector<double> dv, dc, gw;
    node_tables_or_fail(s, e, n_v, n_c, ns, &dv, &dc, &gw);
    DBuf dpv = upload(c, pv, (size_t)n_mu * n_v), dpc = upload(c, pc, (size_t)n_mu * n_c);
    DBuf dt = dalloc(c, (size_t)n_mu * n_mu);
    quad_run(c, dpv.d(), n_mu, dpc.d(), n_mu, n_mu, n_v, n_c, dv, dc, gw, n_nodes, nullptr, 0.0, 1.0, dt.d(), n_mu);
    download(c, acc, dt.p, sizeof(double) * n_mu * n_mu);
  });
}

int lrgw_coupled_coefficients_fixed(lrgw_ctx c, const double* pv, const double* pc, int n_mu, int n_v, int n_c,
                                    const double* e, int n_e, int n_lambda, double* t) {
  return guarded(c, [&] {
    check_coupled(n_mu, n_v, n_c, n_e);
    DBuf dpv = upload(c, pv, (size_t)n_mu * n_v), dpc = upload(c, pc, (size_t)n_mu * n_c);
    DBuf dt = dalloc(c, (size_t)n_mu * n_mu);
    fixed_impl(c, dpv.d(), n_mu, dpc.d(), n_mu, n_mu, n_v, n_c, e, n_e, n_lambda, dt.d(), n_mu);
    download(c, t, dt.p, sizeof(double) * n_mu * n_mu);
  });
}

int lrgw_coupled_coefficients_contour(lrgw_ctx c, const double* pv, const double* pc, int n_mu, int n_v, int n_c,
                                      const double* e, int n_e, double delta_rel, int max_nodes, double* t,
                                      int* nodes_used, double* est_rel) {
  return guarded(c, [&] {
    check_coupled(n_mu, n_v, n_c, n_e);
    lrgw_host::Spec s;
    host_status(lrgw_host::elliptic_params(e, n_e, n_v, n_c, delta_rel, max_nodes, &s), "elliptic_params");
    DBuf dpv = upload(c, pv, (size_t)n_mu * n_v), dpc = upload(c, pc, (size_t)n_mu * n_c);
    const size_t nn = (size_t)n_mu * n_mu;
    DBuf prev = dalloc(c, nn), best = dalloc(c, nn), red = dalloc(c, 512);
    bool have_prev = false, converged = false;
    int best_nodes = 0;
    double best_rel = 1.0;
    levels_impl(c, dpv.d(), n_mu, dpc.d(), n_mu, n_mu, n_v, n_c, e, s, s.max_nodes, [&](int n_nodes, double* tl) {
      ck(cudaMemcpyAsync(best.p, tl, nn * sizeof(double), cudaMemcpyDeviceToDevice, c->stream), "D2D");
      best_nodes = n_nodes;
      if (!have_prev) {
        best_rel = 1.0;
        have_prev = true;
        ck(cudaMemcpyAsync(prev.p, tl, nn * sizeof(double), cudaMemcpyDeviceToDevice, c->stream), "D2D");
        return true;
      }
      double h[2];
      ck(frob_diff(c->stream, tl, prev.d(), nn, red.d()), "frob");
      ck(cudaMemcpyAsync(&h[0], red.d() + 296, sizeof(double), cudaMemcpyDeviceToHost, c->stream), "D2H");
      ck(frob_diff(c->stream, tl, nullptr, nn, red.d()), "frob");
      download(c, &h[1], red.d() + 296, sizeof(double));
      const double scale = std::max(std::sqrt(h[1]), 1e-300);
      best_rel = std::sqrt(h[0]) / scale;
      ck(cudaMemcpyAsync(prev.p, tl, nn * sizeof(double), cudaMemcpyDeviceToDevice, c->stream), "D2D");
      if (best_rel <= s.delta_rel) {
        converged = true;
        return false;
      }
      return true;
    });
    download(c, t, best.p, nn * sizeof(double));
    if (nodes_used) *nodes_used = best_nodes;
    if (est_rel) *est_rel = best_rel;
    if (!converged)
      fail(LRGW_ERR_CONTOUR_CONVERGENCE, "coupled_coefficients_contour: did not reach delta_rel within max_nodes");
  });
}

int lrgw_contour_refinement_levels(lrgw_ctx c, const double* pv, const double* pc, int n_mu, int n_v, int n_c,
                                   const double* e, int n_e, int max_level_nodes, int max_levels, double* out,
                                   int* counts, int* n_levels) {
  return guarded(c, [&] {
    check_coupled(n_mu, n_v, n_c, n_e);
    lrgw_host::Spec s;
    host_status(lrgw_host::elliptic_params(e, n_e, n_v, n_c, 1e-7, 1025, &s), "elliptic_params");
    DBuf dpv = upload(c, pv, (size_t)n_mu * n_v), dpc = upload(c, pc, (size_t)n_mu * n_c);
    const size_t nn = (size_t)n_mu * n_mu;
    int n = 0;
    levels_impl(c, dpv.d(), n_mu, dpc.d(), n_mu, n_mu, n_v, n_c, e, s, max_level_nodes, [&](int nodes, double* tl) {
      if (n >= max_levels) return false;
      counts[n] = nodes;
      download(c, out + n * nn, tl, nn * sizeof(double));
      ++n;
      return true;
    });
    *n_levels = n;
  });
}

int lrgw_apply_coulomb(lrgw_ctx c, const int* dims, const double* cell, int zero, const double* x, int m, double* y) {
  return guarded(c, [&] {
    check_grid(dims, cell);
    const long long n_r = (long long)dims[0] * dims[1] * dims[2];
    DBuf dx = upload(c, x, (size_t)n_r * m), dy = dalloc(c, (size_t)n_r * m);
    coulomb_apply(c, dims, cell, zero, dx.d(), n_r, m, dy.d(), n_r);
    download(c, y, dy.p, sizeof(double) * n_r * m);
  });
}

int lrgw_assemble_K(lrgw_ctx c, const double* t, const double* p, int n_r, int n_mu, const int* dims,
                    const double* cell, int zero, double* k) {
  return guarded(c, [&] {
    check_grid(dims, cell);
    if ((long long)dims[0] * dims[1] * dims[2] != n_r || n_mu < 1)
      fail(LRGW_ERR_INVALID_INPUT, "assemble_K: T / P_vc shape mismatch");
    DBuf dt = upload(c, t, (size_t)n_mu * n_mu), dp = upload(c, p, (size_t)n_r * n_mu);
    DBuf pvp = dalloc(c, (size_t)n_mu * n_mu), dk = dalloc(c, (size_t)n_mu * n_mu);
    pvp_impl(c, dims, cell, zero, dp.d(), n_r, n_mu, pvp.d());
    smw_core(c, dt.d(), pvp.d(), n_mu, dk.d());
    download(c, k, dk.p, sizeof(double) * n_mu * n_mu);
  });
}

int lrgw_eps_from_parts(lrgw_ctx c, const double* p, const double* k, int n_r, int n_mu, const int* dims,
                        const double* cell, int zero, lrgw_eps* out) {
  return guarded(c, [&] {
    check_grid(dims, cell);
    if ((long long)dims[0] * dims[1] * dims[2] != n_r) fail(LRGW_ERR_INVALID_INPUT, "eps: grid / N_r mismatch");
    auto* e = new_eps(c);
    e->ctx = c;
    e->n_r = n_r;
    e->n_mu = n_mu;
    std::memcpy(e->dims, dims, sizeof(e->dims));
    std::memcpy(e->cell, cell, sizeof(e->cell));
    e->zero = zero;
    DBuf dp = upload(c, p, (size_t)n_r * n_mu), dk = upload(c, k, (size_t)n_mu * n_mu);
    e->theta = static_cast<double*>(dp.take());
    e->k = static_cast<double*>(dk.take());
    ck(cudaStreamSynchronize(c->stream), "sync");
    *out = e;
  });
}

int lrgw_build_epsilon_inverse(lrgw_ctx c, const double* t, const double* p, int n_r, int n_mu, const int* dims,
                               const double* cell, int zero, lrgw_eps* out) {
  return guarded(c, [&] {
    check_grid(dims, cell);
    if ((long long)dims[0] * dims[1] * dims[2] != n_r || n_mu < 1)
      fail(LRGW_ERR_INVALID_INPUT, "assemble_K: T / P_vc shape mismatch");
    DBuf dt = upload(c, t, (size_t)n_mu * n_mu), dp = upload(c, p, (size_t)n_r * n_mu);
    DBuf pvp = dalloc(c, (size_t)n_mu * n_mu), dk = dalloc(c, (size_t)n_mu * n_mu);
    pvp_impl(c, dims, cell, zero, dp.d(), n_r, n_mu, pvp.d());
    smw_core(c, dt.d(), pvp.d(), n_mu, dk.d());
    ck(cudaStreamSynchronize(c->stream), "sync");
    auto* e = new_eps(c);
    e->ctx = c;
    e->n_r = n_r;
    e->n_mu = n_mu;
    std::memcpy(e->dims, dims, sizeof(e->dims));
    std::memcpy(e->cell, cell, sizeof(e->cell));
    e->zero = zero;
    e->theta = static_cast<double*>(dp.take());
    e->k = static_cast<double*>(dk.take());
    e->t = static_cast<double*>(dt.take());
    *out = e;
  });
}

}  // extern "C"

bool lrgw_impl::eps_is_panel(const lrgw_eps_s* e) { return e->rows > 0 && e->rows < e->n_r; }

void lrgw_impl::eps_apply_impl(lrgw_ctx c, lrgw_eps e, const double* x, long long ldx, int m, double* y, long long ldy) {
  const int n_r = e->n_r, n_mu = e->n_mu;
  DBuf u = dalloc(c, (size_t)n_mu * m), w = dalloc(c, (size_t)n_mu * m), z = dalloc(c, (size_t)n_r * m);
  Work wk = make_work(c, (size_t)1200 * n_mu * m);
  // u = Theta^T x ; w = K u ; z = Theta w ; y = x + V z   (smw.hpp:101-102)
  if (skinny_supported(m)) {
    ck(skinny_tn(c->stream, e->theta, n_r, n_r, n_mu, x, ldx, m, u.d(), n_mu, wk.buf.d(), wk.elems, c->sm_count),
       "skinny_tn");
  } else {
    gemm(c, n_mu, m, n_r, e->theta, n_r, Lay::K, x, ldx, Lay::K, u.d(), n_mu, 1.0, 0.0, nullptr, false, &wk);
  }
  if (skinny_supported(m))  // w = K u = K^T u (K symmetric): the row-chunked stream
    ck(skinny_tn(c->stream, e->k, n_mu, n_mu, n_mu, u.d(), n_mu, m, w.d(), n_mu, wk.buf.d(), wk.elems, c->sm_count),
       "skinny_tn(K)");
  else
    gemm(c, n_mu, m, n_mu, e->k, n_mu, Lay::MN, u.d(), n_mu, Lay::K, w.d(), n_mu, 1.0, 0.0);
  if (skinny_supported(m) && (size_t)n_mu * m * 8 <= 200 * 1024) {
    ck(skinny_nn(c->stream, e->theta, n_r, n_r, n_mu, w.d(), n_mu, m, z.d(), n_r, c->sm_count), "skinny_nn");
  } else {
    gemm(c, n_r, m, n_mu, e->theta, n_r, Lay::MN, w.d(), n_mu, Lay::K, z.d(), n_r, 1.0, 0.0);
  }
  coulomb_apply(c, e->dims, e->cell, e->zero, z.d(), n_r, m, y, ldy);
  ck(axpby(c->stream, n_r, m, 1.0, x, ldx, 1.0, y, ldy), "axpby");
}

// Implicit handle -> ordinary handle: Theta = (L L_P^-1) scattered to the
// sorted-point columns (the fused fit's GEMM), K = Pi^T L_P K' L_P^T Pi,
// Theta^T V Theta = Pi^T L_P^-T P' L_P^-1 Pi, T = Pi^T T_pi Pi.
void lrgw_impl::eps_explicit(lrgw_ctx c, lrgw_eps_s* e) {
  if (!e->implicit) return;
  const int n_r = e->n_r, n_mu = e->n_mu;
  const size_t nn = (size_t)n_mu * n_mu;
  DBuf dmap = upload_i(c, e->colmap.data(), n_mu);
  std::vector<int> inv(n_mu);
  for (int q = 0; q < n_mu; ++q) inv[e->colmap[q]] = q;
  DBuf dinv = upload_i(c, inv.data(), n_mu);
  DBuf theta = dalloc(c, (size_t)n_r * n_mu);
  DBuf xt = dalloc(c, nn);
  ck(transpose(c->stream, e->lpinv, n_mu, n_mu, n_mu, xt.d(), n_mu), "transpose");
  ck(dgemm(c->stream, n_r, n_mu, n_mu, e->theta, n_r, Lay::MN, xt.d(), n_mu, Lay::MN, theta.d(), n_r, 1.0, 0.0,
           nullptr, false, c->sm_count, nullptr, 0, true, dmap.i()),
     "dgemm(theta)");
  Work w = make_work(c, 8 * nn);
  DBuf a = dalloc(c, nn), b = dalloc(c, nn);
  auto to_sorted = [&](const double* piv, double* out) {  // out = Pi^T piv Pi
    ck(gather_rows(c->stream, piv, n_mu, n_mu, dinv.i(), n_mu, b.d(), n_mu), "gather_rows");
    ck(gather_cols(c->stream, b.d(), n_mu, n_mu, dinv.i(), n_mu, out, n_mu), "gather_cols");
  };
  // K_pi = L_P K' L_P^T
  gemm(c, n_mu, n_mu, n_mu, e->lp, n_mu, Lay::MN, e->k, n_mu, Lay::K, a.d(), n_mu, 1.0, 0.0);
  DBuf kpi = dalloc(c, nn);
  gemm(c, n_mu, n_mu, n_mu, a.d(), n_mu, Lay::MN, e->lp, n_mu, Lay::MN, kpi.d(), n_mu, 1.0, 0.0, nullptr, true, &w);
  ck(mirror_lower(c->stream, kpi.d(), n_mu, n_mu, false), "mirror");
  to_sorted(kpi.d(), e->k);
  // pvp_pi = L_P^-T P' L_P^-1
  gemm(c, n_mu, n_mu, n_mu, e->lpinv, n_mu, Lay::K, e->pvp, n_mu, Lay::K, a.d(), n_mu, 1.0, 0.0);
  gemm(c, n_mu, n_mu, n_mu, a.d(), n_mu, Lay::MN, e->lpinv, n_mu, Lay::K, kpi.d(), n_mu, 1.0, 0.0, nullptr, true,
       &w);
  ck(mirror_lower(c->stream, kpi.d(), n_mu, n_mu, false), "mirror");
  to_sorted(kpi.d(), e->pvp);
  ck(cudaMemcpyAsync(a.p, e->t, nn * sizeof(double), cudaMemcpyDeviceToDevice, c->stream), "D2D");
  to_sorted(a.d(), e->t);
  ck(cudaStreamSynchronize(c->stream), "sync");
  ctx_free(c, e->theta);
  e->theta = static_cast<double*>(theta.take());
  ctx_free(c, e->lp);
  ctx_free(c, e->lpinv);
  e->lp = e->lpinv = nullptr;
  e->implicit = false;
}

extern "C" {

int lrgw_epsilon_inverse_apply(lrgw_ctx c, lrgw_eps e, const double* x, int m, double* y) {
  return guarded(c, [&] {
    if (!e || !e->ctx) fail(LRGW_ERR_INVALID_INPUT, "epsilon_inverse_apply: null handle");
    if (eps_is_panel(e)) fail(LRGW_ERR_INVALID_INPUT, "epsilon_inverse_apply: row-panel handle (use lrgw_eps_apply_sharded)");
    const size_t n = (size_t)e->n_r * m;
    DBuf dx = upload(c, x, n), dy = dalloc(c, n);
    eps_apply_impl(c, e, dx.d(), e->n_r, m, dy.d(), e->n_r);
    download(c, y, dy.p, n * sizeof(double));
  });
}

int lrgw_eps_apply_dev(lrgw_ctx c, lrgw_eps e, const double* x, long long ldx, int m, double* y, long long ldy) {
  return guarded(c, [&] {
    if (!e || !e->ctx) fail(LRGW_ERR_INVALID_INPUT, "epsilon_inverse_apply: null handle");
    if (eps_is_panel(e)) fail(LRGW_ERR_INVALID_INPUT, "epsilon_inverse_apply: row-panel handle (use lrgw_eps_apply_sharded)");
    if (ldx < e->n_r || ldy < e->n_r) fail(LRGW_ERR_INVALID_INPUT, "epsilon_inverse_apply: row mismatch");
    eps_apply_impl(c, e, x, ldx, m, y, ldy);
    ck(cudaStreamSynchronize(c->stream), "sync");
  });
}

int lrgw_eps_get(lrgw_ctx c, lrgw_eps e, double* k, double* p, double* vp, double* t, int32_t* pts) {
  return guarded(c, [&] {
    if (!e || !e->ctx) fail(LRGW_ERR_INVALID_INPUT, "eps: null handle");
    const size_t nn = (size_t)e->n_mu * e->n_mu, np = (size_t)e->n_r * e->n_mu;
    if ((p || vp) && eps_is_panel(e)) fail(LRGW_ERR_INVALID_INPUT, "eps_get: P / VP of a row-panel handle (use lrgw_eps_info_get)");
    if (k || p || vp || t) eps_explicit(c, e);
    if (k) download(c, k, e->k, nn * sizeof(double));
    if (p) download(c, p, e->theta, np * sizeof(double));
    if (t && e->t) download(c, t, e->t, nn * sizeof(double));
    if (pts && !e->pts.empty()) std::copy(e->pts.begin(), e->pts.end(), pts);
    if (vp) {
      DBuf dvp = dalloc(c, np);
      coulomb_apply(c, e->dims, e->cell, e->zero, e->theta, e->n_r, e->n_mu, dvp.d(), e->n_r);
      download(c, vp, dvp.p, np * sizeof(double));
    }
  });
}

int lrgw_eps_shape(lrgw_eps e, int* n_r, int* n_mu) {
  if (!e) return LRGW_ERR_INVALID_INPUT;
  if (n_r) *n_r = e->n_r;
  if (n_mu) *n_mu = e->n_mu;
  return LRGW_OK;
}

int lrgw_eps_destroy(lrgw_eps e) {
  if (!e) return LRGW_OK;
  if (lrgw_ctx c = e->ctx) {  // null once the context is gone (buffers already freed)
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    ctx_free(c, e->theta);
    ctx_free(c, e->k);
    ctx_free(c, e->t);
    ctx_free(c, e->pvp);
    ctx_free(c, e->lp);
    ctx_free(c, e->lpinv);
    std::lock_guard<std::mutex> lk(c->mem_mu);
    c->live_eps.erase(e);
  }
  delete e;
  return LRGW_OK;
}

int lrgw_eps_info_get(lrgw_eps e, lrgw_eps_info* out) {
  if (!e || !out) return LRGW_ERR_INVALID_INPUT;
  if (e->implicit) {  // the pointers below are the explicit Theta / K / T
    const int st = guarded(e->ctx, [&] { eps_explicit(e->ctx, e); });
    if (st != LRGW_OK) return st;
  }
  out->n_r = e->n_r;
  out->n_mu = e->n_mu;
  out->theta = e->theta;
  out->k = e->k;
  out->t = e->t;
  out->pvp = e->pvp;
  out->min_margin = e->min_margin;
  out->min_margin_step = e->min_margin_step;
  out->fit_path = e->fit_path;
  out->lp_diag_ratio = e->lp_diag_ratio;
  out->select_blocks = e->select_blocks;
  return LRGW_OK;
}

int lrgw_eps_device_ptrs(lrgw_eps e, double** theta, double** k, double** t) {
  if (!e) return LRGW_ERR_INVALID_INPUT;
  if (e->implicit) {
    const int st = guarded(e->ctx, [&] { eps_explicit(e->ctx, e); });
    if (st != LRGW_OK) return st;
  }
  if (theta) *theta = e->theta;
  if (k) *k = e->k;
  if (t) *t = e->t;
  return LRGW_OK;
}

// ---- the whole build --------------------------------------------------------
}  // extern "C"

namespace lrgw_impl {

BuildSetup validate_build(lrgw_ctx c, const lrgw_build_params* prm, const double* phi_v, long long ldv,
                          const double* phi_c, long long ldc, const double* energies, int panel_rows) {
  if (!prm) fail(LRGW_ERR_INVALID_INPUT, "lrgw_build: null argument");
  const lrgw_build_params& P = *prm;
  check_grid(P.dims, P.cell);
  const int n_r = P.n_r, n_v = P.n_v, n_c = P.n_c;
  if ((long long)P.dims[0] * P.dims[1] * P.dims[2] != n_r) fail(LRGW_ERR_INVALID_INPUT, "lrgw_build: grid / N_r mismatch");
  if (n_v < 1 || n_c < 1) fail(LRGW_ERR_INVALID_INPUT, "lrgw_build: need n_v >= 1 and n_c >= 1");
  if (P.n_e < n_v + n_c) fail(LRGW_ERR_INVALID_INPUT, "lrgw_build: energies must hold n_v + n_c values");
  if (!phi_v || !phi_c || !energies) fail(LRGW_ERR_INVALID_INPUT, "lrgw_build: null orbital / energy pointer");
  if (ldv < panel_rows || ldc < panel_rows) fail(LRGW_ERR_INVALID_INPUT, "lrgw_build: leading dimension below the row count");
  for (const double* ph : {phi_v, phi_c}) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, ph) != cudaSuccess || at.type != cudaMemoryTypeDevice || at.device != c->device) {
      cudaGetLastError();
      fail(LRGW_ERR_INVALID_INPUT, "lrgw_build: orbitals must be device memory on the context's GPU");
    }
  }
  BuildSetup b;
  if (lrgw_num_aux(P.k_mu, n_v, n_c, &b.n_mu) != LRGW_OK) fail(LRGW_ERR_INVALID_INPUT, "num_aux: k_mu must be > 0");
  b.n_mu = std::clamp(b.n_mu, 1, n_r);
  host_status(lrgw_host::elliptic_params(energies, P.n_e, n_v, n_c, P.delta_rel > 0 ? P.delta_rel : 1e-7,
                                         P.max_nodes > 0 ? P.max_nodes : 1025, &b.spec),
              "elliptic_params");
  return b;
}

void timing_begin(lrgw_ctx c) {
  for (auto& x : c->ev)
    if (!x) ck(cudaEventCreate(&x), "event");
  for (auto& x : c->ev_quad)
    if (!x) ck(cudaEventCreate(&x), "event");
  for (auto& x : c->ev_lib)
    if (!x) ck(cudaEventCreate(&x), "event");
  c->lib_ms = 0.0;
  c->timing = true;
  mark(c, 0);
}

// Stage times of the build from its 9 boundary events (mark 0 .. 8).
void timing_end(lrgw_ctx c) {
  ck(cudaEventSynchronize(c->ev[8]), "sync");
  float ms;
  for (int i = 0; i < 8; ++i) {
    cudaEventElapsedTime(&ms, c->ev[i], c->ev[i + 1]);
    c->stage_ms[i] = ms;
  }
  cudaEventElapsedTime(&ms, c->ev[0], c->ev[8]);
  c->stage_ms[LRGW_STAGE_TOTAL] = ms;
  c->stage_ms[LRGW_STAGE_QUAD_KERNEL] = 0.0;
  if (c->quad_timed && cudaEventElapsedTime(&ms, c->ev_quad[0], c->ev_quad[1]) == cudaSuccess)
    c->stage_ms[LRGW_STAGE_QUAD_KERNEL] = ms;
  c->quad_timed = false;
  c->stage_ms[LRGW_STAGE_CUSOLVER] = c->lib_ms;
  c->stage_ms[LRGW_STAGE_CUFFT] = c->stage_ms[LRGW_STAGE_FFT];
  c->timing = false;
}

// Implicit-Theta build, stages 2-5 after the selection (lrgw_ctx_set_theta_implicit).
// Theta = L L_P^-1 (the fused fit's identity) is kept factored instead of
// formed: with T_pi (T over the points in pivot order),
//   T' = L_P^-1 T_pi L_P^-T,  P' = L^T V L,  K' = (T'^-1 / 2 - P')^-1
// gives Theta K Theta^T = L K' L^T exactly (K' = L_P^-1 K_pi L_P^-T), so the
// probe apply runs on (L, K') unchanged and the N_r x N_mu^2 fit GEMM is not
// needed by the build; eps_explicit() forms Theta, K, T, Theta^T V Theta in
// the sorted-point order when a caller asks for them. Returns nullptr when
// L_P has a tiny pivot (the caller takes the explicit path).
lrgw_eps_s* build_implicit(lrgw_ctx c, const lrgw_build_params& P, const BuildSetup& bs, const double* phi_v,
                           long long ldv, const double* phi_c, long long ldc, const double* energies,
                           const std::vector<int32_t>& pts, SelectKeep& keep) {
  const int n_r = P.n_r, n_v = P.n_v, n_c = P.n_c, n_mu = bs.n_mu, n_e = P.n_e;
  const size_t nn = (size_t)n_mu * n_mu;
  const lrgw_host::Spec& spec = bs.spec;
  // stage 2 (solve only): L_P and L_P^-1 (the fused fit's checks)
  mark(c, 2);
  std::vector<int> order(keep.order.begin(), keep.order.end());
  DBuf dorder = upload_i(c, order.data(), n_mu);
  DBuf lp = dalloc(c, nn), lpinv = dalloc(c, nn);
  ck(gather_rows(c->stream, keep.L.d(), n_r, n_mu, dorder.i(), n_mu, lp.d(), n_mu), "gather");
  ck(zero_strict_upper(c->stream, lp.d(), n_mu, n_mu), "zero_upper");
  std::vector<double> diag(n_mu);
  ck(cudaMemcpy2DAsync(diag.data(), sizeof(double), lp.d(), (size_t)(n_mu + 1) * sizeof(double), sizeof(double),
                       n_mu, cudaMemcpyDeviceToHost, c->stream),
     "D2H diag");
  ck(cudaStreamSynchronize(c->stream), "sync");
  double gmax = 0.0, dmin = HUGE_VAL, dmax = 0.0;
  for (double v : diag) {
    gmax = std::max(gmax, v * v);
    dmin = std::min(dmin, std::abs(v));
    dmax = std::max(dmax, std::abs(v));
  }
  const double tiny = 1e-14 * (gmax > 0.0 ? gmax : 1.0);
  for (double v : diag)
    if (!(v * v >= tiny)) return nullptr;
  ck(cudaMemcpyAsync(lpinv.p, lp.p, nn * sizeof(double), cudaMemcpyDeviceToDevice, c->stream), "D2D");
  {
    DBuf work = dalloc(c, trtri_work_elems(n_mu));
    DBuf bad = ialloc(c, 1);
    const int big = 0x7fffffff;
    ck(cudaMemcpyAsync(bad.p, &big, sizeof(int), cudaMemcpyHostToDevice, c->stream), "H2D");
    ck(lrgw_dev::trtri_lower(c->stream, lpinv.d(), n_mu, n_mu, work.d(), bad.i(), c->sm_count), "trtri");
    int h = 0;
    download(c, &h, bad.p, sizeof(int));
    if (h != big) return nullptr;
  }
  mark(c, 3);
  mark(c, 4);  // no fit GEMM
  // stage 3: T over the points in pivot order
  DBuf pv = dalloc(c, (size_t)n_mu * n_v), pc = dalloc(c, (size_t)n_mu * n_c);
  ck(gather_rows(c->stream, phi_v, ldv, n_v, dorder.i(), n_mu, pv.d(), n_mu), "gather");
  ck(gather_rows(c->stream, phi_c, ldc, n_c, dorder.i(), n_mu, pc.d(), n_mu), "gather");
  DBuf t = dalloc(c, nn);
  if (spec.bypass) {
    direct_impl(c, pv.d(), n_mu, pc.d(), n_mu, n_mu, n_v, n_c, energies, t.d(), n_mu);
  } else if (P.n_lambda > 0) {
    fixed_impl(c, pv.d(), n_mu, pc.d(), n_mu, n_mu, n_v, n_c, energies, n_e, P.n_lambda, t.d(), n_mu);
  } else {
    adaptive_impl(c, pv.d(), n_mu, pc.d(), n_mu, n_mu, n_v, n_c, energies, spec, t.d());
  }
  // T' = L_P^-1 T L_P^-T (symmetric by the mirror of its lower triangle)
  DBuf tp = dalloc(c, nn), tmp = dalloc(c, nn);
  {
    Work w = make_work(c, 8 * nn);
    gemm(c, n_mu, n_mu, n_mu, lpinv.d(), n_mu, Lay::MN, t.d(), n_mu, Lay::K, tmp.d(), n_mu, 1.0, 0.0);
    gemm(c, n_mu, n_mu, n_mu, tmp.d(), n_mu, Lay::MN, lpinv.d(), n_mu, Lay::MN, tp.d(), n_mu, 1.0, 0.0, nullptr,
         true, &w);
    ck(mirror_lower(c->stream, tp.d(), n_mu, n_mu, false), "mirror");
  }
  mark(c, 5);
  // stages 4-5 on (L, T'): chol(-T') under the Coulomb stage, P' = L^T V L
  DBuf pvp = dalloc(c, nn), k = dalloc(c, nn);
  SmwState smw;
  cudaStream_t side = side_stream(c);
  ck(cudaEventRecord(c->ev_side, c->stream), "cudaEventRecord");
  ck(cudaStreamWaitEvent(side, c->ev_side, 0), "cudaStreamWaitEvent");
  smw_factor_t(c, side, tp.d(), n_mu, smw);
  pvp_impl(c, P.dims, P.cell, P.zero_kernel, keep.L.d(), n_r, n_mu, pvp.d());
  mark(c, 7);
  smw_join(c, smw);
  smw_finish(c, smw, pvp.d(), n_mu, k.d());
  mark(c, 8);
  timing_end(c);
  auto* e = new_eps(c);
  e->ctx = c;
  e->n_r = n_r;
  e->n_mu = n_mu;
  std::memcpy(e->dims, P.dims, sizeof(e->dims));
  std::memcpy(e->cell, P.cell, sizeof(e->cell));
  e->zero = P.zero_kernel;
  e->theta = static_cast<double*>(keep.L.take());
  e->k = static_cast<double*>(k.take());
  e->t = static_cast<double*>(t.take());
  e->pvp = static_cast<double*>(pvp.take());
  e->lp = static_cast<double*>(lp.take());
  e->lpinv = static_cast<double*>(lpinv.take());
  e->pts = pts;
  e->colmap.resize(n_mu);
  for (int q = 0; q < n_mu; ++q)
    e->colmap[q] = (int)(std::lower_bound(pts.begin(), pts.end(), order[q]) - pts.begin());
  e->implicit = true;
  e->fit_path = 2;  // implicit
  e->lp_diag_ratio = dmin > 0.0 ? (dmax / dmin) * (dmax / dmin) : HUGE_VAL;
  e->row0 = 0;
  e->rows = n_r;
  return e;
}

// The one-GPU build, stages 1-5 (stage boundaries marked for the timings).
lrgw_eps_s* build_one(lrgw_ctx c, const lrgw_build_params& P, const BuildSetup& bs, const double* phi_v,
                      long long ldv, const double* phi_c, long long ldc, const double* energies) {
  const int n_r = P.n_r, n_v = P.n_v, n_c = P.n_c, n_mu = bs.n_mu, n_e = P.n_e;
  const lrgw_host::Spec& spec = bs.spec;
  struct TimingGuard {
    lrgw_ctx c;
    ~TimingGuard() { c->timing = false; }
  } tg{c};
  timing_begin(c);
  // stage 1
  SelectKeep keep;
  keep.min_l_elems = (size_t)2 * half_len(P.dims) * n_mu;
  double min_margin = -1.0;  // smallest relative top-2 residual margin over all steps (linalg.hpp:45-47)
  std::vector<int32_t> pts = select_impl(c, phi_v, ldv, n_v, phi_c, ldc, n_c, n_r, n_mu, &min_margin, &keep);
  mark(c, 1);
  if (c->theta_implicit && keep.steps == n_mu) {
    lrgw_eps_s* e = build_implicit(c, P, bs, phi_v, ldv, phi_c, ldc, energies, pts, keep);
    if (e) {
      e->min_margin = min_margin;
      e->min_margin_step = keep.min_margin_step;
      e->select_blocks = keep.blocks;
      return e;
    }
  }
  // stage 2: fused fit from the selection's factor (explicit path otherwise)
  DBuf theta = dalloc(c, (size_t)n_r * n_mu);
  mark(c, 2);  // FIT_LHS is empty on the fused path (lhs lives in L)
  FusedFit ff;
  bool fused = fused_fit(c, keep, n_r, pts, n_mu, theta.d(), n_r, ff);
  keep.L.release();
  if (!fused) {  // explicit path re-marks its own lhs / solve boundaries
    fit_impl(c, phi_v, ldv, n_v, phi_c, ldc, n_c, n_r, pts.data(), n_mu, theta.d(), n_r);
  }
  mark(c, 4);
  // stage 3
  DBuf dpts = upload_i(c, pts.data(), n_mu);
  DBuf pv = dalloc(c, (size_t)n_mu * n_v), pc = dalloc(c, (size_t)n_mu * n_c);
  ck(gather_rows(c->stream, phi_v, ldv, n_v, dpts.i(), n_mu, pv.d(), n_mu), "gather");
  ck(gather_rows(c->stream, phi_c, ldc, n_c, dpts.i(), n_mu, pc.d(), n_mu), "gather");
  DBuf t = dalloc(c, (size_t)n_mu * n_mu);
  if (spec.bypass) {
    direct_impl(c, pv.d(), n_mu, pc.d(), n_mu, n_mu, n_v, n_c, energies, t.d(), n_mu);
  } else if (P.n_lambda > 0) {
    fixed_impl(c, pv.d(), n_mu, pc.d(), n_mu, n_mu, n_v, n_c, energies, n_e, P.n_lambda, t.d(), n_mu);
  } else {
    adaptive_impl(c, pv.d(), n_mu, pc.d(), n_mu, n_mu, n_v, n_c, energies, spec, t.d());
  }
  mark(c, 5);
  // stages 4-5: R = chol(-T) (a latency-bound leaf that needs T only) runs on
  // the side stream under the Coulomb stage; smw_factor_t joins it back
  DBuf pvp = dalloc(c, (size_t)n_mu * n_mu), k = dalloc(c, (size_t)n_mu * n_mu);
  SmwState smw;
  cudaStream_t side = side_stream(c);
  ck(cudaEventRecord(c->ev_side, c->stream), "cudaEventRecord");
  ck(cudaStreamWaitEvent(side, c->ev_side, 0), "cudaStreamWaitEvent");
  smw_factor_t(c, side, t.d(), n_mu, smw);
  pvp_impl(c, P.dims, P.cell, P.zero_kernel, theta.d(), n_r, n_mu, pvp.d());
  mark(c, 7);
  smw_join(c, smw);
  double lp_ratio = 0.0;
  if (smw_finish(c, smw, pvp.d(), n_mu, k.d(), fused ? &ff : nullptr)) {
    if (fused) lp_ratio = ff.ratio();
  } else {  // L_P failed the LU rule: the reference's explicit fit, then stages 4-5 again
    fused = false;
    fit_impl(c, phi_v, ldv, n_v, phi_c, ldc, n_c, n_r, pts.data(), n_mu, theta.d(), n_r);
    pvp_impl(c, P.dims, P.cell, P.zero_kernel, theta.d(), n_r, n_mu, pvp.d());
    smw_core(c, t.d(), pvp.d(), n_mu, k.d());
  }
  mark(c, 8);
  timing_end(c);
  auto* e = new_eps(c);
  e->ctx = c;
  e->n_r = n_r;
  e->n_mu = n_mu;
  std::memcpy(e->dims, P.dims, sizeof(e->dims));
  std::memcpy(e->cell, P.cell, sizeof(e->cell));
  e->zero = P.zero_kernel;
  e->theta = static_cast<double*>(theta.take());
  e->k = static_cast<double*>(k.take());
  e->t = static_cast<double*>(t.take());
  e->pvp = static_cast<double*>(pvp.take());
  e->pts = pts;
  e->min_margin = min_margin;
  e->min_margin_step = keep.min_margin_step;
  e->fit_path = fused ? 0 : 1;
  e->lp_diag_ratio = lp_ratio;
  e->select_blocks = keep.blocks;
  e->row0 = 0;
  e->rows = n_r;
  return e;
}

}  // namespace lrgw_impl

extern "C" {

int lrgw_build(lrgw_ctx c, const lrgw_build_params* prm, const double* phi_v, long long ldv, const double* phi_c,
               long long ldc, const double* energies, lrgw_eps* out) {
  return guarded(c, [&] {
    if (!out) fail(LRGW_ERR_INVALID_INPUT, "lrgw_build: null argument");
    const BuildSetup bs = validate_build(c, prm, phi_v, ldv, phi_c, ldc, energies, prm ? prm->n_r : 0);
    *out = build_one(c, *prm, bs, phi_v, ldv, phi_c, ldc, energies);
  });
}

// ---- stage-level device API -------------------------------------------------
int lrgw_dev_select(lrgw_ctx c, const double* a, long long lda, int n1, const double* b, long long ldb, int n2,
                    int n_r, int n_mu, int32_t* pts_host, double* min_margin) {
  return guarded(c, [&] {
    std::vector<int32_t> p = select_impl(c, a, lda, n1, b, ldb, n2, n_r, n_mu, min_margin);
    std::copy(p.begin(), p.end(), pts_host);
  });
}

int lrgw_dev_fit(lrgw_ctx c, const double* a, long long lda, int n1, const double* b, long long ldb, int n2, int n_r,
                 const int32_t* pts_host, int n_mu, double* theta, long long ldt) {
  return guarded(c, [&] {
    fit_impl(c, a, lda, n1, b, ldb, n2, n_r, pts_host, n_mu, theta, ldt);
    ck(cudaStreamSynchronize(c->stream), "sync");
  });
}

int lrgw_dev_fit_panel(lrgw_ctx c, const double* a, long long lda, int n1, const double* b, long long ldb, int n2,
                       int rows, const double* a_mu, const double* b_mu, const double* g_inv, int n_mu, double* theta,
                       long long ldt) {
  return guarded(c, [&] {
    DBuf lhs = dalloc(c, (size_t)rows * n_mu);
    ck(hadamard_gemm(c->stream, rows, n_mu, a, lda, a_mu, n_mu, n1, b, ldb, b_mu, n_mu, n2, lhs.d(), rows, 1.0, 0.0),
       "hadamard_gemm");
    gemm(c, rows, n_mu, n_mu, lhs.d(), rows, Lay::MN, g_inv, n_mu, Lay::MN, theta, ldt, 1.0, 0.0);
    ck(cudaStreamSynchronize(c->stream), "sync");
  });
}

int lrgw_dev_contour_partial(lrgw_ctx c, const double* pv, long long ldv, const double* pc, long long ldpc, int n_mu,
                             int n_v, int n_c, const double* e, int n_e, int n_lambda, int node0, int count,
                             double* acc) {
  return guarded(c, [&] {
    check_coupled(n_mu, n_v, n_c, n_e);
    lrgw_host::Spec s;
    host_status(lrgw_host::elliptic_params(e, n_e, n_v, n_c, 1e-7, 1025, &s), "elliptic_params");
    if (s.bypass) fail(LRGW_ERR_INVALID_INPUT, "contour quadrature: spec is bypass-flagged; use the direct sum");
    NodeSet all = trapezoid(s, n_lambda), ns;
    for (int k = node0; k < node0 + count && k < (int)all.nodes.size(); ++k) {
      ns.nodes.push_back(all.nodes[k]);
      ns.weights.push_back(all.weights[k]);
    }
    std::vector<double> dv, dc, gw;
    node_tables_or_fail(s, e, n_v, n_c, ns, &dv, &dc, &gw);
    quad_run(c, pv, ldv, pc, ldpc, n_mu, n_v, n_c, dv, dc, gw, (int)ns.nodes.size(), nullptr, 0.0, 1.0, acc, n_mu);
    ck(cudaStreamSynchronize(c->stream), "sync");
  });
}

int lrgw_dev_contour_fixed(lrgw_ctx c, const double* pv, long long ldv, const double* pc, long long ldpc, int n_mu,
                           int n_v, int n_c, const double* e, int n_e, int n_lambda, double* t, long long ldt) {
  return guarded(c, [&] {
    check_coupled(n_mu, n_v, n_c, n_e);
    fixed_impl(c, pv, ldv, pc, ldpc, n_mu, n_v, n_c, e, n_e, n_lambda, t, ldt);
    ck(cudaStreamSynchronize(c->stream), "sync");
  });
}

int lrgw_dev_pvp(lrgw_ctx c, const int* dims, const double* cell, int zero, const double* theta, long long ldt,
                 int n_mu, double* pvp) {
  return guarded(c, [&] {
    check_grid(dims, cell);
    pvp_impl(c, dims, cell, zero, theta, ldt, n_mu, pvp);
    ck(cudaStreamSynchronize(c->stream), "sync");
  });
}

int lrgw_dev_smw_core(lrgw_ctx c, const double* t, const double* pvp, int n_mu, double* k) {
  return guarded(c, [&] {
    smw_core(c, t, pvp, n_mu, k);
    ck(cudaStreamSynchronize(c->stream), "sync");
  });
}

int lrgw_dev_coulomb_apply(lrgw_ctx c, const int* dims, const double* cell, int zero, const double* x, long long ldx,
                           int m, double* y, long long ldy) {
  return guarded(c, [&] {
    check_grid(dims, cell);
    coulomb_apply(c, dims, cell, zero, x, ldx, m, y, ldy);
    ck(cudaStreamSynchronize(c->stream), "sync");
  });
}

int lrgw_dev_dgemm(lrgw_ctx c, char ta, char tb, int m, int n, int k, double alpha, const double* a, long long lda,
                   const double* b, long long ldb, double beta, double* cm, long long ldc) {
  return guarded(c, [&] {
    const bool at = ta == 'T' || ta == 't', bt = tb == 'T' || tb == 't';
    // probe-shaped products (<= 16 columns against a tall panel): the K7
    // streams of the probe apply instead of the tiled engine
    const bool plain = alpha == 1.0 && beta == 0.0 && !bt && skinny_supported(n) && k > 0 && m > 0;
    if (plain && at && (long long)k >= 8LL * m) {  // u = A^T x, A: k x m (Theta panel), x: k x n
      Work w = make_work(c, (size_t)1200 * m * n);
      ck(skinny_tn(c->stream, a, lda, k, m, b, ldb, n, cm, ldc, w.buf.d(), w.elems, c->sm_count), "skinny_tn");
    } else if (plain && !at && (long long)m >= 8LL * k && (size_t)k * n * 8 <= 200 * 1024) {  // z = A w
      ck(skinny_nn(c->stream, a, lda, m, k, b, ldb, n, cm, ldc, c->sm_count), "skinny_nn");
    } else {
      Work w = make_work(c, (size_t)8 * m * n);
      gemm(c, m, n, k, a, lda, at ? Lay::K : Lay::MN, b, ldb, bt ? Lay::MN : Lay::K, cm, ldc, alpha, beta, nullptr,
           false, &w);
    }
    ck(cudaStreamSynchronize(c->stream), "sync");
  });
}

int lrgw_dev_hadamard(lrgw_ctx c, int m, int n, const double* a1, long long lda1, const double* b1, long long ldb1,
                      int k1, const double* a2, long long lda2, const double* b2, long long ldb2, int k2, double* cm,
                      long long ldc) {
  return guarded(c, [&] {
    if (m < 0 || n < 0 || k1 < 1 || k2 < 1 || lda1 < m || lda2 < m || ldb1 < n || ldb2 < n || ldc < m)
      fail(LRGW_ERR_INVALID_INPUT, "hadamard: bad sizes");
    ck(hadamard_gemm(c->stream, m, n, a1, lda1, b1, ldb1, k1, a2, lda2, b2, ldb2, k2, cm, ldc, 1.0, 0.0),
       "hadamard_gemm");
    ck(cudaStreamSynchronize(c->stream), "sync");
  });
}

int lrgw_dev_trtri_lower(lrgw_ctx c, double* a, int n, long long lda) {
  return guarded(c, [&] {
    if (n < 0 || lda < std::max(1, n)) fail(LRGW_ERR_INVALID_INPUT, "trtri: bad sizes");
    DBuf work = dalloc(c, trtri_work_elems(n));
    DBuf bad = ialloc(c, 1);
    const int big = 0x7fffffff;
    ck(cudaMemcpyAsync(bad.p, &big, sizeof(int), cudaMemcpyHostToDevice, c->stream), "H2D");
    ck(lrgw_dev::trtri_lower(c->stream, a, n, lda, work.d(), bad.i(), c->sm_count), "trtri");
    int h = 0;
    download(c, &h, bad.p, sizeof(int));
    if (h != big) fail(LRGW_ERR_SINGULAR, "trtri: singular factor", h - 1);
  });
}

int lrgw_dev_select_topk(lrgw_ctx c, const double* d, const int32_t* pos, int n_r, int k, int s1, int32_t* rows,
                         double* vals, int32_t* poss) {
  return guarded(c, [&] {
    if (n_r < 1 || s1 < 1 || s1 > select_max_candidates() + 1) fail(LRGW_ERR_INVALID_INPUT, "select_topk: bad sizes");
    DBuf tmp(c, select_topk_tmp_bytes(n_r, s1));
    DBuf out(c, (size_t)s1 * sizeof(HostEnt));
    ck(select_topk_reset(c->stream, tmp.p), "select_topk_reset");
    ck(select_topk(c->stream, d, pos, n_r, k, s1, tmp.p, out.p), "select_topk");
    std::vector<HostEnt> h(s1);
    download(c, h.data(), out.p, sizeof(HostEnt) * s1);
    for (int i = 0; i < s1; ++i) {
      if (rows) rows[i] = h[i].row;
      if (vals) vals[i] = h[i].v;
      if (poss) poss[i] = h[i].pos;
    }
  });
}

int lrgw_dev_cand_greedy(lrgw_ctx c, int n_r, int s, int steps, int k, const double* top_vals,
                         const int32_t* top_pos, const int32_t* top_rows, const double* wcc, int32_t* pos,
                         int32_t* perm, double* x, int32_t* piv_rows, double* margins, int32_t* b) {
  return guarded(c, [&] {
    if (n_r < 1 || s < 1 || s > select_max_candidates() || k < 0 || steps > n_r || k >= steps)
      fail(LRGW_ERR_INVALID_INPUT, "cand_greedy: bad sizes");
    std::vector<HostEnt> h(s + 1);
    for (int i = 0; i <= s; ++i) h[i] = HostEnt{top_vals[i], top_pos[i], top_rows[i]};
    DBuf top(c, sizeof(HostEnt) * (s + 1));
    ck(cudaMemcpyAsync(top.p, h.data(), sizeof(HostEnt) * (s + 1), cudaMemcpyHostToDevice, c->stream), "H2D");
    DBuf order = ialloc(c, steps);
    DBuf marg = dalloc(c, steps);
    DBuf bout = ialloc(c, 2);
    ck(select_cand_greedy(c->stream, n_r, s, steps, k, top.p, wcc, pos, perm, x, (int*)order.p,
                          margins ? (double*)marg.p : nullptr, (int*)bout.p, s, 0),
       "cand_greedy");
    int nb[2] = {0, 0};
    download(c, nb, bout.p, sizeof(nb));
    *b = nb[0];
    if (nb[0] > 0) {
      download(c, piv_rows, (int*)order.p + k, sizeof(int) * nb[0]);
      if (margins) download(c, margins, (double*)marg.p + k, sizeof(double) * nb[0]);
    }
  });
}

int lrgw_dev_theta_from_factor(lrgw_ctx c, const double* l, long long ldl, int rows, int n_mu, const double* x,
                               long long ldx, const int32_t* colmap, double* theta, long long ldt) {
  return guarded(c, [&] {
    if (rows < 0 || n_mu < 1 || ldl < std::max(rows, 1) || ldx < n_mu || ldt < std::max(rows, 1))
      fail(LRGW_ERR_INVALID_INPUT, "theta_from_factor: bad sizes");
    std::vector<int> map(colmap, colmap + n_mu);
    std::vector<char> seen(n_mu, 0);
    for (int q : map) {
      if (q < 0 || q >= n_mu || seen[q]) fail(LRGW_ERR_INVALID_INPUT, "theta_from_factor: colmap is not a permutation");
      seen[q] = 1;
    }
    if (rows == 0) return;
    DBuf dmap = upload_i(c, map.data(), n_mu);
    DBuf xt = dalloc(c, (size_t)n_mu * n_mu);
    ck(transpose(c->stream, x, ldx, n_mu, n_mu, xt.d(), n_mu), "transpose");
    ck(dgemm(c->stream, rows, n_mu, n_mu, l, ldl, Lay::MN, xt.d(), n_mu, Lay::MN, theta, ldt, 1.0, 0.0, nullptr,
             false, c->sm_count, nullptr, 0, true, dmap.i()),
       "dgemm(theta)");
    ck(cudaStreamSynchronize(c->stream), "sync");
  });
}

int lrgw_dev_select_panel_update(lrgw_ctx c, const double* a, long long lda, int n1, const double* b, long long ldb,
                                 int n2, int rows, double* l, long long ldl, int k, int nb, const double* piv,
                                 long long ldpiv, const double* x, long long ldx, const int32_t* pos, double* d) {
  return guarded(c, [&] {
    if (rows < 1 || n1 < 1 || n2 < 1 || nb < 1 || k < 0 || ldl != rows || lda < rows || ldb < rows || ldx < nb ||
        ldpiv < nb)
      fail(LRGW_ERR_INVALID_INPUT, "select_panel_update: bad sizes");
    const int width = n1 + n2 + k;
    const int ldp = nb + (nb & 1);  // even leading dim: 16-byte operand loads
    DBuf pr = dalloc(c, (size_t)ldp * width);
    ck(cudaMemcpy2DAsync(pr.d(), ldp * sizeof(double), piv, ldpiv * sizeof(double), nb * sizeof(double), width,
                         cudaMemcpyDeviceToDevice, c->stream),
       "D2D");
    const double* amu = pr.d();
    const double* bmu = amu + (size_t)ldp * n1;
    const double* lsel = bmu + (size_t)ldp * n2;
    const cudaError_t pe =
        (fused_downdate_enabled() && select_panel_enabled(n1, n2))
            ? select_panel(c->stream, rows, nb, a, lda, amu, ldp, n1, b, ldb, bmu, ldp, n2, l, ldl, lsel, ldp, k, x,
                           ldx, l + (size_t)k * ldl, ldl, d, pos, k + nb)
            : cudaErrorNotSupported;
    if (pe != cudaErrorNotSupported) {
      ck(pe, "select_panel");
      ck(cudaStreamSynchronize(c->stream), "sync");
      return;
    }
    cudaGetLastError();
    DBuf wsel = dalloc(c, (size_t)rows * nb);
    ck(hadamard_gemm(c->stream, rows, nb, a, lda, amu, ldp, n1, b, ldb, bmu, ldp, n2, wsel.d(), rows, 1.0, 0.0),
       "hadamard_gemm");
    if (k > 0) gemm(c, rows, nb, k, l, ldl, Lay::MN, lsel, ldp, Lay::MN, wsel.d(), rows, -1.0, 1.0);
    cudaError_t fe = fused_downdate_enabled() && ldl == rows
                         ? dgemm_tall_downdate(c->stream, rows, nb, nb, wsel.d(), rows, x, ldx, l + (size_t)k * ldl,
                                               ldl, d, pos, k + nb)
                         : cudaErrorNotSupported;
    if (fe == cudaErrorNotSupported) {
      cudaGetLastError();
      gemm(c, rows, nb, nb, wsel.d(), rows, Lay::MN, x, ldx, Lay::MN, l + (size_t)k * ldl, ldl, 1.0, 0.0);
      ck(select_downdate(c->stream, l, rows, k, nb, pos, d), "downdate");
    } else {
      ck(fe, "dgemm_tall_downdate");
    }
    ck(cudaStreamSynchronize(c->stream), "sync");
  });
}

int lrgw_dev_gram_weighted(lrgw_ctx c, const double* x, long long ldx, int kdim, int m, const double* w,
                           double* out, long long ldo) {
  return guarded(c, [&] {
    if (kdim < 1 || m < 1 || ldx < kdim || ldo < m) fail(LRGW_ERR_INVALID_INPUT, "gram_weighted: bad sizes");
    Work wk = make_work(c, (size_t)16 * m * m);
    gemm(c, m, m, kdim, x, ldx, Lay::K, x, ldx, Lay::K, out, ldo, 1.0, 0.0, w, true, &wk);
    ck(mirror_lower(c->stream, out, m, ldo, false), "mirror");
    ck(cudaStreamSynchronize(c->stream), "sync");
  });
}

int lrgw_project_screened_interactions(lrgw_ctx c, lrgw_eps e, const double* p_vn, int n_vn, const double* p_nn,
                                       int n_nn, double* w_vn, double* w_nn, double* v_vn) {
  return guarded(c, [&] {
    if (!e || !e->ctx) fail(LRGW_ERR_INVALID_INPUT, "project_screened_interactions: null handle");
    eps_explicit(c, e);
    if (n_vn < 0 || n_nn < 0 || (n_vn > 0 && !p_vn) || (n_nn > 0 && !p_nn))
      fail(LRGW_ERR_INVALID_INPUT, "project_screened_interactions: bad sizes");
    const size_t n_r = e->n_r;
    DBuf dvn = upload(c, p_vn, n_r * n_vn), dnn = upload(c, p_nn, n_r * n_nn);
    DBuf wvn = dalloc(c, (size_t)n_vn * n_vn), wnn = dalloc(c, (size_t)n_nn * n_nn), vvn = dalloc(c, (size_t)n_vn * n_vn);
    project_impl(c, e, dvn.d(), e->n_r, n_vn, dnn.d(), e->n_r, n_nn, wvn.d(), wnn.d(), vvn.d());
    download(c, w_vn, wvn.p, sizeof(double) * n_vn * n_vn);
    download(c, w_nn, wnn.p, sizeof(double) * n_nn * n_nn);
    download(c, v_vn, vvn.p, sizeof(double) * n_vn * n_vn);
  });
}

int lrgw_dev_project_screened(lrgw_ctx c, lrgw_eps e, const double* p_vn, long long ld_vn, int n_vn,
                              const double* p_nn, long long ld_nn, int n_nn, double* w_vn, double* w_nn,
                              double* v_vn) {
  return guarded(c, [&] {
    if (!e || !e->ctx) fail(LRGW_ERR_INVALID_INPUT, "project_screened_interactions: null handle");
    eps_explicit(c, e);
    if (n_vn < 0 || n_nn < 0 || (n_vn > 0 && ld_vn < e->n_r) || (n_nn > 0 && ld_nn < e->n_r))
      fail(LRGW_ERR_INVALID_INPUT, "project_screened_interactions: bad sizes");
    project_impl(c, e, p_vn, ld_vn, n_vn, p_nn, ld_nn, n_nn, w_vn, w_nn, v_vn);
    ck(cudaStreamSynchronize(c->stream), "sync");
  });
}

int lrgw_self_energies_lowrank(lrgw_ctx c, const double* psi, int n_r, int n_v, int n_c, const int32_t* pts_vn,
                               int n_vn, const int32_t* pts_nn, int n_nn, const double* w_vn, const double* w_nn,
                               const double* v_vn, double* sigma_sex_x, double* sigma_x, double* sigma_coh,
                               double* sigma_total) {
  return guarded(c, [&] {
    const int nb = n_v + n_c;
    if (n_r < 1 || n_v < 0 || n_c < 0 || nb < 1 || n_vn < 0 || n_nn < 0 || !psi)
      fail(LRGW_ERR_INVALID_INPUT, "self_energies_lowrank: bad sizes");
    if ((n_vn > 0 && (!w_vn || !v_vn)) || (n_nn > 0 && !w_nn))
      fail(LRGW_ERR_INVALID_INPUT, "self_energies_lowrank: null interaction block");
    check_points(pts_vn, n_vn, n_r, "self_energies_lowrank: vn");
    check_points(pts_nn, n_nn, n_r, "self_energies_lowrank: nn");
    DBuf dpsi = upload(c, psi, (size_t)n_r * nb);
    DBuf dwvn = upload(c, w_vn, (size_t)n_vn * n_vn), dvvn = upload(c, v_vn, (size_t)n_vn * n_vn);
    DBuf dwnn = upload(c, w_nn, (size_t)n_nn * n_nn);
    DBuf out = dalloc(c, (size_t)3 * nb);
    sigma_impl(c, dpsi.d(), n_r, n_v, nb, pts_vn, n_vn, pts_nn, n_nn, dwvn.d(), dvvn.d(), dwnn.d(), out.d(),
               out.d() + nb, out.d() + 2 * nb);
    std::vector<double> h((size_t)3 * nb);
    download(c, h.data(), out.p, sizeof(double) * 3 * nb);
    for (int n = 0; n < nb; ++n) {
      const double tot = h[n] + h[nb + n] + h[2 * nb + n];  // SelfEnergies::finalize order (gw.hpp:36)
      if (sigma_sex_x) sigma_sex_x[n] = h[n];
      if (sigma_x) sigma_x[n] = h[nb + n];
      if (sigma_coh) sigma_coh[n] = h[2 * nb + n];
      if (sigma_total) sigma_total[n] = tot;
      if (!std::isfinite(tot))
        fail(LRGW_ERR_NUMERIC, "self-energies: non-finite value at band " + std::to_string(n));
    }
  });
}

int lrgw_dev_self_energies(lrgw_ctx c, const double* psi, long long ldp, int n_r, int n_v, int n_c,
                           const int32_t* pts_vn, int n_vn, const int32_t* pts_nn, int n_nn, const double* w_vn,
                           const double* w_nn, const double* v_vn, double* sigma_sex_x, double* sigma_x,
                           double* sigma_coh) {
  return guarded(c, [&] {
    const int nb = n_v + n_c;
    if (n_r < 1 || n_v < 0 || n_c < 0 || nb < 1 || n_vn < 0 || n_nn < 0 || ldp < n_r)
      fail(LRGW_ERR_INVALID_INPUT, "self_energies_lowrank: bad sizes");
    check_points(pts_vn, n_vn, n_r, "self_energies_lowrank: vn");
    check_points(pts_nn, n_nn, n_r, "self_energies_lowrank: nn");
    sigma_impl(c, psi, ldp, n_v, nb, pts_vn, n_vn, pts_nn, n_nn, w_vn, v_vn, w_nn, sigma_sex_x, sigma_x,
               sigma_coh);
    ck(cudaStreamSynchronize(c->stream), "sync");
  });
}

}  // extern "C"

// ---- WFN1 orbital files (model.hpp:236-339) -------------------------------
namespace {
thread_local std::string g_thread_err;

template <class F>
int io_guarded(F&& f) {
  try {
    g_thread_err.clear();
    f();
    return LRGW_OK;
  } catch (const lrgw_host::Wfn1Error& e) {
    g_thread_err = e.what();
    return LRGW_ERR_IO;
  } catch (const Fail& e) {
    g_thread_err = e.msg;
    return e.code;
  } catch (const std::bad_alloc&) {
    g_thread_err = "host allocation failure";
    return LRGW_ERR_INTERNAL;
  } catch (...) {
    g_thread_err = "internal error";
    return LRGW_ERR_INTERNAL;
  }
}
}  // namespace

extern "C" {

const char* lrgw_last_error(void) { return g_thread_err.c_str(); }

int lrgw_wfn1_info(const char* path, int* dims, double* cell, int* n_v, int* n_c) {
  return io_guarded([&] {
    if (!path) fail(LRGW_ERR_INVALID_INPUT, "load_system: null path");
    const lrgw_host::Wfn1Header h = lrgw_host::wfn1_read_header(path);
    for (int k = 0; k < 3; ++k) {
      if (dims) dims[k] = h.dims[k];
      if (cell) cell[k] = h.cell[k];
    }
    if (n_v) *n_v = h.n_v;
    if (n_c) *n_c = h.n_c;
  });
}

int lrgw_wfn1_load(const char* path, double* psi, double* energies, double* vxc) {
  return io_guarded([&] {
    if (!path) fail(LRGW_ERR_INVALID_INPUT, "load_system: null path");
    const lrgw_host::Wfn1Header h = lrgw_host::wfn1_read_header(path);
    const size_t nb = static_cast<size_t>(h.n_v) + h.n_c, n_psi = static_cast<size_t>(h.n_r) * nb;
    const long long off_e = h.payload_offset + static_cast<long long>(n_psi * sizeof(double));
    if (psi) lrgw_host::wfn1_read_payload(path, h.payload_offset, psi, n_psi, "psi");
    std::vector<double> tmp(nb);
    lrgw_host::wfn1_read_payload(path, off_e, energies ? energies : tmp.data(), nb, "energies");
    lrgw_host::wfn1_read_payload(path, off_e + static_cast<long long>(nb * sizeof(double)), vxc ? vxc : tmp.data(),
                                 nb, "vxc");
  });
}

int lrgw_wfn1_load_device(lrgw_ctx c, const char* path, double* psi, long long ld, double* energies, double* vxc) {
  if (!c) return LRGW_ERR_INVALID_INPUT;
  int st = io_guarded([&] {
    use_device(c);
    if (!path || !psi) fail(LRGW_ERR_INVALID_INPUT, "load_system: null argument");
    const lrgw_host::Wfn1Header h = lrgw_host::wfn1_read_header(path);
    const int nb = h.n_v + h.n_c;
    const size_t n_r = static_cast<size_t>(h.n_r);
    if (ld < h.n_r) fail(LRGW_ERR_INVALID_INPUT, "load_system: device leading dimension < N_r");
    // psi streamed in whole-column blocks through two pinned staging buffers:
    // block i is read from the file while block i - 1 is copied to HBM.
    const size_t target = size_t(64) << 20;
    const int cols_blk = static_cast<int>(std::max<size_t>(1, std::min<size_t>(nb, target / (n_r * sizeof(double)))));
    const size_t blk_elems = n_r * cols_blk;
    double* pin[2] = {nullptr, nullptr};
    cudaEvent_t done[2] = {nullptr, nullptr};
    auto cleanup = [&] {
      for (int i = 0; i < 2; ++i) {
        if (done[i]) {
          cudaEventSynchronize(done[i]);
          cudaEventDestroy(done[i]);
        }
        if (pin[i]) cudaFreeHost(pin[i]);
      }
    };
    try {
      for (int i = 0; i < 2; ++i) {
        ck(cudaMallocHost(&pin[i], blk_elems * sizeof(double)), "cudaMallocHost");
        ck(cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming), "cudaEventCreate");
      }
      int slot = 0;
      for (int j0 = 0; j0 < nb; j0 += cols_blk, slot ^= 1) {
        const int cols = std::min(cols_blk, nb - j0);
        ck(cudaEventSynchronize(done[slot]), "cudaEventSynchronize");
        lrgw_host::wfn1_read_payload(path, h.payload_offset + static_cast<long long>(n_r * j0 * sizeof(double)),
                                     pin[slot], n_r * cols, "psi");
        ck(cudaMemcpy2DAsync(psi + static_cast<size_t>(j0) * ld, ld * sizeof(double), pin[slot],
                             n_r * sizeof(double), n_r * sizeof(double), cols, cudaMemcpyHostToDevice, c->stream),
           "H2D psi");
        ck(cudaEventRecord(done[slot], c->stream), "cudaEventRecord");
      }
      const long long off_e = h.payload_offset + static_cast<long long>(n_r * nb * sizeof(double));
      std::vector<double> tmp(nb);
      lrgw_host::wfn1_read_payload(path, off_e, energies ? energies : tmp.data(), nb, "energies");
      lrgw_host::wfn1_read_payload(path, off_e + static_cast<long long>(nb * sizeof(double)),
                                   vxc ? vxc : tmp.data(), nb, "vxc");
      ck(cudaStreamSynchronize(c->stream), "sync");
    } catch (...) {
      cleanup();
      throw;
    }
    cleanup();
  });
  if (st != LRGW_OK) c->err = g_thread_err;
  return st;
}

int lrgw_wfn1_save(const char* path, const int* dims, const double* cell, int n_v, int n_c, const double* psi,
                   const double* energies, const double* vxc) {
  return io_guarded([&] {
    if (!path || !dims || !cell || (n_v + n_c > 0 && (!psi || !energies || !vxc)))
      fail(LRGW_ERR_INVALID_INPUT, "save_system: null argument");
    lrgw_host::wfn1_write(path, dims, cell, n_v, n_c, psi, energies, vxc);
  });
}

}  // extern "C"
