// internal.h — host-side internals of liblrgw_cuda shared by the C-ABI
// translation units (capi.cu: single-GPU entry points; sharded.cu: the
// multi-rank build over a communicator). Not part of the public ABI.
#pragma once

#include <cufft.h>
#include <cusolverDn.h>

#include <cstdint>
#include <map>
#include <mutex>
#include <set>
#include <string>
#include <tuple>
#include <unordered_map>
#include <vector>

#include "elliptic.h"
#include "kernels.h"
#include "lrgw_cuda.h"

namespace lrgw_impl {
using namespace lrgw_dev;

struct Fail {
  int code;
  std::string msg;
  int pivot;
};

[[noreturn]] inline void fail(int code, const std::string& msg, int pivot = -1) { throw Fail{code, msg, pivot}; }

inline void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(LRGW_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
inline void ckf(cufftResult r, const char* what) {
  if (r != CUFFT_SUCCESS) fail(LRGW_ERR_CUDA, std::string(what) + ": cufft error " + std::to_string((int)r));
}
inline void cks(cusolverStatus_t r, const char* what) {
  if (r != CUSOLVER_STATUS_SUCCESS)
    fail(LRGW_ERR_CUDA, std::string(what) + ": cusolver error " + std::to_string((int)r));
}
inline void host_status(int st, const char* what) {
  if (st != lrgw_host::kOk) fail(st, what);
}

}  // namespace lrgw_impl

struct lrgw_comm_s;

struct lrgw_ctx_s {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t own_stream = nullptr;
  cudaStream_t side = nullptr;  // the build's side stream (chol(-T) under the Coulomb stage)
  cudaEvent_t ev_side = nullptr, ev_join = nullptr;
  int* sel_pinned = nullptr;  // the selection's device-loop read-back slots (pinned)
  size_t sel_pinned_n = 0;
  int* sel_flag = nullptr;      // host-mapped slot the greedy writes b into (select_wait_b)
  int* sel_flag_dev = nullptr;  // its device address
  cudaEvent_t sel_ev[4] = {};
  int sm_count = 148;
  cusolverDnHandle_t solver = nullptr;
  std::map<std::tuple<int, int, int, int, long long, long long, int>, cufftHandle> plans;
  std::map<std::vector<long long>, cufftHandle> plans_many;  // slab / pencil plans of the multi-rank build
  std::string err;
  int pivot = -1;
  double stage_ms[LRGW_NUM_STAGES] = {};
  cudaEvent_t ev[LRGW_NUM_STAGES + 1] = {};
  cudaEvent_t ev_quad[2] = {};  // around the K3 kernel (timing builds only)
  cudaEvent_t ev_lib[4] = {};   // around the cuSOLVER leaves of a timed build
  double lib_ms = 0.0;          // their sum
  bool quad_timed = false;
  bool timing = false;  // record stage events (lrgw_build only)
  long long launches0 = 0;
  int select_batch = 128;
  bool theta_implicit = false;  // lrgw_build keeps Theta factored as L L_P^-1 (see lrgw_eps_s)
  // Device-memory cache of this context: freed blocks are kept (by size) and
  // handed out again to later requests on the context's stream. A build
  // repeats the same sizes every call, so from the second call on no
  // allocation reaches the driver (cudaMallocAsync pools fragment under the
  // 0.1-1 GB blocks of a build and then grow or trim, stalling the host for
  // milliseconds).
  std::mutex mem_mu;
  std::multimap<size_t, void*> mem_free;
  std::unordered_map<void*, size_t> mem_live;
  size_t mem_cached = 0;
  // Factored-inverse handles created on this context: destroying the context
  // frees their device buffers and orphans them (lrgw_eps_destroy then only
  // deletes the handle), so handles may outlive their context safely.
  std::set<struct lrgw_eps_s*> live_eps;
};

struct lrgw_eps_s {
  lrgw_ctx ctx = nullptr;
  int n_r = 0, n_mu = 0;
  int dims[3] = {0, 0, 0};
  double cell[3] = {0, 0, 0};
  int zero = 0;
  double* theta = nullptr;
  double* k = nullptr;
  double* t = nullptr;
  double* pvp = nullptr;  // Theta^T V Theta (lrgw_build only)
  std::vector<int32_t> pts;
  // build diagnostics (lrgw_build only; lrgw_eps_info)
  double min_margin = -1.0;
  int min_margin_step = -1;
  int fit_path = -1;
  double lp_diag_ratio = 0.0;
  int select_blocks = 0;
  // row panel of a multi-rank build (lrgw_build_sharded): theta holds grid
  // rows [row0, row0 + rows); rows == 0 means all n_r rows (one GPU)
  int row0 = 0, rows = 0;
  // implicit-Theta handle (lrgw_ctx_set_theta_implicit): theta holds the
  // selection factor L (pivot order) and k, t, pvp the pivot-order K' =
  // L_P^-1 K L_P^-T, T and L^T V L, so Theta K Theta^T = L K' L^T; lp / lpinv
  // keep L_P and L_P^-1, colmap the pivot -> sorted-point column map.
  // eps_explicit() turns it into the ordinary handle on first demand.
  bool implicit = false;
  double* lp = nullptr;
  double* lpinv = nullptr;
  std::vector<int> colmap;
};

namespace lrgw_impl {

void* ctx_alloc(lrgw_ctx c, size_t bytes);
void ctx_free(lrgw_ctx c, void* p);

// Device buffer from the context cache (returned on scope exit).
struct DBuf {
  lrgw_ctx ctx = nullptr;
  void* p = nullptr;
  size_t bytes = 0;
  DBuf() = default;
  DBuf(lrgw_ctx c, size_t b) : ctx(c), bytes(b) {
    if (b) p = ctx_alloc(c, b);
  }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : ctx(o.ctx), p(o.p), bytes(o.bytes) { o.p = nullptr; }
  DBuf& operator=(DBuf&& o) noexcept {
    release();
    ctx = o.ctx;
    p = o.p;
    bytes = o.bytes;
    o.p = nullptr;
    return *this;
  }
  ~DBuf() { release(); }
  void release() {
    if (p) ctx_free(ctx, p);
    p = nullptr;
  }
  double* d() const { return static_cast<double*>(p); }
  int* i() const { return static_cast<int*>(p); }
  void* take() {
    void* q = p;
    p = nullptr;
    return q;
  }
};

inline DBuf dalloc(lrgw_ctx c, size_t n) { return DBuf(c, n * sizeof(double)); }
inline DBuf ialloc(lrgw_ctx c, size_t n) { return DBuf(c, n * sizeof(int)); }

DBuf upload(lrgw_ctx c, const double* h, size_t n);
DBuf upload_i(lrgw_ctx c, const int32_t* h, size_t n);
void download(lrgw_ctx c, void* h, const void* d, size_t bytes);
void use_device(lrgw_ctx c);
lrgw_eps_s* new_eps(lrgw_ctx c);
void mark(lrgw_ctx c, int i);

// The ABI wrapper: run the body, map failures onto status codes.
template <class F>
int guarded(lrgw_ctx c, F&& f) {
  if (!c) return LRGW_ERR_INVALID_INPUT;
  try {
    use_device(c);
    c->pivot = -1;
    f();
    return LRGW_OK;
  } catch (const Fail& e) {
    c->err = e.msg;
    if (e.code == LRGW_ERR_SINGULAR) c->pivot = e.pivot;
    return e.code;
  } catch (const std::bad_alloc&) {
    c->err = "host allocation failure";
    return LRGW_ERR_INTERNAL;
  } catch (...) {
    c->err = "unknown failure";
    return LRGW_ERR_INTERNAL;
  }
}

template <class F>
int guarded_host(F&& f) {
  try {
    f();
    return LRGW_OK;
  } catch (const Fail& e) {
    return e.code;
  } catch (...) {
    return LRGW_ERR_INTERNAL;
  }
}

// Split-K scratch for the skinny / symmetric GEMMs.
struct Work {
  DBuf buf;
  size_t elems = 0;
};
Work make_work(lrgw_ctx c, size_t elems);
void gemm(lrgw_ctx c, int M, int N, int K, const double* A, long long lda, Lay la, const double* B,
          long long ldb, Lay lb, double* C, long long ldc, double alpha, double beta,
          const double* scale = nullptr, bool lower = false, Work* w = nullptr);

void check_grid(const int* dims, const double* cell);
long long half_len(const int* dims);
void fft_forward(lrgw_ctx c, const int* dims, const double* x, long long ldx, int m, double* xhat);
void fft_inverse(lrgw_ctx c, const int* dims, double* xhat, int m, double* y, long long ldy);
void coulomb_apply(lrgw_ctx c, const int* dims, const double* cell, int zero, const double* x, long long ldx, int m,
                   double* y, long long ldy);
void pvp_impl(lrgw_ctx c, const int* dims, const double* cell, int zero, const double* theta, long long ldt,
              int n_mu, double* pvp);
void smw_core(lrgw_ctx c, const double* t, const double* pvp, int n, double* k);
// An implicit-Theta handle made explicit in place (no-op otherwise).
void eps_explicit(lrgw_ctx c, lrgw_eps_s* e);
void trtri_lower(lrgw_ctx c, double* a, int n);
double dev_max_abs(lrgw_ctx c, const double* x, size_t n);
void gram_inverse(lrgw_ctx c, const double* gram, int n, double* ginv);

// Validated inputs of a build (lrgw_build / lrgw_build_sharded).
struct BuildSetup {
  int n_mu = 0;
  lrgw_host::Spec spec;
};
BuildSetup validate_build(lrgw_ctx c, const lrgw_build_params* prm, const double* phi_v, long long ldv,
                          const double* phi_c, long long ldc, const double* energies, int panel_rows);
void timing_begin(lrgw_ctx c);
void timing_end(lrgw_ctx c);
lrgw_eps_s* build_one(lrgw_ctx c, const lrgw_build_params& P, const BuildSetup& bs, const double* phi_v,
                      long long ldv, const double* phi_c, long long ldc, const double* energies);
void eps_apply_impl(lrgw_ctx c, lrgw_eps e, const double* x, long long ldx, int m, double* y, long long ldy);
bool eps_is_panel(const lrgw_eps_s* e);

// Stage 1 (select.cu): host mirror of the candidate entry (d, position, grid row).
struct HostEnt {
  double v;
  int pos, row;
};
bool fused_downdate_enabled();
// the selection's per-block read of the greedy's accepted count (capi.cu)
int* select_flag_arm(lrgw_ctx c);
int select_wait_b(lrgw_ctx c, const int* b_dev);
struct SelectKeep {
  DBuf L;
  std::vector<int> order;
  int steps = 0;
  int blocks = 0;           // candidate blocks (one host sync each)
  int min_margin_step = -1; // step of the smallest top-2 margin (when margins are requested)
  size_t min_l_elems = 0;   // allocate L at least this large (cache block reuse; see select_impl)
};
std::vector<int32_t> select_impl(lrgw_ctx c, const double* a, long long lda, int n1, const double* b, long long ldb,
                                 int n2, int n_r, int n_mu, double* min_margin, SelectKeep* keep = nullptr);

// Stage 3 (quadrature.cu)
struct NodeSet {
  std::vector<double> nodes, weights;
};
NodeSet trapezoid(const lrgw_host::Spec& s, int n_intervals);
void quad_run(lrgw_ctx c, const double* pv, long long ldv, const double* pc, long long ldpc, int n_mu, int n_v,
              int n_c, const std::vector<double>& dv, const std::vector<double>& dc, const std::vector<double>& gw,
              int n_nodes, double* running, double beta, double pref, double* out, long long ldo);
void node_tables_or_fail(const lrgw_host::Spec& s, const double* e, int n_v, int n_c, const NodeSet& ns,
                         std::vector<double>* dv, std::vector<double>* dc, std::vector<double>* gw);
void direct_impl(lrgw_ctx c, const double* pv, long long ldv, const double* pc, long long ldpc, int n_mu, int n_v,
                 int n_c, const double* e, double* t, long long ldt);
// Adaptive levels to delta_rel (contour.hpp:298-329) into t (n_mu^2).
void adaptive_impl(lrgw_ctx c, const double* pv, long long ldv, const double* pc, long long ldpc, int n_mu, int n_v,
                   int n_c, const double* e, const lrgw_host::Spec& spec, double* t);

}  // namespace lrgw_impl
