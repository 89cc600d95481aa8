// sharded.cu — the multi-rank eps^-1 build behind the C-ABI:
// one process per GPU, a communicator (NCCL over NVLink, or a host
// transport supplied by the caller) and z-plane row panels of the grid.
//
// The exchange scheme (the same as the Python design in dist.py, which the
// CPU tests run with a numpy backend):
//   stage 1  per candidate block: local top-(s+1) (select_topk on the panel)
//            -> all-gather -> device merge (pivot order: residual desc,
//            position asc); the candidates' rows [Phi_v | Phi_c | L[:, :k]]
//            owner-contributed (zero elsewhere) -> one all-reduce; W[C, C]
//            and the certified greedy replicated (bit-identical on every
//            rank: same kernel, same inputs, replicated position arrays);
//            W columns of the accepted pivots, L block and residual downdate
//            on the local panel only. One host sync per block (its size).
//   stage 2  L_P owner-contributed -> all-reduce; Theta panel = L_p L_P^-1.
//   stage 3  the trapezoid's nodes split across ranks -> all-reduce.
//   stage 4-5  2-D D2Z of each owned plane, all-to-all of y-chunks, 1-D FFT
//            along z, G-slab SYRK with the Hermitian v(G) weights ->
//            all-reduce; SMW core replicated.
#include <dlfcn.h>
#include <nccl.h>  // types only: every NCCL entry point is resolved with dlsym

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "internal.h"
#include "select.h"
#include "shard.h"

using namespace lrgw_impl;

// ---------------------------------------------------------------------------
// NCCL, loaded at run time (libnccl.so.2: the process's own when one is
// already mapped, e.g. torch's, else the system library)
// ---------------------------------------------------------------------------
namespace {

struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

template <class F>
void sym(void* h, const char* name, F*& f, bool& ok) {
  f = reinterpret_cast<F*>(dlsym(h, name));
  if (!f) ok = false;
}

const NcclApi& nccl() {
  static const NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.why = std::string("dlopen(libnccl.so.2): ") + dlerror();
      return a;
    }
    bool ok = true;
    sym(h, "ncclGetUniqueId", a.GetUniqueId, ok);
    sym(h, "ncclCommInitRank", a.CommInitRank, ok);
    sym(h, "ncclCommDestroy", a.CommDestroy, ok);
    sym(h, "ncclAllReduce", a.AllReduce, ok);
    sym(h, "ncclAllGather", a.AllGather, ok);
    sym(h, "ncclSend", a.Send, ok);
    sym(h, "ncclRecv", a.Recv, ok);
    sym(h, "ncclGroupStart", a.GroupStart, ok);
    sym(h, "ncclGroupEnd", a.GroupEnd, ok);
    sym(h, "ncclGetErrorString", a.GetErrorString, ok);
    a.ok = ok;
    if (!ok) a.why = "libnccl.so.2 lacks an entry point";
    return a;
  }();
  return api;
}

void ckn(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    fail(LRGW_ERR_CUDA, std::string(what) + ": " + (nccl().GetErrorString ? nccl().GetErrorString(r) : "nccl error"));
}

}  // namespace

struct lrgw_comm_s {
  int rank = 0, world = 1;
  bool is_nccl = false;
  ncclComm_t nccl = nullptr;
  lrgw_host_transport host{};
  // pinned staging of the host transport
  char* pin = nullptr;
  size_t pin_bytes = 0;
  ~lrgw_comm_s() {
    if (nccl && nccl_api_ok()) ::nccl().CommDestroy(nccl);
    if (pin) cudaFreeHost(pin);
  }
  static bool nccl_api_ok() { return ::nccl().ok; }
  char* staging(size_t bytes) {
    if (bytes > pin_bytes) {
      if (pin) cudaFreeHost(pin);
      pin = nullptr;
      pin_bytes = 0;
      ck(cudaMallocHost(&pin, bytes), "cudaMallocHost(staging)");
      pin_bytes = bytes;
    }
    return pin;
  }
};

namespace {

// ---- collectives on device buffers, ordered on the context stream -----------
void allreduce(lrgw_ctx c, lrgw_comm m, double* buf, size_t n) {
  if (m->world == 1 || n == 0) return;
  if (m->is_nccl) {
    ckn(nccl().AllReduce(buf, buf, n, ncclFloat64, ncclSum, m->nccl, c->stream), "ncclAllReduce");
    return;
  }
  char* h = m->staging(n * sizeof(double));
  ck(cudaMemcpyAsync(h, buf, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream), "D2H");
  ck(cudaStreamSynchronize(c->stream), "sync");
  if (m->host.allreduce_sum_f64(m->host.user, reinterpret_cast<double*>(h), (long long)n) != 0)
    fail(LRGW_ERR_CUDA, "host transport: allreduce failed");
  ck(cudaMemcpyAsync(buf, h, n * sizeof(double), cudaMemcpyHostToDevice, c->stream), "H2D");
}

void allgather(lrgw_ctx c, lrgw_comm m, const void* send, void* recv, size_t bytes) {
  if (m->world == 1) {
    ck(cudaMemcpyAsync(recv, send, bytes, cudaMemcpyDeviceToDevice, c->stream), "D2D");
    return;
  }
  if (m->is_nccl) {
    ckn(nccl().AllGather(send, recv, bytes, ncclUint8, m->nccl, c->stream), "ncclAllGather");
    return;
  }
  char* h = m->staging(bytes * (m->world + 1));
  ck(cudaMemcpyAsync(h, send, bytes, cudaMemcpyDeviceToHost, c->stream), "D2H");
  ck(cudaStreamSynchronize(c->stream), "sync");
  if (m->host.allgather(m->host.user, h, h + bytes, (long long)bytes) != 0)
    fail(LRGW_ERR_CUDA, "host transport: allgather failed");
  ck(cudaMemcpyAsync(recv, h + bytes, bytes * m->world, cudaMemcpyHostToDevice, c->stream), "H2D");
}

// counts / displacements in doubles
void alltoallv(lrgw_ctx c, lrgw_comm m, const double* send, const std::vector<size_t>& sc,
               const std::vector<size_t>& sd, double* recv, const std::vector<size_t>& rc,
               const std::vector<size_t>& rd) {
  const int w = m->world;
  if (m->is_nccl) {
    ckn(nccl().GroupStart(), "ncclGroupStart");
    for (int q = 0; q < w; ++q) {
      if (sc[q]) ckn(nccl().Send(send + sd[q], sc[q], ncclFloat64, q, m->nccl, c->stream), "ncclSend");
      if (rc[q]) ckn(nccl().Recv(recv + rd[q], rc[q], ncclFloat64, q, m->nccl, c->stream), "ncclRecv");
    }
    ckn(nccl().GroupEnd(), "ncclGroupEnd");
    return;
  }
  size_t st = 0, rt = 0;
  for (int q = 0; q < w; ++q) {
    st += sc[q];
    rt += rc[q];
  }
  char* h = m->staging((st + rt) * sizeof(double));
  double* hs = reinterpret_cast<double*>(h);
  double* hr = hs + st;
  ck(cudaMemcpyAsync(hs, send, st * sizeof(double), cudaMemcpyDeviceToHost, c->stream), "D2H");
  ck(cudaStreamSynchronize(c->stream), "sync");
  std::vector<long long> sb(w), rb(w);
  for (int q = 0; q < w; ++q) {
    sb[q] = (long long)(sc[q] * sizeof(double));
    rb[q] = (long long)(rc[q] * sizeof(double));
  }
  if (m->host.alltoallv(m->host.user, hs, sb.data(), hr, rb.data()) != 0)
    fail(LRGW_ERR_CUDA, "host transport: alltoallv failed");
  ck(cudaMemcpyAsync(recv, hr, rt * sizeof(double), cudaMemcpyHostToDevice, c->stream), "H2D");
}

// ---- partitioning -------------------------------------------------------------
void z_panel(const int* dims, int world, int rank, int* row0, int* rows) {
  const long long plane = (long long)dims[0] * dims[1];
  const int z0 = (int)((long long)dims[2] * rank / world), z1 = (int)((long long)dims[2] * (rank + 1) / world);
  *row0 = (int)(z0 * plane);
  *rows = (int)((z1 - z0) * plane);
}

struct Panels {
  std::vector<int> row0, rows;
  int max_rows = 0;
};

Panels panels(const int* dims, int world) {
  Panels p;
  p.row0.resize(world);
  p.rows.resize(world);
  for (int q = 0; q < world; ++q) {
    z_panel(dims, world, q, &p.row0[q], &p.rows[q]);
    p.max_rows = std::max(p.max_rows, p.rows[q]);
  }
  return p;
}

// ---- stage 1 --------------------------------------------------------------------
struct PanelSelect {
  DBuf L;                    // rows x steps, pivot order
  std::vector<int> order;    // pivot sequence (global grid rows)
  std::vector<int32_t> pts;  // first n_mu pivots, sorted
  int steps = 0, blocks = 0, min_step = -1;
  double min_margin = 1.0;
};

PanelSelect select_panel(lrgw_ctx c, lrgw_comm m, const Panels& pn, const double* a, long long lda, int n1,
                         const double* b, long long ldb, int n2, int n_r, int n_mu) {
  const int row0 = pn.row0[m->rank], rows = pn.rows[m->rank], world = m->world;
  const int steps = (int)std::min<long long>(n_mu, std::min<long long>((long long)n1 * n2, n_r));
  const int s = std::max(1, std::min({c->select_batch, select_max_candidates(), n_r}));
  const int lds = s + (s & 1);
  if (select_ent_bytes() != shard_ent_bytes() || select_ent_bytes() != sizeof(HostEnt))
    fail(LRGW_ERR_INTERNAL, "select: entry layout mismatch");
  PanelSelect ps;
  ps.steps = steps;
  DBuf d = dalloc(c, rows), pos = ialloc(c, n_r), perm = ialloc(c, n_r), scratch = ialloc(c, 2 * (size_t)rows);
  ck(select_init(c->stream, a, lda, n1, b, ldb, n2, rows, d.d(), scratch.i(), scratch.i() + rows), "select_init");
  ck(shard_iota(c->stream, pos.i(), n_r), "iota");  // positions / permutation: replicated, global
  ck(shard_iota(c->stream, perm.i(), n_r), "iota");
  ps.L = dalloc(c, (size_t)rows * std::max(steps, 1));
  const int wmax = n1 + n2 + steps;
  DBuf rowbuf = dalloc(c, (size_t)lds * wmax), pick = dalloc(c, (size_t)lds * wmax);
  DBuf wcc = dalloc(c, (size_t)s * s), xcol = dalloc(c, (size_t)s * s);
  DBuf wsel, xperm;  // the three-launch fallback's W columns / the TMA panel's permuted X (allocated on use)
  const size_t eb = select_ent_bytes();
  DBuf top_loc(c, eb * (s + 1)), gathered(c, eb * (s + 1) * world), top(c, eb * (s + 1));
  DBuf tmp(c, select_topk_tmp_bytes(rows, s + 1));
  DBuf cand = ialloc(c, s), order = ialloc(c, std::max(steps, 1)), margin = dalloc(c, std::max(steps, 1));
  DBuf bout = ialloc(c, 4);
  DBuf dr0 = upload_i(c, pn.row0.data(), world);
  Work w = make_work(c, (size_t)8 * s * s);
  ck(select_topk_reset(c->stream, tmp.p), "select_topk_reset");
  double* amu = rowbuf.d();
  double* bmu = amu + (size_t)lds * n1;
  double* lrow = bmu + (size_t)lds * n2;
  int k = 0;
  while (k < steps) {
    const int se = std::min(s, n_r - k);
    ck(select_topk(c->stream, d.d(), pos.i() + row0, rows, k, se + 1, tmp.p, top_loc.p), "select_topk");
    allgather(c, m, top_loc.p, gathered.p, eb * (se + 1));
    ck(shard_merge_top(c->stream, gathered.p, world, se + 1, dr0.i(), top.p), "merge_top");
    ck(select_cand_rows(c->stream, top.p, se, cand.i()), "cand_rows");
    ck(shard_gather_owned(c->stream, a, lda, n1, b, ldb, n2, ps.L.d(), rows, k, cand.i(), se, row0, rows, amu, lds),
       "gather_owned");
    allreduce(c, m, rowbuf.d(), (size_t)lds * (n1 + n2 + k));
    // the candidates' Schur block, replicated
    ck(hadamard_gemm(c->stream, se, se, amu, lds, amu, lds, n1, bmu, lds, bmu, lds, n2, wcc.d(), se, 1.0, 0.0),
       "hadamard_gemm(W_CC)");
    if (k > 0) gemm(c, se, se, k, lrow, lds, Lay::MN, lrow, lds, Lay::MN, wcc.d(), se, -1.0, 1.0, nullptr, false, &w);
    const bool use_panel = fused_downdate_enabled() && select_panel_enabled(n1, n2);
    const bool use_p4 = use_panel && select_panel_tma_enabled();
    if (use_p4 && !xperm.p) xperm = dalloc(c, (size_t)s * s);
    ck(select_cand_greedy(c->stream, n_r, se, steps, k, top.p, wcc.d(), pos.i(), perm.i(), xcol.d(), order.i(),
                          margin.d(), bout.i(), select_accept_cap(se, n_r, use_p4), select_accept_round(), nullptr,
                          nullptr, use_p4 ? xperm.d() : nullptr, select_flag_arm(c)),
       "cand_greedy");
    const int nb = select_wait_b(c, bout.i());  // the one host wait per block
    if (nb <= 0) fail(LRGW_ERR_INTERNAL, "select: no progress (non-finite residuals?)");
    // the accepted pivots' rows (they are candidates: already exchanged)
    const int ldp = nb + (nb & 1);
    ck(shard_pick_rows(c->stream, top.p, se, order.i() + k, nb, rowbuf.d(), lds, n1 + n2 + k, pick.d(), ldp),
       "pick_rows");
    const double* asel = pick.d();
    const double* bsel = asel + (size_t)ldp * n1;
    const double* lsel = bsel + (size_t)ldp * n2;
    double* lblk = ps.L.d() + (size_t)k * rows;
    // the fused panel (panel4.cu / panel.cu) on this rank's rows, as in the one-GPU loop
    cudaError_t pe = cudaErrorNotSupported;
    if (use_p4)
      pe = select_panel_tma(c->stream, rows, nb, a, lda, asel, ldp, n1, b, ldb, bsel, ldp, n2, ps.L.d(), rows, lsel,
                            ldp, k, xperm.d(), se, lblk, rows, d.d(), pos.i() + row0, k + nb);
    if (pe == cudaErrorNotSupported && use_panel) {
      cudaGetLastError();
      pe = lrgw_dev::select_panel(c->stream, rows, nb, a, lda, asel, ldp, n1, b, ldb, bsel, ldp, n2, ps.L.d(), rows,
                                  lsel, ldp, k, xcol.d(), se, lblk, rows, d.d(), pos.i() + row0, k + nb);
    }
    if (pe != cudaErrorNotSupported) {
      ck(pe, "select_panel");
      k += nb;
      ++ps.blocks;
      continue;
    }
    cudaGetLastError();
    if (!wsel.p) wsel = dalloc(c, (size_t)rows * s);
    ck(hadamard_gemm(c->stream, rows, nb, a, lda, asel, ldp, n1, b, ldb, bsel, ldp, n2, wsel.d(), rows, 1.0, 0.0),
       "hadamard_gemm");
    if (k > 0) gemm(c, rows, nb, k, ps.L.d(), rows, Lay::MN, lsel, ldp, Lay::MN, wsel.d(), rows, -1.0, 1.0);
    cudaError_t fe = fused_downdate_enabled() ? dgemm_tall_downdate(c->stream, rows, nb, nb, wsel.d(), rows, xcol.d(),
                                                                    se, lblk, rows, d.d(), pos.i() + row0, k + nb)
                                              : cudaErrorNotSupported;
    if (fe == cudaErrorNotSupported) {
      cudaGetLastError();
      gemm(c, rows, nb, nb, wsel.d(), rows, Lay::MN, xcol.d(), se, Lay::MN, lblk, rows, 1.0, 0.0);
      ck(select_downdate(c->stream, ps.L.d(), rows, k, nb, pos.i() + row0, d.d()), "downdate");
    } else {
      ck(fe, "dgemm_tall_downdate");
    }
    k += nb;
    ++ps.blocks;
  }
  ps.order.resize(steps);
  download(c, ps.order.data(), order.p, sizeof(int) * steps);
  std::vector<double> mg(std::max(steps, 1));
  download(c, mg.data(), margin.p, sizeof(double) * std::max(steps, 1));
  for (int i = 0; i < steps; ++i)
    if (mg[i] < ps.min_margin) {
      ps.min_margin = mg[i];
      ps.min_step = i;
    }
  ps.pts.resize(n_mu);
  download(c, ps.pts.data(), perm.p, sizeof(int) * n_mu);
  std::sort(ps.pts.begin(), ps.pts.end());
  return ps;
}

// ---- stage 2 --------------------------------------------------------------------
// Theta panel = L_p L_P^-1 (capi.cu fused_fit with the pivot rows of the
// factor owner-contributed). false: L_P has a pivot below the LU threshold.
bool fit_panel_fused(lrgw_ctx c, lrgw_comm m, const PanelSelect& ps, int row0, int rows, int n_mu, double* theta,
                     double* diag_ratio) {
  if (ps.steps != n_mu) return false;
  DBuf dorder = upload_i(c, ps.order.data(), n_mu);
  DBuf lp = dalloc(c, (size_t)n_mu * n_mu);
  ck(shard_gather_owned(c->stream, nullptr, 0, 0, nullptr, 0, 0, ps.L.d(), rows, n_mu, dorder.i(), n_mu, row0, rows,
                        lp.d(), n_mu),
     "gather_owned(L_P)");
  allreduce(c, m, lp.d(), (size_t)n_mu * n_mu);
  ck(zero_strict_upper(c->stream, lp.d(), n_mu, n_mu), "zero_upper");
  std::vector<double> diag(n_mu);
  ck(cudaMemcpy2DAsync(diag.data(), sizeof(double), lp.d(), (size_t)(n_mu + 1) * sizeof(double), sizeof(double), n_mu,
                       cudaMemcpyDeviceToHost, c->stream),
     "D2H diag");
  ck(cudaStreamSynchronize(c->stream), "sync");
  double gmax = 0.0, dmin = HUGE_VAL, dmax = 0.0;
  for (double v : diag) {
    gmax = std::max(gmax, v * v);
    dmin = std::min(dmin, std::abs(v));
    dmax = std::max(dmax, std::abs(v));
  }
  *diag_ratio = dmin > 0.0 ? (dmax / dmin) * (dmax / dmin) : HUGE_VAL;
  const double tiny = 1e-14 * (gmax > 0.0 ? gmax : 1.0);
  for (double v : diag)
    if (!(v * v >= tiny)) return false;
  {
    DBuf work = dalloc(c, trtri_work_elems(n_mu));
    DBuf bad = ialloc(c, 1);
    const int big = 0x7fffffff;
    ck(cudaMemcpyAsync(bad.p, &big, sizeof(int), cudaMemcpyHostToDevice, c->stream), "H2D");
    ck(lrgw_dev::trtri_lower(c->stream, lp.d(), n_mu, n_mu, work.d(), bad.i(), c->sm_count), "trtri");
    int h = 0;
    download(c, &h, bad.p, sizeof(int));
    if (h != big) return false;
  }
  mark(c, 3);
  std::vector<int> colmap(n_mu);
  for (int q = 0; q < n_mu; ++q)
    colmap[q] = (int)(std::lower_bound(ps.pts.begin(), ps.pts.end(), ps.order[q]) - ps.pts.begin());
  DBuf dmap = upload_i(c, colmap.data(), n_mu);
  DBuf xt = dalloc(c, (size_t)n_mu * n_mu);
  ck(transpose(c->stream, lp.d(), n_mu, n_mu, n_mu, xt.d(), n_mu), "transpose");
  ck(dgemm(c->stream, rows, n_mu, n_mu, ps.L.d(), rows, Lay::MN, xt.d(), n_mu, Lay::MN, theta, rows, 1.0, 0.0, nullptr,
           false, c->sm_count, nullptr, 0, true, dmap.i()),
     "dgemm(theta)");
  return true;
}

// Explicit fit of the panel (isdf.hpp:132-161): point rows replicated, the
// Gram inverted with the reference's LU rule / pseudo-inverse fallback.
void fit_panel_explicit(lrgw_ctx c, const double* pmu, int n_mu, int n1, int n2, const double* a, long long lda,
                        const double* b, long long ldb, int rows, double* theta) {
  const double* amu = pmu;
  const double* bmu = pmu + (size_t)n_mu * n1;
  DBuf gram = dalloc(c, (size_t)n_mu * n_mu), ginv = dalloc(c, (size_t)n_mu * n_mu);
  ck(hadamard_gemm(c->stream, n_mu, n_mu, amu, n_mu, amu, n_mu, n1, bmu, n_mu, bmu, n_mu, n2, gram.d(), n_mu, 1.0,
                   0.0),
     "hadamard_gemm(gram)");
  ck(mirror_lower(c->stream, gram.d(), n_mu, n_mu, true), "symmetrize");
  mark(c, 2);
  gram_inverse(c, gram.d(), n_mu, ginv.d());
  mark(c, 3);
  DBuf lhs = dalloc(c, (size_t)rows * n_mu);
  ck(hadamard_gemm(c->stream, rows, n_mu, a, lda, amu, n_mu, n1, b, ldb, bmu, n_mu, n2, lhs.d(), rows, 1.0, 0.0),
     "hadamard_gemm(lhs)");
  gemm(c, rows, n_mu, n_mu, lhs.d(), rows, Lay::MN, ginv.d(), n_mu, Lay::MN, theta, rows, 1.0, 0.0);
}

// ---- stage 4-5a -----------------------------------------------------------------
cufftHandle plan_many(lrgw_ctx c, int rank, const long long* n, const long long* inembed, long long idist,
                      const long long* onembed, long long odist, cufftType type, long long batch) {
  std::vector<long long> key = {rank, (long long)type, idist, odist, batch};
  for (int i = 0; i < rank; ++i) {
    key.push_back(n[i]);
    key.push_back(inembed[i]);
    key.push_back(onembed[i]);
  }
  auto it = c->plans_many.find(key);
  if (it != c->plans_many.end()) return it->second;
  cufftHandle plan;
  size_t work = 0;
  ckf(cufftCreate(&plan), "cufftCreate");
  ckf(cufftMakePlanMany64(plan, rank, const_cast<long long*>(n), const_cast<long long*>(inembed), 1, idist,
                          const_cast<long long*>(onembed), 1, odist, type, batch, &work),
      "cufftMakePlanMany64");
  ckf(cufftSetStream(plan, c->stream), "cufftSetStream");
  c->plans_many[key] = plan;
  return plan;
}

constexpr int kColsPerFft = 1024;

// Partial Theta_p^T V Theta_p over this rank's G-slab (lower tiles, mirrored);
// the caller all-reduces. theta: the panel (rows x n_mu, ld rows).
void pvp_panel(lrgw_ctx c, lrgw_comm m, const Panels& pn, const int* dims, const double* cell, int zero,
               const double* theta, int n_mu, double* pvp) {
  const int n1 = dims[0], n2 = dims[1], n3 = dims[2], n1h = n1 / 2 + 1, world = m->world, me = m->rank;
  const long long plane = (long long)n1 * n2;
  const int rows = pn.rows[me], zl = (int)(rows / plane);
  std::vector<int> ya(world), ny(world), z0(world), zls(world);
  for (int q = 0; q < world; ++q) {
    ya[q] = (int)((long long)n2 * q / world);
    ny[q] = (int)((long long)n2 * (q + 1) / world) - ya[q];
    z0[q] = (int)(pn.row0[q] / plane);
    zls[q] = (int)(pn.rows[q] / plane);
  }
  // A: 2-D D2Z of every owned plane of every column -> (n_mu, zl, n2, n1h)
  const long long cpl = (long long)n2 * n1h;  // complex entries per plane
  DBuf xa = dalloc(c, (size_t)2 * n_mu * zl * cpl);
  {
    const long long n[2] = {n2, n1}, in[2] = {n2, n1}, on[2] = {n2, n1h};
    for (int j0 = 0; j0 < n_mu; j0 += kColsPerFft) {
      const int nc = std::min(kColsPerFft, n_mu - j0);
      cufftHandle p = plan_many(c, 2, n, in, plane, on, cpl, CUFFT_D2Z, (long long)zl * nc);
      ckf(cufftExecD2Z(p, const_cast<double*>(theta) + (size_t)j0 * rows,
                       reinterpret_cast<cufftDoubleComplex*>(xa.d() + (size_t)2 * j0 * zl * cpl)),
          "cufftExecD2Z(planes)");
    }
  }
  // B: y-chunks to their owners (one all-to-all)
  std::vector<size_t> sc(world), sd(world), rc(world), rd(world);
  size_t st = 0, rt = 0;
  for (int q = 0; q < world; ++q) {
    sc[q] = (size_t)2 * n_mu * zl * ny[q] * n1h;
    sd[q] = st;
    st += sc[q];
    rc[q] = (size_t)2 * n_mu * zls[q] * ny[me] * n1h;
    rd[q] = rt;
    rt += rc[q];
  }
  DBuf sendb = dalloc(c, st), recvb = dalloc(c, rt);
  for (int q = 0; q < world; ++q)
    ck(shard_slab_pack(c->stream, xa.d(), n_mu, zl, n2, n1h, ya[q], ny[q], sendb.d() + sd[q]), "slab_pack");
  xa.release();
  alltoallv(c, m, sendb.d(), sc, sd, recvb.d(), rc, rd);
  sendb.release();
  // C: z-pencils (n_mu, ny, n1h, n3), then D: 1-D FFT along z
  const long long kc = (long long)ny[me] * n1h * n3;  // complex G-points of this slab
  if (kc == 0) {
    ck(fill(c->stream, pvp, (size_t)n_mu * n_mu, 0.0), "fill");
    mark(c, 6);
    return;
  }
  DBuf pen = dalloc(c, (size_t)2 * n_mu * kc);
  for (int q = 0; q < world; ++q)
    ck(shard_slab_unpack(c->stream, recvb.d() + rd[q], n_mu, zls[q], ny[me], n1h, z0[q], n3, pen.d()),
       "slab_unpack");
  recvb.release();
  {
    const long long n[1] = {n3}, in[1] = {n3}, on[1] = {n3};
    const long long lines = (long long)ny[me] * n1h;
    for (int j0 = 0; j0 < n_mu; j0 += kColsPerFft) {
      const int nc = std::min(kColsPerFft, n_mu - j0);
      cufftHandle p = plan_many(c, 1, n, in, n3, on, n3, CUFFT_Z2Z, lines * nc);
      auto* ptr = reinterpret_cast<cufftDoubleComplex*>(pen.d() + (size_t)2 * j0 * kc);
      ckf(cufftExecZ2Z(p, ptr, ptr, CUFFT_FORWARD), "cufftExecZ2Z(z)");
    }
  }
  mark(c, 6);
  // E: the G-slab SYRK with w_G v(G) / N_r as the k-scale
  DBuf wts = dalloc(c, (size_t)2 * kc);
  ck(coulomb_slab_weights(c->stream, n1, n2, n3, cell[0], cell[1], cell[2], zero, ya[me], ny[me], wts.d()),
     "slab_weights");
  Work w = make_work(c, (size_t)16 * n_mu * n_mu);
  gemm(c, n_mu, n_mu, (int)(2 * kc), pen.d(), 2 * kc, Lay::K, pen.d(), 2 * kc, Lay::K, pvp, n_mu, 1.0, 0.0, wts.d(),
       true, &w);
  ck(mirror_lower(c->stream, pvp, n_mu, n_mu, false), "mirror");
}

// ---- the build ------------------------------------------------------------------
lrgw_eps_s* build_panel(lrgw_ctx c, lrgw_comm m, const lrgw_build_params& P, const BuildSetup& bs,
                        const double* phi_v, long long ldv, const double* phi_c, long long ldc,
                        const double* energies) {
  const int n_r = P.n_r, n_v = P.n_v, n_c = P.n_c, n_mu = bs.n_mu;
  const Panels pn = panels(P.dims, m->world);
  const int row0 = pn.row0[m->rank], rows = pn.rows[m->rank];
  const size_t nn = (size_t)n_mu * n_mu;
  struct TimingGuard {
    lrgw_ctx c;
    ~TimingGuard() { c->timing = false; }
  } tg{c};
  timing_begin(c);
  // stage 1
  PanelSelect ps = select_panel(c, m, pn, phi_v, ldv, n_v, phi_c, ldc, n_c, n_r, n_mu);
  mark(c, 1);
  mark(c, 2);
  // point rows [Phi_v | Phi_c] at the sorted points, replicated (stage 3; explicit fit)
  DBuf dpts = upload_i(c, ps.pts.data(), n_mu);
  DBuf pmu = dalloc(c, (size_t)n_mu * (n_v + n_c));
  ck(shard_gather_owned(c->stream, phi_v, ldv, n_v, phi_c, ldc, n_c, nullptr, 0, 0, dpts.i(), n_mu, row0, rows,
                        pmu.d(), n_mu),
     "gather_owned(points)");
  allreduce(c, m, pmu.d(), (size_t)n_mu * (n_v + n_c));
  // stage 2
  DBuf theta = dalloc(c, (size_t)rows * n_mu);
  double lp_ratio = 0.0;
  const bool fused = fit_panel_fused(c, m, ps, row0, rows, n_mu, theta.d(), &lp_ratio);
  ps.L.release();
  if (!fused) fit_panel_explicit(c, pmu.d(), n_mu, n_v, n_c, phi_v, ldv, phi_c, ldc, rows, theta.d());
  mark(c, 4);
  // stage 3
  const double* pv = pmu.d();
  const double* pc = pmu.d() + (size_t)n_mu * n_v;
  DBuf t = dalloc(c, nn);
  const lrgw_host::Spec& spec = bs.spec;
  if (spec.bypass) {
    direct_impl(c, pv, n_mu, pc, n_mu, n_mu, n_v, n_c, energies, t.d(), n_mu);
  } else if (P.n_lambda > 0) {
    const NodeSet all = trapezoid(spec, P.n_lambda);
    const int n_nodes = (int)all.nodes.size();
    const int k0 = (int)((long long)n_nodes * m->rank / m->world), k1 = (int)((long long)n_nodes * (m->rank + 1) / m->world);
    NodeSet mine;
    for (int k = k0; k < k1; ++k) {
      mine.nodes.push_back(all.nodes[k]);
      mine.weights.push_back(all.weights[k]);
    }
    DBuf acc = dalloc(c, nn);
    if (k1 > k0) {
      std::vector<double> dv, dc, gw;
      node_tables_or_fail(spec, energies, n_v, n_c, mine, &dv, &dc, &gw);
      quad_run(c, pv, n_mu, pc, n_mu, n_mu, n_v, n_c, dv, dc, gw, k1 - k0, nullptr, 0.0, 1.0, acc.d(), n_mu);
    } else {
      ck(fill(c->stream, acc.d(), nn, 0.0), "fill");
    }
    allreduce(c, m, acc.d(), nn);
    ck(scale_copy(c->stream, acc.d(), t.d(), nn, lrgw_host::prefactor(spec)), "scale");
  } else {
    adaptive_impl(c, pv, n_mu, pc, n_mu, n_mu, n_v, n_c, energies, spec, t.d());
  }
  mark(c, 5);
  // stages 4-5
  DBuf pvp = dalloc(c, nn), k = dalloc(c, nn);
  pvp_panel(c, m, pn, P.dims, P.cell, P.zero_kernel, theta.d(), n_mu, pvp.d());
  allreduce(c, m, pvp.d(), nn);
  mark(c, 7);
  smw_core(c, t.d(), pvp.d(), n_mu, k.d());
  mark(c, 8);
  timing_end(c);
  auto* e = new_eps(c);
  e->n_r = n_r;
  e->n_mu = n_mu;
  std::memcpy(e->dims, P.dims, sizeof(e->dims));
  std::memcpy(e->cell, P.cell, sizeof(e->cell));
  e->zero = P.zero_kernel;
  e->theta = static_cast<double*>(theta.take());
  e->k = static_cast<double*>(k.take());
  e->t = static_cast<double*>(t.take());
  e->pvp = static_cast<double*>(pvp.take());
  e->pts = ps.pts;
  e->min_margin = ps.min_margin;
  e->min_margin_step = ps.min_step;
  e->fit_path = fused ? 0 : 1;
  e->lp_diag_ratio = lp_ratio;
  e->select_blocks = ps.blocks;
  e->row0 = row0;
  e->rows = rows;
  return e;
}

}  // namespace

// ===========================================================================
// C-ABI
// ===========================================================================
extern "C" {

int lrgw_nccl_available(void) { return nccl().ok ? 1 : 0; }

int lrgw_nccl_unique_id(unsigned char id[128]) {
  return guarded_host([&] {
    if (!id) fail(LRGW_ERR_INVALID_INPUT, "nccl_unique_id: null buffer");
    if (!nccl().ok) fail(LRGW_ERR_UNSUPPORTED, nccl().why);
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    ncclUniqueId u;
    ckn(nccl().GetUniqueId(&u), "ncclGetUniqueId");
    std::memcpy(id, &u, 128);
  });
}

int lrgw_comm_create_nccl(lrgw_ctx c, int rank, int world, const unsigned char id[128], lrgw_comm* out) {
  return guarded(c, [&] {
    if (!out || !id || world < 1 || rank < 0 || rank >= world) fail(LRGW_ERR_INVALID_INPUT, "comm_create_nccl: bad arguments");
    if (!nccl().ok) fail(LRGW_ERR_UNSUPPORTED, nccl().why);
    auto* m = new lrgw_comm_s;
    m->rank = rank;
    m->world = world;
    m->is_nccl = true;
    ncclUniqueId u;
    std::memcpy(&u, id, 128);
    const ncclResult_t r = nccl().CommInitRank(&m->nccl, world, u, rank);
    if (r != ncclSuccess) {
      delete m;
      ckn(r, "ncclCommInitRank");
    }
    *out = m;
  });
}

int lrgw_comm_create_host(int rank, int world, const lrgw_host_transport* t, lrgw_comm* out) {
  if (!out || world < 1 || rank < 0 || rank >= world) return LRGW_ERR_INVALID_INPUT;
  if (world > 1 && (!t || !t->allreduce_sum_f64 || !t->allgather || !t->alltoallv)) return LRGW_ERR_INVALID_INPUT;
  auto* m = new lrgw_comm_s;
  m->rank = rank;
  m->world = world;
  if (t) m->host = *t;
  *out = m;
  return LRGW_OK;
}

int lrgw_comm_destroy(lrgw_comm m) {
  delete m;
  return LRGW_OK;
}

int lrgw_comm_info(lrgw_comm m, int* rank, int* world) {
  if (!m) return LRGW_ERR_INVALID_INPUT;
  if (rank) *rank = m->rank;
  if (world) *world = m->world;
  return LRGW_OK;
}

int lrgw_z_panel(const int* dims, int world, int rank, int* row0, int* rows) {
  if (!dims || !row0 || !rows || world < 1 || rank < 0 || rank >= world || dims[2] < world)
    return LRGW_ERR_INVALID_INPUT;
  z_panel(dims, world, rank, row0, rows);
  return LRGW_OK;
}

int lrgw_build_sharded(lrgw_ctx c, lrgw_comm m, const lrgw_build_params* prm, const double* phi_v, long long ldv,
                       const double* phi_c, long long ldc, const double* energies, lrgw_eps* out) {
  return guarded(c, [&] {
    if (!m || !out || !prm) fail(LRGW_ERR_INVALID_INPUT, "build_sharded: null argument");
    check_grid(prm->dims, prm->cell);
    if (prm->dims[2] < m->world) fail(LRGW_ERR_INVALID_INPUT, "build_sharded: fewer z-planes than ranks");
    int row0 = 0, rows = 0;
    z_panel(prm->dims, m->world, m->rank, &row0, &rows);
    const BuildSetup bs = validate_build(c, prm, phi_v, ldv, phi_c, ldc, energies, rows);
    if (m->world == 1) {  // one rank: the one-GPU build (a single slab is the whole 3-D FFT)
      *out = build_one(c, *prm, bs, phi_v, ldv, phi_c, ldc, energies);
      return;
    }
    *out = build_panel(c, m, *prm, bs, phi_v, ldv, phi_c, ldc, energies);
  });
}

int lrgw_eps_apply_sharded(lrgw_ctx c, lrgw_comm m, lrgw_eps e, const double* x, long long ldx, int mc, double* y,
                           long long ldy) {
  return guarded(c, [&] {
    if (!m || !e || !e->ctx) fail(LRGW_ERR_INVALID_INPUT, "eps_apply_sharded: null handle");
    if (mc < 0) fail(LRGW_ERR_INVALID_INPUT, "eps_apply_sharded: negative column count");
    const Panels pn = panels(e->dims, m->world);
    const int me = m->rank, rows = pn.rows[me], row0 = pn.row0[me];
    const int erows = e->rows > 0 ? e->rows : e->n_r;
    if (erows != rows || (e->rows > 0 && e->row0 != row0))
      fail(LRGW_ERR_INVALID_INPUT, "eps_apply_sharded: handle panel does not match the communicator");
    if (ldx < rows || ldy < rows) fail(LRGW_ERR_INVALID_INPUT, "eps_apply_sharded: leading dimension below the panel");
    if (mc == 0) return;
    if (m->world == 1) {
      eps_apply_impl(c, e, x, ldx, mc, y, ldy);
      ck(cudaStreamSynchronize(c->stream), "sync");
      return;
    }
    const int n_r = e->n_r, n_mu = e->n_mu;
    DBuf u = dalloc(c, (size_t)n_mu * mc), w = dalloc(c, (size_t)n_mu * mc);
    Work wk = make_work(c, (size_t)1200 * n_mu * mc);
    if (skinny_supported(mc))
      ck(skinny_tn(c->stream, e->theta, rows, rows, n_mu, x, ldx, mc, u.d(), n_mu, wk.buf.d(), wk.elems, c->sm_count),
         "skinny_tn");
    else
      gemm(c, n_mu, mc, rows, e->theta, rows, Lay::K, x, ldx, Lay::K, u.d(), n_mu, 1.0, 0.0, nullptr, false, &wk);
    allreduce(c, m, u.d(), (size_t)n_mu * mc);
    gemm(c, n_mu, mc, n_mu, e->k, n_mu, Lay::MN, u.d(), n_mu, Lay::K, w.d(), n_mu, 1.0, 0.0);
    // z_p = Theta_p w, padded to the largest panel for the all-gather
    const int mr = pn.max_rows;
    DBuf zs = dalloc(c, (size_t)mr * mc), zg = dalloc(c, (size_t)mr * mc * m->world), z = dalloc(c, (size_t)n_r * mc);
    gemm(c, rows, mc, n_mu, e->theta, rows, Lay::MN, w.d(), n_mu, Lay::K, zs.d(), mr, 1.0, 0.0);
    allgather(c, m, zs.p, zg.p, sizeof(double) * (size_t)mr * mc);
    for (int q = 0; q < m->world; ++q)
      ck(cudaMemcpy2DAsync(z.d() + pn.row0[q], sizeof(double) * n_r, zg.d() + (size_t)q * mr * mc,
                           sizeof(double) * mr, sizeof(double) * pn.rows[q], mc, cudaMemcpyDeviceToDevice, c->stream),
         "D2D");
    // V z on the full grid (m columns), then this rank's rows: y_p = x_p + (V z)_p
    DBuf vz = dalloc(c, (size_t)n_r * mc);
    coulomb_apply(c, e->dims, e->cell, e->zero, z.d(), n_r, mc, vz.d(), n_r);
    ck(cudaMemcpy2DAsync(y, sizeof(double) * ldy, vz.d() + row0, sizeof(double) * n_r, sizeof(double) * rows, mc,
                         cudaMemcpyDeviceToDevice, c->stream),
       "D2D");
    ck(axpby(c->stream, rows, mc, 1.0, x, ldx, 1.0, y, ldy), "axpby");
    ck(cudaStreamSynchronize(c->stream), "sync");
  });
}

}  // extern "C"
