// select.h — K1 ISDF point-selection device entry points (select.cu).
#pragma once

#include <cstddef>
#include <cuda_runtime.h>

namespace lrgw_dev {

// d[r] = (sum_i a_ri^2)(sum_j b_rj^2) (diag of the Hadamard Gram), pos = perm = identity.
cudaError_t select_init(cudaStream_t st, const double* a, long long lda, int n1, const double* b,
                        long long ldb, int n2, int n_r, double* d, int* pos, int* perm);
// Top s1 unselected rows (positions >= k) by (d desc, position asc) into `out`
// (s1 opaque entries of select_ent_bytes()); missing entries have row -1.
size_t select_ent_bytes();
size_t select_topk_tmp_bytes(int n_r, int s1);
// tmp must be zeroed once before the first select_topk (each call leaves it zeroed).
cudaError_t select_topk_reset(cudaStream_t st, void* tmp);
cudaError_t select_topk(cudaStream_t st, const double* d, const int* pos, int n_r, int k, int s1, void* tmp,
                        void* out, const int* k_dev = nullptr);
cudaError_t select_cand_rows(cudaStream_t st, const void* top, int n, int* rows);
int select_max_candidates();
size_t select_cand_smem_bytes(int s);
// Certified greedy on the s candidates (one CTA) from their Schur block
// wcc = W[C, C] (s x s, ld s, symmetric): accepted steps -> *b_out (and the
// next block start -> b_out[1]), pivots (perm / pos / piv_order), margins (if
// margin != nullptr); xcol (ld s) = X = L_sel^-1 column-major (b x b lower,
// L_sel the accepted steps' l values at the accepted rows, in pivot order).
cudaError_t select_cand_greedy(cudaStream_t st, int n_r, int s, int steps, int kb, const void* top, const double* wcc,
                               int* pos, int* perm, double* xcol, int* piv_order, double* margin, int* b_out,
                               int bmax, int bround, const int* kb_dev = nullptr, int* k_next = nullptr,
                               double* xperm = nullptr, int* b_host = nullptr);
// W[C, C] -= Lr Lr^T over the device-side pivot count *k_dev (Lr: s x k, ld
// ldl; s <= 128); work: select_wcc_work_elems() doubles.
size_t select_wcc_work_elems();
cudaError_t select_wcc_lsub(cudaStream_t st, const double* lr, long long ldl, int s, const int* k_dev, double* wcc,
                            double* work);
// Pivots the block pipeline accepts per candidate block (a prefix of the
// certified greedy run): at most select_accept_cap, and a run that stops
// between select_accept_round and the cap keeps select_accept_round — the
// widths the tall-skinny GEMM tiles run best at.
int select_accept_cap(int s, int n_r, bool panel_tma = false);
int select_accept_round();
// d -= rowsum(L[:, kb:kb+b]^2) over unselected rows.
cudaError_t select_downdate(cudaStream_t st, const double* L, int n_r, int kb, int b, const int* pos, double* d,
                            const int* b_dev = nullptr);

}  // namespace lrgw_dev
