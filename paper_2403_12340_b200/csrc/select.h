// select.h — K1 ISDF point-selection device entry points (select.cu).
#pragma once

#include <cstddef>
#include <cuda_runtime.h>

namespace lrgw_dev {

// d[r] = (sum_i a_ri^2)(sum_j b_rj^2) (diag of the Hadamard Gram), pos[r] = r.
cudaError_t select_init(cudaStream_t st, const double* a, long long lda, int n1, const double* b,
                        long long ldb, int n2, int n_r, double* d, int* pos);
// Top-s rows by (d desc, position asc) among positions >= k -> cand[0..n_cand).
size_t select_topk_tmp_elems(int n_r, int s);
cudaError_t select_topk(cudaStream_t st, const double* d, const int* pos, int n_r, int k, int s,
                        double* tmp_v, int* tmp_p, int* tmp_g, int* cand, int* n_cand);
int select_grid_blocks(int sm_count);
size_t select_part_bytes(int grid_blocks);
int select_max_candidates();
// Exact greedy steps from kb while the argmax stays among the candidates.
cudaError_t select_steps(cudaStream_t st, int grid_blocks, int n_r, int steps, int kb, double* d,
                         int* pos, double* L, const double* W, const int* cand, int n_cand,
                         void* part, int* piv_order, double* margin, int* k_out);
cudaError_t select_scatter_perm(cudaStream_t st, const int* pos, int n_r, int* perm);

}  // namespace lrgw_dev
