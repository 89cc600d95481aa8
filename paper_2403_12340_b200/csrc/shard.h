// shard.h — device entry points of the multi-rank build (shard_kernels.cu,
// coulomb.cu) used by sharded.cu.
#pragma once

#include <cstddef>
#include <cuda_runtime.h>

namespace lrgw_dev {

size_t shard_ent_bytes();
cudaError_t shard_iota(cudaStream_t st, int* a, int n);
// gathered: world x s1 candidate entries (each rank's local top, panel rows);
// top: the global top s1 by the pivot order, rows made global with row0[rank].
cudaError_t shard_merge_top(cudaStream_t st, const void* gathered, int world, int s1, const int* row0, void* top);
// out(i, [a | b | l(:, :nl)]) = the panel's row rows[i] - row0 when owned, else 0 (ld ldo).
cudaError_t shard_gather_owned(cudaStream_t st, const double* a, long long lda, int n1, const double* b, long long ldb,
                               int n2, const double* l, long long ldl, int nl, const int* rows, int n, int row0,
                               int panel_rows, double* out, long long ldo);
// dst(t, :) = src(j, :) with top[j].row == piv[t], t < nb (nb <= 128).
cudaError_t shard_pick_rows(cudaStream_t st, const void* top, int s, const int* piv, int nb, const double* src,
                            long long lds, int width, double* dst, long long ldd);
// (n_mu, zl, n2, n1h) complex -> (n_mu, zl, ny, n1h), y in [ya, ya + ny)
cudaError_t shard_slab_pack(cudaStream_t st, const double* xa, int n_mu, int zl, int n2, int n1h, int ya, int ny,
                            double* dst);
// (n_mu, zl, ny, n1h) complex of planes [z0, z0 + zl) -> pencil (n_mu, ny, n1h, n3)
cudaError_t shard_slab_unpack(cudaStream_t st, const double* src, int n_mu, int zl, int ny, int n1h, int z0, int n3,
                              double* pencil);
// Weights of the y-slab [ya, ya + ny) in pencil order (y, x, z), z fastest:
// w_G v(G) / N_r twice (re, im) — the slab SYRK's k-scale (coulomb.cu).
cudaError_t coulomb_slab_weights(cudaStream_t st, int n1, int n2, int n3, double c1, double c2, double c3,
                                 int zero_kernel, int ya, int ny, double* w);

}  // namespace lrgw_dev
