// shard_kernels.cu — device pieces of the multi-rank build (sharded.cu):
// the global candidate merge of a selection block, owner-contributed row
// gathers, the accepted-pivot row pick, and the y-slab pack / z-pencil
// unpack of the slab-decomposed 3-D FFT.
#include <cfloat>
#include <climits>

#include "kernels.h"
#include "shard.h"

namespace lrgw_dev {

namespace {

struct Ent {  // select.cu's candidate entry (checked against select_ent_bytes())
  double v;
  int pos, row;
};

__device__ __forceinline__ bool ent_before(const Ent& a, int ia, const Ent& b, int ib) {
  // pivot order: larger residual, then the lower current position
  // (strict '>' scan over positions, linalg.hpp:45-53); absent entries last,
  // ties between absent entries by slot
  const bool pa = a.row >= 0, pb = b.row >= 0;
  if (pa != pb) return pa;
  if (!pa) return ia < ib;
  if (a.v != b.v) return a.v > b.v;
  if (a.pos != b.pos) return a.pos < b.pos;
  return ia < ib;
}

// One CTA: rank every gathered entry by counting the entries ahead of it;
// the first s1 land in rank order. Local panel rows become global rows.
__global__ void merge_top_kernel(const Ent* in, int world, int s1, const int* row0, Ent* out) {
  extern __shared__ Ent sh[];
  const int n = world * s1;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    Ent e = in[i];
    if (e.row >= 0) e.row += row0[i / s1];
    sh[i] = e;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const Ent e = sh[i];
    int r = 0;
    for (int j = 0; j < n; ++j) r += ent_before(sh[j], j, e, i) ? 1 : 0;
    if (r < s1) out[r] = e.row >= 0 ? e : Ent{-DBL_MAX, INT_MAX, -1};
  }
}

// out(i, [a | b | l]) = row rows[i] of the panel when this rank owns it, else 0.
__global__ void gather_owned_kernel(const double* a, long long lda, int n1, const double* b, long long ldb, int n2,
                                    const double* l, long long ldl, int nl, const int* rows, int n, int row0,
                                    int panel_rows, double* out, long long ldo) {
  const int width = n1 + n2 + nl;
  const long long total = (long long)n * width;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
       q += (long long)gridDim.x * blockDim.x) {
    const int i = static_cast<int>(q % n);
    const int c = static_cast<int>(q / n);
    const int g = rows[i] - row0;
    double v = 0.0;
    if (g >= 0 && g < panel_rows) {
      if (c < n1)
        v = a[(long long)c * lda + g];
      else if (c < n1 + n2)
        v = b[(long long)(c - n1) * ldb + g];
      else
        v = l[(long long)(c - n1 - n2) * ldl + g];
    }
    out[(long long)c * ldo + i] = v;
  }
}

// dst(t, :) = src(j, :) where top[j].row == piv[t] (the accepted pivots are
// candidates of the block).
__global__ void pick_rows_kernel(const Ent* top, int s, const int* piv, int nb, const double* src, long long lds,
                                 int width, double* dst, long long ldd) {
  __shared__ int at[128];
  for (int t = threadIdx.x; t < nb; t += blockDim.x) {
    int j = 0;
    for (int q = 0; q < s; ++q)
      if (top[q].row == piv[t]) j = q;
    at[t] = j;
  }
  __syncthreads();
  for (long long q = threadIdx.x; q < (long long)nb * width; q += blockDim.x) {
    const int t = static_cast<int>(q % nb);
    const int c = static_cast<int>(q / nb);
    dst[(long long)c * ldd + t] = src[(long long)c * lds + at[t]];
  }
}

// xa: (n_mu, zl, n2, n1h) complex -> dst (n_mu, zl, ny, n1h), y in [ya, ya+ny)
__global__ void slab_pack_kernel(const double2* xa, int n_mu, int zl, int n2, int n1h, int ya, int ny, double2* dst) {
  const long long total = (long long)n_mu * zl * ny * n1h;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
       q += (long long)gridDim.x * blockDim.x) {
    const int x = static_cast<int>(q % n1h);
    long long r = q / n1h;
    const int y = static_cast<int>(r % ny);
    r /= ny;  // (j, z)
    dst[q] = xa[(r * n2 + ya + y) * n1h + x];
  }
}

// src (n_mu, zl, ny, n1h) from the rank owning planes [z0, z0+zl) -> pencil (n_mu, ny, n1h, n3)
__global__ void slab_unpack_kernel(const double2* src, int n_mu, int zl, int ny, int n1h, int z0, int n3,
                                   double2* pencil) {
  const long long total = (long long)n_mu * zl * ny * n1h;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
       q += (long long)gridDim.x * blockDim.x) {
    const int x = static_cast<int>(q % n1h);
    long long r = q / n1h;
    const int y = static_cast<int>(r % ny);
    r /= ny;
    const int z = static_cast<int>(r % zl);
    const long long j = r / zl;
    pencil[((j * ny + y) * n1h + x) * n3 + z0 + z] = src[q];
  }
}

__global__ void iota_kernel(int* a, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) a[i] = i;
}

inline int blocks_for(long long n, int per = 256, int cap = 1184) {
  const long long b = (n + per - 1) / per;
  return static_cast<int>(b < 1 ? 1 : (b > cap ? cap : b));
}

}  // namespace

size_t shard_ent_bytes() { return sizeof(Ent); }

cudaError_t shard_iota(cudaStream_t st, int* a, int n) {
  iota_kernel<<<blocks_for(n), 256, 0, st>>>(a, n);
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t shard_merge_top(cudaStream_t st, const void* gathered, int world, int s1, const int* row0, void* top) {
  const size_t smem = sizeof(Ent) * (size_t)world * s1;
  if (smem > 48 * 1024) return cudaErrorInvalidValue;
  merge_top_kernel<<<1, 512, smem, st>>>(static_cast<const Ent*>(gathered), world, s1, row0, static_cast<Ent*>(top));
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t shard_gather_owned(cudaStream_t st, const double* a, long long lda, int n1, const double* b, long long ldb,
                               int n2, const double* l, long long ldl, int nl, const int* rows, int n, int row0,
                               int panel_rows, double* out, long long ldo) {
  const long long total = (long long)n * (n1 + n2 + nl);
  if (total == 0) return cudaSuccess;
  gather_owned_kernel<<<blocks_for(total), 256, 0, st>>>(a, lda, n1, b, ldb, n2, l, ldl, nl, rows, n, row0,
                                                         panel_rows, out, ldo);
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t shard_pick_rows(cudaStream_t st, const void* top, int s, const int* piv, int nb, const double* src,
                            long long lds, int width, double* dst, long long ldd) {
  if (nb > 128) return cudaErrorInvalidValue;
  pick_rows_kernel<<<1, 512, 0, st>>>(static_cast<const Ent*>(top), s, piv, nb, src, lds, width, dst, ldd);
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t shard_slab_pack(cudaStream_t st, const double* xa, int n_mu, int zl, int n2, int n1h, int ya, int ny,
                            double* dst) {
  const long long total = (long long)n_mu * zl * ny * n1h;
  if (total == 0) return cudaSuccess;
  slab_pack_kernel<<<blocks_for(total), 256, 0, st>>>(reinterpret_cast<const double2*>(xa), n_mu, zl, n2, n1h, ya, ny,
                                                      reinterpret_cast<double2*>(dst));
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t shard_slab_unpack(cudaStream_t st, const double* src, int n_mu, int zl, int ny, int n1h, int z0, int n3,
                              double* pencil) {
  const long long total = (long long)n_mu * zl * ny * n1h;
  if (total == 0) return cudaSuccess;
  slab_unpack_kernel<<<blocks_for(total), 256, 0, st>>>(reinterpret_cast<const double2*>(src), n_mu, zl, ny, n1h, z0,
                                                        n3, reinterpret_cast<double2*>(pencil));
  count_launches(1);
  return cudaGetLastError();
}

}  // namespace lrgw_dev
