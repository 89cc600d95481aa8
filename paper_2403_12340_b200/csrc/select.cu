// select.cu — K1: ISDF interpolation-point selection on the GPU.
//
// Reference: select_interpolation_points (isdf.hpp:95-112) -> Householder QRCP
// on the materialised pair matrix Z (linalg.hpp:26-111, guard 2^26 entries).
// B200 design: matrix-free greedy pivoted Cholesky on the Hadamard Gram
// G = (Phi_a Phi_a^T) o (Phi_b Phi_b^T) = Z^T Z, whose residual diagonal d
// equals QRCP's residual column norms, so the greedy pivots coincide. The
// pivot rule is mirrored exactly: argmax over remaining positions with strict
// '>' (ties to the lowest current position; positions follow the
// perm[step] <-> perm[p] swap of linalg.hpp:48-53), min(N1 N2, N_r) steps, the
// first N_mu positions sorted ascending.
//
// Certified candidate blocks (no grid-wide barrier per pivot):
//   1. C = the top-s unselected rows by (d desc, position asc), tau = the
//      (s+1)-th residual. Residuals only decrease, so every non-candidate
//      stays <= tau for the whole block.
//   2. W = G(:, C) - L[:, :k0] L[C, :k0]^T for all rows (two DMMA GEMM passes).
//   3. One CTA runs the exact greedy on the s x s candidate Schur complement
//      W[C, C] in shared memory; a step is accepted only while the best
//      candidate beats tau strictly (the first step of a block is the exact
//      argmax by construction of C), so every accepted pivot is the global
//      greedy pivot.
//   4. The block's L columns for all rows follow from one GEMM,
//      L[:, k0:k0+b] = W L_sel^-T, and d -= rowsum(L_blk^2).
// Block lengths are ~60-80% of s; the pivot sequence is that of the plain
// greedy (the tests check it bit-exactly against the reference).
#include <cfloat>

#include "common.cuh"
#include "kernels.h"
#include "select.h"

namespace lrgw_dev {

namespace {

// (value, position) ordering: larger value first, then the lower position
// (the reference's strict '>' scan in position order, linalg.hpp:45-47).
__device__ __forceinline__ bool better(double v1, int p1, double v2, int p2) {
  return v1 > v2 || (v1 == v2 && p1 < p2);
}

// l of the pivot itself: sqrt(d_piv) = 1 / inv (0 for an exhausted pivot).
__device__ __forceinline__ double s_bv_sqrt(double inv) { return inv > 0.0 ? 1.0 / inv : 0.0; }

__global__ void init_diag_kernel(const double* a, long long lda, int n1, const double* b,
                                 long long ldb, int n2, int n_r, double* d, int* pos, int* perm) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n_r; r += gridDim.x * blockDim.x) {
    double sa = 0.0, sb = 0.0;
    for (int i = 0; i < n1; ++i) {
      const double x = a[r + (long long)i * lda];
      sa = fma(x, x, sa);
    }
    for (int j = 0; j < n2; ++j) {
      const double x = b[r + (long long)j * ldb];
      sb = fma(x, x, sb);
    }
    d[r] = sa * sb;
    pos[r] = r;
    perm[r] = r;
  }
}

// ---- top-(s+1) by (d desc, position asc): per-CTA bitonic + merge passes ----
constexpr int TOPK_CHUNK = 2048;

struct Ent {
  double v;
  int pos, row;
};

__device__ __forceinline__ bool ent_better(const Ent& a, const Ent& b) { return better(a.v, a.pos, b.v, b.pos); }

__device__ void bitonic_desc(Ent* e, int n) {
  for (int size = 2; size <= n; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      __syncthreads();
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int j = i ^ stride;
        if (j > i) {
          const Ent a = e[i], b = e[j];
          const bool desc = ((i & size) == 0);
          if (desc ? ent_better(b, a) : ent_better(a, b)) {
            e[i] = b;
            e[j] = a;
          }
        }
      }
    }
  }
  __syncthreads();
}

__device__ __forceinline__ Ent ent_none() { return Ent{-DBL_MAX, INT_MAX, -1}; }

__global__ void topk_pass1_kernel(const double* d, const int* pos, int n_r, int k, const int* k_dev, int s, Ent* out) {
  __shared__ Ent e[TOPK_CHUNK];
  if (k_dev) k = *k_dev;
  const int base = blockIdx.x * TOPK_CHUNK;
  for (int i = threadIdx.x; i < TOPK_CHUNK; i += blockDim.x) {
    const int r = base + i;
    const int pr = r < n_r ? pos[r] : -1;
    e[i] = (r < n_r && pr >= k) ? Ent{d[r], pr, r} : ent_none();
  }
  bitonic_desc(e, TOPK_CHUNK);
  for (int i = threadIdx.x; i < s; i += blockDim.x) out[blockIdx.x * s + i] = e[i];
}

__global__ void topk_merge_kernel(const Ent* in, int n_in, int s, Ent* out) {
  __shared__ Ent e[TOPK_CHUNK];
  const int base = blockIdx.x * TOPK_CHUNK;
  for (int i = threadIdx.x; i < TOPK_CHUNK; i += blockDim.x) {
    const int r = base + i;
    e[i] = r < n_in ? in[r] : ent_none();
  }
  bitonic_desc(e, TOPK_CHUNK);
  for (int i = threadIdx.x; i < s; i += blockDim.x) out[blockIdx.x * s + i] = e[i];
}

// ---- the certified candidate greedy (one CTA) -------------------------------
constexpr int CG_THREADS = 512;
constexpr int CG_WARPS = CG_THREADS / 32;
constexpr int CG_ROWS = 128 / CG_WARPS;  // candidate rows per warp

struct CandParams {
  int n_r, s, steps, kb;
  const Ent* top;       // s + 1 entries: candidates then the tau entry
  const double* W;      // n_r x s
  int* pos;             // grid row -> position
  int* perm;            // position -> grid row
  double* lc;           // s x s: l vectors of the accepted steps (column t)
  double* mprime;       // s x s: E L_sel^-T (rows of unselected candidates zero)
  int* piv_order;       // [steps]
  double* margin;       // [steps]
  int* b_out;           // number of accepted steps
};

// Register-resident candidate block: warp w owns candidate rows
// i = CG_ROWS w + r (r < CG_ROWS) and lane l holds their columns l, l+32, l+64,
// l+96 (s <= 128); lane r additionally carries row r's residual and position.
// Per accepted pivot: post per-warp best (lanes 0..CG_ROWS-1), barrier, every
// warp reduces the CG_WARPS partials redundantly and the owner publishes the
// pivot row, barrier, every warp applies the rank-1 elimination in registers.
__device__ __forceinline__ void argmax_xor(double& v, double& sv, int& i, int& p, int off) {
  const double v2 = __shfl_xor_sync(0xffffffffu, v, off);
  const double s2 = __shfl_xor_sync(0xffffffffu, sv, off);
  const int i2 = __shfl_xor_sync(0xffffffffu, i, off);
  const int p2 = __shfl_xor_sync(0xffffffffu, p, off);
  if (better(v2, p2, v, p)) {
    sv = fmax(fmax(sv, s2), v);
    v = v2;
    p = p2;
    i = i2;
  } else {
    sv = fmax(fmax(sv, s2), v2);
  }
}

__global__ void __launch_bounds__(CG_THREADS, 1) cand_greedy_kernel(CandParams p) {
  extern __shared__ __align__(16) double sm[];
  const int s = p.s, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  double* rowbuf = sm;                             // 128: published pivot row
  int* usedv = reinterpret_cast<int*>(rowbuf + 128);  // 128 flags
  int* rowid = usedv + 128;                        // 128 grid rows
  int* sel = rowid + 128;                          // 128: candidate index per accepted step
  int* pslot = sel + 128;                          // 128: perm[kb .. kb + s)
  __shared__ double part_v[CG_WARPS], part_s[CG_WARPS];
  __shared__ int part_i[CG_WARPS], part_p[CG_WARPS];
  __shared__ double s_tau;

  for (int i = tid; i < 128; i += blockDim.x) {
    const Ent e = i < s ? p.top[i] : ent_none();
    rowid[i] = e.row;
    usedv[i] = e.row < 0 ? 1 : 0;
    pslot[i] = (i < s && p.kb + i < p.n_r) ? p.perm[p.kb + i] : -1;
  }
  if (tid == 0) s_tau = p.top[s].row >= 0 ? p.top[s].v : -DBL_MAX;
  __syncthreads();
  const double tau = s_tau;
  const int tmax = min(s, p.steps - p.kb);

  const int base = CG_ROWS * wid;
  double w[CG_ROWS][4];
#pragma unroll
  for (int r = 0; r < CG_ROWS; ++r) {
    const int g = rowid[base + r];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int j = lane + 32 * c;
      w[r][c] = (g >= 0 && j < s) ? p.W[g + (long long)j * p.n_r] : 0.0;
    }
  }
  // lane r < CG_ROWS: metadata of row base + r
  const int my_i = base + (lane < CG_ROWS ? lane : 0);
  double my_d = -DBL_MAX;
  int my_pos = INT_MAX;
  if (lane < CG_ROWS && my_i < s && rowid[my_i] >= 0) {
    my_d = p.top[my_i].v;
    my_pos = p.top[my_i].pos;
  }

  int t = 0;
  for (;; ++t) {
    // ---- post this warp's best unused row ----
    double bv = -DBL_MAX, sv = -DBL_MAX;
    int bi = -1, bp = INT_MAX;
    if (lane < CG_ROWS && !usedv[my_i]) {
      bv = my_d;
      bp = my_pos;
      bi = my_i;
    }
#pragma unroll
    for (int off = CG_ROWS / 2; off > 0; off >>= 1) argmax_xor(bv, sv, bi, bp, off);
    if (lane == 0) {
      part_v[wid] = bv;
      part_s[wid] = sv;
      part_i[wid] = bi;
      part_p[wid] = bp;
    }
    __syncthreads();
    // ---- every warp reduces the partials ----
    double v0 = -DBL_MAX, s0 = -DBL_MAX;
    int i0 = -1, p0 = INT_MAX;
    if (lane < CG_WARPS) {
      v0 = part_v[lane];
      s0 = part_s[lane];
      i0 = part_i[lane];
      p0 = part_p[lane];
    }
#pragma unroll
    for (int off = CG_WARPS / 2; off > 0; off >>= 1) argmax_xor(v0, s0, i0, p0, off);
    v0 = __shfl_sync(0xffffffffu, v0, 0);
    s0 = __shfl_sync(0xffffffffu, s0, 0);
    i0 = __shfl_sync(0xffffffffu, i0, 0);
    p0 = __shfl_sync(0xffffffffu, p0, 0);
    // certified iff it beats every non-candidate (<= tau); the first step of
    // the block is the exact argmax (C is sorted by the pivot rule)
    const bool ok = t < tmax && i0 >= 0 && (t == 0 || v0 > tau);
    if (!ok) break;  // uniform across the CTA
    const int k = p.kb + t;
    const int ppos = p0;       // pivot's position before the swap
    const int occ = pslot[t];  // perm[k] before the swap (linalg.hpp:48-53)
    if (wid == i0 / CG_ROWS) {
      const int r0 = i0 % CG_ROWS;
#pragma unroll
      for (int r = 0; r < CG_ROWS; ++r)
        if (r == r0)
#pragma unroll
          for (int c = 0; c < 4; ++c) rowbuf[lane + 32 * c] = w[r][c];
    }
    __syncthreads();
    // ---- eliminate the pivot from the register block ----
    const double inv = v0 > 0.0 ? 1.0 / sqrt(v0) : 0.0;
    const double lpiv = v0 > 0.0 ? sqrt(v0) : 0.0;
    double lj[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int j = lane + 32 * c;
      lj[c] = (j == i0) ? lpiv : rowbuf[j] * inv;
    }
    double my_l = 0.0;
#pragma unroll
    for (int r = 0; r < CG_ROWS; ++r) {
      const int i = base + r;
      const double li = (i == i0) ? lpiv : (usedv[i] ? 0.0 : rowbuf[i] * inv);
#pragma unroll
      for (int c = 0; c < 4; ++c) w[r][c] = fma(-li, lj[c], w[r][c]);
      if (lane == r) my_l = li;
    }
    if (lane < CG_ROWS && my_i < s) {
      p.lc[my_i + (size_t)t * s] = my_l;
      if (my_i == i0) {
        usedv[my_i] = 1;
        my_pos = k;
      } else {
        if (!usedv[my_i]) my_d = fma(-my_l, my_l, my_d);
        if (rowid[my_i] == occ) my_pos = ppos;
      }
    }
    if (tid == 0) {
      const int gp = rowid[i0];
      p.perm[k] = gp;
      p.perm[ppos] = occ;
      p.pos[gp] = k;
      p.pos[occ] = ppos;
      if (ppos - p.kb < s) pslot[ppos - p.kb] = occ;
      pslot[t] = gp;
      sel[t] = i0;
      p.piv_order[k] = gp;
      if (p.margin) p.margin[k] = v0 > 0.0 ? (v0 - fmax(s0, tau)) / v0 : 0.0;
    }
    // usedv / pslot / sel are next read after the next step's first barrier
  }
  __syncthreads();
  const int b = t;
  // M' = E L_sel^-T. L_sel[t1][t2] = lc[sel[t1] + t2 s] is lower triangular in
  // pivot order: pack it into shared memory and invert row by row
  // (X[i][:] = (e_i - sum_{m<i} L[i][m] X[m][:]) / L[i][i], columns in parallel).
  double* lp = reinterpret_cast<double*>(pslot + 128);  // b (b + 1) / 2, packed lower
  double* xp = lp + (size_t)b * (b + 1) / 2;              // b (b + 1) / 2
  for (int idx = tid; idx < b * b; idx += blockDim.x) {
    const int i = idx / b, m = idx % b;
    if (m <= i) lp[(size_t)i * (i + 1) / 2 + m] = p.lc[sel[i] + (size_t)m * s];
  }
  for (int idx = tid; idx < s * b; idx += blockDim.x) p.mprime[idx] = 0.0;
  __syncthreads();
  {
    // G = CG_THREADS / 128 threads per column j (128 >= s columns), m-sum
    // split across them and reduced with shuffles inside the group.
    constexpr int G = CG_THREADS / 128;
    const int j = tid / G, q = tid % G;
    for (int i = 0; i < b; ++i) {
      const double* li = lp + (size_t)i * (i + 1) / 2;
      double acc = 0.0;
      if (j <= i)
        for (int m = j + q; m < i; m += G) acc = fma(li[m], xp[(size_t)m * (m + 1) / 2 + j], acc);
#pragma unroll
      for (int off = G / 2; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
      if (j <= i && q == 0) {
        const double lii = li[i];
        const double x = lii != 0.0 ? (((i == j) ? 1.0 : 0.0) - acc) / lii : 0.0;
        xp[(size_t)i * (i + 1) / 2 + j] = x;
        p.mprime[sel[j] + (size_t)i * s] = x;  // (L_sel^-T)[j][i] = X[i][j]
      }
      __syncthreads();
    }
  }
  if (tid == 0) {
    p.b_out[0] = b;
    p.b_out[1] = p.kb + b;  // next block start, consumed on the device
  }
}

__global__ void cand_rows_kernel(const Ent* top, int n, int* rows) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) rows[i] = top[i].row < 0 ? 0 : top[i].row;
}

// d[r] -= sum_t L[r, kb + t]^2 for the rows still unselected.
__global__ void downdate_kernel(const double* L, int n_r, int kb, int b, const int* b_dev, const int* pos, double* d) {
  if (b_dev) b = *b_dev;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n_r; r += gridDim.x * blockDim.x) {
    if (pos[r] < kb + b) continue;
    double v = d[r];
    const double* lr = L + (long long)kb * n_r + r;
    for (int t = 0; t < b; ++t) {
      const double l = lr[(long long)t * n_r];
      v = fma(-l, l, v);
    }
    d[r] = v;
  }
}

}  // namespace

size_t select_topk_tmp_bytes(int n_r, int s1) {
  return 2 * (size_t)((n_r + TOPK_CHUNK - 1) / TOPK_CHUNK) * s1 * sizeof(Ent) + 64;
}

size_t select_ent_bytes() { return sizeof(Ent); }

cudaError_t select_init(cudaStream_t st, const double* a, long long lda, int n1, const double* b,
                        long long ldb, int n2, int n_r, double* d, int* pos, int* perm) {
  init_diag_kernel<<<592, 256, 0, st>>>(a, lda, n1, b, ldb, n2, n_r, d, pos, perm); count_launches(1);
  return cudaGetLastError();
}

cudaError_t select_topk(cudaStream_t st, const double* d, const int* pos, int n_r, int k, int s1, void* tmp,
                        void* out, const int* k_dev) {
  Ent* t = static_cast<Ent*>(tmp);
  const int n = (n_r + TOPK_CHUNK - 1) / TOPK_CHUNK;
  const size_t half = (size_t)n * s1;
  topk_pass1_kernel<<<n, 1024, 0, st>>>(d, pos, n_r, k, k_dev, s1, t); count_launches(1);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  int n_in = n * s1, src = 0;
  while (true) {
    const int chunks = (n_in + TOPK_CHUNK - 1) / TOPK_CHUNK;
    Ent* from = t + src * half;
    Ent* to = chunks == 1 ? static_cast<Ent*>(out) : t + (1 - src) * half;
    topk_merge_kernel<<<chunks, 1024, 0, st>>>(from, n_in, s1, to); count_launches(1);
    e = cudaGetLastError();
    if (e != cudaSuccess || chunks == 1) return e;
    n_in = chunks * s1;
    src = 1 - src;
  }
}

size_t select_cand_smem_bytes(int s) { return 128 * 8 + 4 * 128 * 4 + (size_t)s * (s + 1) * 8 + 64; }

int select_max_candidates() { return 128; }

cudaError_t select_cand_greedy(cudaStream_t st, int n_r, int s, int steps, int kb, const void* top, const double* W,
                               int* pos, int* perm, double* lc, double* mprime, int* piv_order, double* margin,
                               int* b_out) {
  CandParams p{n_r, s, steps, kb, static_cast<const Ent*>(top), W, pos, perm, lc, mprime, piv_order, margin, b_out};
  const size_t smem = select_cand_smem_bytes(s);
  cudaError_t e = cudaFuncSetAttribute(cand_greedy_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  cand_greedy_kernel<<<1, CG_THREADS, smem, st>>>(p); count_launches(1);
  return cudaGetLastError();
}

cudaError_t select_cand_rows(cudaStream_t st, const void* top, int n, int* rows) {
  cand_rows_kernel<<<1, 256, 0, st>>>(static_cast<const Ent*>(top), n, rows); count_launches(1);
  return cudaGetLastError();
}

cudaError_t select_downdate(cudaStream_t st, const double* L, int n_r, int kb, int b, const int* pos, double* d,
                            const int* b_dev) {
  if (b <= 0 && !b_dev) return cudaSuccess;
  downdate_kernel<<<592, 256, 0, st>>>(L, n_r, kb, b, b_dev, pos, d); count_launches(1);
  return cudaGetLastError();
}

}  // namespace lrgw_dev
