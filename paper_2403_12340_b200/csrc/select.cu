// select.cu — K1: ISDF interpolation-point selection on the GPU.
//
// Reference: select_interpolation_points (isdf.hpp:95-112) -> Householder QRCP
// on the materialised pair matrix Z (linalg.hpp:26-111, guard 2^26 entries).
// B200 design: matrix-free greedy pivoted Cholesky on the Hadamard Gram
// G = (Phi_a Phi_a^T) o (Phi_b Phi_b^T) = Z^T Z, whose residual diagonal equals
// QRCP's residual column norms, so the greedy pivots coincide. The pivot rule
// is mirrored exactly: argmax over remaining positions with strict '>' (ties
// to the lowest current position, positions following the perm swap of
// linalg.hpp:48-53), min(N1 N2, N_r) steps, first N_mu sorted ascending.
//
// Speculative candidate batching: each block takes the top-s
// residuals as candidates, forms their kernel columns for all rows in one
// GEMM pass, W = G(:, cand) - L[:, :k0] L[cand, :k0]^T (DMMA), then a single
// cooperative kernel resolves exact greedy steps while the argmax stays inside
// the candidate set: per step one grid barrier, the new L column
// L[:, k] = (W[:, c_p] - L[:, kb:k] L[p, kb:k]^T) / sqrt(d_p), the residual
// downdate d -= L[:, k]^2 and a warp-shuffle (value, position) argmax. The
// pivot sequence is identical to the unbatched greedy; only the number of
// passes over Phi and L shrinks.
#include <cooperative_groups.h>

#include <cfloat>

#include "common.cuh"
#include "kernels.h"
#include "select.h"

namespace cg = cooperative_groups;

namespace lrgw_dev {

namespace {

// (value, position, grid index) ordering: larger value first, then the lower
// position (the reference's strict '>' scan in position order).
struct Cand {
  double v;
  int pos;
  int g;
};

__device__ __forceinline__ bool better(double v1, int p1, double v2, int p2) {
  return v1 > v2 || (v1 == v2 && p1 < p2);
}

__device__ __forceinline__ void warp_argmax(double& v, int& pos, int& g) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const double v2 = __shfl_down_sync(0xffffffffu, v, off);
    const int p2 = __shfl_down_sync(0xffffffffu, pos, off);
    const int g2 = __shfl_down_sync(0xffffffffu, g, off);
    if (better(v2, p2, v, pos)) {
      v = v2;
      pos = p2;
      g = g2;
    }
  }
}

__global__ void init_diag_kernel(const double* a, long long lda, int n1, const double* b,
                                 long long ldb, int n2, int n_r, double* d, int* pos) {
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
  }
}

// ---- top-s candidates: per-CTA bitonic sort of (d, pos) then a merge pass --
constexpr int TOPK_CHUNK = 2048;  // rows per CTA in pass 1 (power of two)

__device__ void bitonic_desc(double* v, int* p, int* gi, int n) {
  for (int size = 2; size <= n; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      __syncthreads();
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int j = i ^ stride;
        if (j > i) {
          const bool desc = ((i & size) == 0);
          const bool swap = desc ? better(v[j], p[j], v[i], p[i]) : better(v[i], p[i], v[j], p[j]);
          if (swap) {
            double tv = v[i];
            v[i] = v[j];
            v[j] = tv;
            int tp = p[i];
            p[i] = p[j];
            p[j] = tp;
            int tg = gi[i];
            gi[i] = gi[j];
            gi[j] = tg;
          }
        }
      }
    }
  }
  __syncthreads();
}

__global__ void topk_pass1_kernel(const double* d, const int* pos, int n_r, int k, int s,
                                  double* out_v, int* out_p, int* out_g) {
  __shared__ double v[TOPK_CHUNK];
  __shared__ int p[TOPK_CHUNK], gi[TOPK_CHUNK];
  const int base = blockIdx.x * TOPK_CHUNK;
  for (int i = threadIdx.x; i < TOPK_CHUNK; i += blockDim.x) {
    const int r = base + i;
    const bool ok = r < n_r && pos[r] >= k;
    v[i] = ok ? d[r] : -DBL_MAX;
    p[i] = ok ? pos[r] : INT_MAX;
    gi[i] = ok ? r : -1;
  }
  bitonic_desc(v, p, gi, TOPK_CHUNK);
  for (int i = threadIdx.x; i < s; i += blockDim.x) {
    out_v[blockIdx.x * s + i] = v[i];
    out_p[blockIdx.x * s + i] = p[i];
    out_g[blockIdx.x * s + i] = gi[i];
  }
}

// Merge pass: each CTA sorts TOPK_CHUNK candidates of the previous pass and
// keeps its top s; the last pass (one CTA) writes the candidate list.
__global__ void topk_merge_kernel(const double* in_v, const int* in_p, const int* in_g, int n_in,
                                  int s, double* out_v, int* out_p, int* out_g, int* cand,
                                  int* n_cand) {
  __shared__ double v[TOPK_CHUNK];
  __shared__ int p[TOPK_CHUNK], gi[TOPK_CHUNK];
  const int base = blockIdx.x * TOPK_CHUNK;
  for (int i = threadIdx.x; i < TOPK_CHUNK; i += blockDim.x) {
    const int r = base + i;
    const bool ok = r < n_in;
    v[i] = ok ? in_v[r] : -DBL_MAX;
    p[i] = ok ? in_p[r] : INT_MAX;
    gi[i] = ok ? in_g[r] : -1;
  }
  bitonic_desc(v, p, gi, TOPK_CHUNK);
  if (cand) {
    if (threadIdx.x == 0) {
      int c = 0;
      for (int i = 0; i < s; ++i) {
        if (gi[i] < 0) break;
        cand[c++] = gi[i];
      }
      *n_cand = c;
    }
    return;
  }
  for (int i = threadIdx.x; i < s; i += blockDim.x) {
    out_v[blockIdx.x * s + i] = v[i];
    out_p[blockIdx.x * s + i] = p[i];
    out_g[blockIdx.x * s + i] = gi[i];
  }
}

// ---- the cooperative step kernel ----------------------------------------
struct Part {
  double v;
  int pos, g, occupant;
};

constexpr int SEL_THREADS = 512;
constexpr int SEL_MAXS = 128;

struct StepParams {
  int n_r, steps;
  int kb;          // block start step (columns of W are for steps >= kb)
  double* d;
  int* pos;
  double* L;       // n_r x n_mu (col-major, ld n_r)
  const double* W; // n_r x s
  const int* cand;
  int n_cand;
  Part* part;      // [2][gridDim.x]
  int* piv_order;  // [steps]
  double* margin;  // [steps] (top-2 relative margin, optional)
  int* k_out;
};

__global__ void __launch_bounds__(SEL_THREADS, 1) select_steps_kernel(StepParams p) {
  cg::grid_group grid = cg::this_grid();
  __shared__ int s_cand[SEL_MAXS];
  __shared__ double s_lp[SEL_MAXS];
  __shared__ double red_v[SEL_THREADS / 32];
  __shared__ int red_p[SEL_THREADS / 32], red_g[SEL_THREADS / 32], red_o[SEL_THREADS / 32];
  __shared__ double s_second[SEL_THREADS / 32];
  __shared__ int s_dec[4];  // p, c_p, pos_p, occupant
  __shared__ double s_dp;

  const int nb = gridDim.x, b = blockIdx.x, tid = threadIdx.x;
  const int r0 = (int)((long long)p.n_r * b / nb), r1 = (int)((long long)p.n_r * (b + 1) / nb);
  for (int i = tid; i < p.n_cand; i += blockDim.x) s_cand[i] = p.cand[i];
  __syncthreads();

  int k = p.kb;
  int piv = -1, cpiv = -1;  // pending pivot (grid index, candidate column)
  double dpiv = 0.0;
  for (int iter = 0;; ++iter) {
    // ---- phase 1: apply the pending pivot, local argmax ----
    if (piv >= 0) {
      const int nt = k - p.kb;  // previous in-block columns
      for (int t = tid; t < nt; t += blockDim.x)
        s_lp[t] = p.L[piv + (long long)(p.kb + t) * p.n_r];
      __syncthreads();
      const double inv = dpiv > 0.0 ? 1.0 / sqrt(dpiv) : 0.0;
      double* Lk = p.L + (long long)k * p.n_r;
      const double* Wc = p.W + (long long)cpiv * p.n_r;
      for (int r = r0 + tid; r < r1; r += blockDim.x) {
        const int pr = p.pos[r];
        if (pr < k) {  // already a pivot: L is zero there (lower triangular)
          Lk[r] = 0.0;
          continue;
        }
        if (r == piv) {
          Lk[r] = dpiv > 0.0 ? sqrt(dpiv) : 0.0;
          continue;
        }
        double c = Wc[r];
        for (int t = 0; t < nt; ++t) c = fma(-p.L[r + (long long)(p.kb + t) * p.n_r], s_lp[t], c);
        const double l = dpiv > 0.0 ? c * inv : 0.0;
        Lk[r] = l;
        p.d[r] = fma(-l, l, p.d[r]);
      }
      ++k;
      __syncthreads();
    }
    // local argmax over rows with pos >= k; also find the occupant of position k
    double bv = -DBL_MAX, sv = -DBL_MAX;
    int bp = INT_MAX, bg = -1, occ = -1;
    for (int r = r0 + tid; r < r1; r += blockDim.x) {
      const int pr = p.pos[r];
      if (pr == k) occ = r;
      if (pr < k) continue;
      const double v = p.d[r];
      if (better(v, pr, bv, bp)) {
        sv = fmax(sv, bv);
        bv = v;
        bp = pr;
        bg = r;
      } else {
        sv = fmax(sv, v);
      }
    }
    {
      // second-best: track by max of non-winners (for margin logging only)
      double v = bv;
      int pp = bp, gg = bg;
      double s2 = sv;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        const double v2 = __shfl_down_sync(0xffffffffu, v, off);
        const int p2 = __shfl_down_sync(0xffffffffu, pp, off);
        const int g2 = __shfl_down_sync(0xffffffffu, gg, off);
        const double s22 = __shfl_down_sync(0xffffffffu, s2, off);
        const int o2 = __shfl_down_sync(0xffffffffu, occ, off);
        if (better(v2, p2, v, pp)) {
          s2 = fmax(fmax(s2, s22), v);
          v = v2;
          pp = p2;
          gg = g2;
        } else {
          s2 = fmax(fmax(s2, s22), v2);
        }
        occ = max(occ, o2);
      }
      const int w = tid >> 5;
      if ((tid & 31) == 0) {
        red_v[w] = v;
        red_p[w] = pp;
        red_g[w] = gg;
        red_o[w] = occ;
        s_second[w] = s2;
      }
      __syncthreads();
      if (tid == 0) {
        double v0 = red_v[0], s0 = s_second[0];
        int p0 = red_p[0], g0 = red_g[0], o0 = red_o[0];
        for (int i = 1; i < SEL_THREADS / 32; ++i) {
          if (better(red_v[i], red_p[i], v0, p0)) {
            s0 = fmax(fmax(s0, s_second[i]), v0);
            v0 = red_v[i];
            p0 = red_p[i];
            g0 = red_g[i];
          } else {
            s0 = fmax(fmax(s0, s_second[i]), red_v[i]);
          }
          o0 = max(o0, red_o[i]);
        }
        Part* out = p.part + (iter & 1) * nb + b;
        out->v = v0;
        out->pos = p0;
        out->g = g0;
        out->occupant = o0;
        // stash the CTA-local second best in the spare slot of the other buffer
        reinterpret_cast<double*>(p.part + 2 * nb)[(iter & 1) * nb + b] = s0;
      }
    }
    grid.sync();
    // ---- phase 2: global decision (identical in every CTA) ----
    if (tid == 0) {
      const Part* in = p.part + (iter & 1) * nb;
      const double* sec = reinterpret_cast<const double*>(p.part + 2 * nb) + (iter & 1) * nb;
      double v0 = in[0].v, s0 = sec[0];
      int p0 = in[0].pos, g0 = in[0].g, o0 = in[0].occupant;
      for (int i = 1; i < nb; ++i) {
        if (better(in[i].v, in[i].pos, v0, p0)) {
          s0 = fmax(fmax(s0, sec[i]), v0);
          v0 = in[i].v;
          p0 = in[i].pos;
          g0 = in[i].g;
        } else {
          s0 = fmax(fmax(s0, sec[i]), in[i].v);
        }
        o0 = max(o0, in[i].occupant);
      }
      int c = -1;
      if (k < p.steps && g0 >= 0)
        for (int i = 0; i < p.n_cand; ++i)
          if (s_cand[i] == g0) {
            c = i;
            break;
          }
      s_dec[0] = g0;
      s_dec[1] = c;
      s_dec[2] = p0;
      s_dec[3] = o0;
      s_dp = v0;
      if (b == 0 && c >= 0) {
        p.piv_order[k] = g0;
        if (p.margin) p.margin[k] = v0 > 0.0 ? (v0 - s0) / v0 : 0.0;
      }
    }
    __syncthreads();
    if (s_dec[1] < 0) break;  // miss (or done): block ends; state is consistent
    piv = s_dec[0];
    cpiv = s_dec[1];
    dpiv = s_dp;
    // mirrored swap: pivot -> position k, previous occupant -> pivot's position
    const int occupant = s_dec[3], pos_p = s_dec[2];
    if (tid == 0) {
      if (piv >= r0 && piv < r1) p.pos[piv] = k;
      if (occupant >= r0 && occupant < r1 && occupant != piv) p.pos[occupant] = pos_p;
    }
    __syncthreads();
  }
  if (b == 0 && tid == 0) *p.k_out = k;
}

__global__ void scatter_perm_kernel(const int* pos, int n_r, int* perm) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n_r; r += gridDim.x * blockDim.x)
    perm[pos[r]] = r;
}

}  // namespace

cudaError_t select_init(cudaStream_t st, const double* a, long long lda, int n1, const double* b,
                        long long ldb, int n2, int n_r, double* d, int* pos) {
  init_diag_kernel<<<592, 256, 0, st>>>(a, lda, n1, b, ldb, n2, n_r, d, pos); count_launches(1);
  return cudaGetLastError();
}

cudaError_t select_topk(cudaStream_t st, const double* d, const int* pos, int n_r, int k, int s,
                        double* tmp_v, int* tmp_p, int* tmp_g, int* cand, int* n_cand) {
  // tmp arrays hold two ping-pong halves of select_topk_tmp_elems(n_r, s) / 2
  int n = (n_r + TOPK_CHUNK - 1) / TOPK_CHUNK;
  const size_t half = (size_t)n * s;
  topk_pass1_kernel<<<n, 1024, 0, st>>>(d, pos, n_r, k, s, tmp_v, tmp_p, tmp_g); count_launches(1);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  int n_in = n * s, src = 0;
  while (true) {
    const int chunks = (n_in + TOPK_CHUNK - 1) / TOPK_CHUNK;
    const size_t so = src * half, dst = (1 - src) * half;
    if (chunks == 1) {
      topk_merge_kernel<<<1, 1024, 0, st>>>(tmp_v + so, tmp_p + so, tmp_g + so, n_in, s, nullptr,
                                            nullptr, nullptr, cand, n_cand); count_launches(1);
      return cudaGetLastError();
    }
    topk_merge_kernel<<<chunks, 1024, 0, st>>>(tmp_v + so, tmp_p + so, tmp_g + so, n_in, s,
                                               tmp_v + dst, tmp_p + dst, tmp_g + dst, nullptr,
                                               nullptr); count_launches(1);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    n_in = chunks * s;
    src = 1 - src;
  }
}

size_t select_topk_tmp_elems(int n_r, int s) {
  return 2 * (size_t)((n_r + TOPK_CHUNK - 1) / TOPK_CHUNK) * s;
}

int select_grid_blocks(int sm_count) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, select_steps_kernel, SEL_THREADS, 0);
  if (per_sm < 1) per_sm = 1;
  return sm_count * (per_sm > 1 ? 1 : per_sm);
}

cudaError_t select_steps(cudaStream_t st, int grid_blocks, int n_r, int steps, int kb, double* d,
                         int* pos, double* L, const double* W, const int* cand, int n_cand,
                         void* part, int* piv_order, double* margin, int* k_out) {
  StepParams p;
  p.n_r = n_r;
  p.steps = steps;
  p.kb = kb;
  p.d = d;
  p.pos = pos;
  p.L = L;
  p.W = W;
  p.cand = cand;
  p.n_cand = n_cand;
  p.part = static_cast<Part*>(part);
  p.piv_order = piv_order;
  p.margin = margin;
  p.k_out = k_out;
  void* args[] = {&p};
  count_launches(1);
  return cudaLaunchCooperativeKernel((const void*)select_steps_kernel, dim3(grid_blocks),
                                     dim3(SEL_THREADS), args, 0, st);
}

cudaError_t select_scatter_perm(cudaStream_t st, const int* pos, int n_r, int* perm) {
  scatter_perm_kernel<<<592, 256, 0, st>>>(pos, n_r, perm); count_launches(1);
  return cudaGetLastError();
}

size_t select_part_bytes(int grid_blocks) { return (size_t)3 * grid_blocks * sizeof(Part) + 64; }
int select_max_candidates() { return SEL_MAXS; }

}  // namespace lrgw_dev
