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
#include <algorithm>
#include <cfloat>
#include <cstdio>
#include <cstdlib>

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

// Order-preserving 64-bit key of a double (larger value -> larger key; NaN
// lowest, so a NaN residual is never picked).
__device__ __forceinline__ unsigned long long dkey(double v) {
  if (v != v) return 0ull;
  const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v));
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

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

// ---- top-(s+1) by (d desc, position asc): histogram select ------------------
// Four passes over the residuals (each a few microseconds at N_r ~ 1e5):
//   max:     the largest eligible key (eligible: position >= k);
//   hist:    4096 log-spaced bins below the max (17 leading bits of the key:
//            sign, exponent and 5 mantissa bits, ~3% wide);
//   compact: every CTA finds the boundary bin b* (first bin where the
//            cumulative count reaches s1); rows of bins < b* are in for sure,
//            rows of bin b* go to a boundary list;
//   final:   one CTA ranks the boundary rows by (d desc, position asc),
//            keeps the best s1 - |sure|, sorts the s1 winners and resets the
//            scratch for the next call. A boundary bin beyond BCAP rows
//            (massive exact ties) is merged in chunks by the same CTA.
struct Ent {
  double v;
  int pos, row;
};

__device__ __forceinline__ bool ent_better(const Ent& a, const Ent& b) { return better(a.v, a.pos, b.v, b.pos); }
__device__ __forceinline__ Ent ent_none() { return Ent{-DBL_MAX, INT_MAX, -1}; }

constexpr int TK_BINS = 4096;
constexpr int TK_BCAP = 4096;  // boundary rows ranked in one go
constexpr int TK_SCAP = 256;   // >= s1

struct TopkScratch {
  unsigned long long maxkey;
  unsigned sure_cnt, bnd_cnt;
  unsigned hist[TK_BINS];
  Ent sure[TK_SCAP];
  Ent bnd[TK_BCAP];
  // refinement of an over-full boundary bin (large grids): the next 12 key
  // bits of its rows, the sure count before it, and the refined boundary rows
  unsigned hist2[TK_BINS];
  unsigned sure0, bnd2_cnt, refine_ran;
  Ent bnd2[TK_BCAP];
};

__device__ __forceinline__ int tk_bin(unsigned long long key, unsigned ref) {
  const long long b = static_cast<long long>(ref) - static_cast<long long>(key >> 47);
  return b < 0 ? 0 : (b >= TK_BINS ? TK_BINS - 1 : static_cast<int>(b));
}

__global__ void topk_max_kernel(const double* d, const int* pos, int n_r, int k, const int* k_dev, TopkScratch* sc) {
  if (k_dev) k = *k_dev;
  unsigned long long m = 0;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n_r; r += gridDim.x * blockDim.x)
    if (pos[r] >= k) m = max(m, dkey(d[r]));
  // warp max of the 64-bit key: high words, then the low words of the lanes holding the top high word
  const unsigned hi = __reduce_max_sync(0xffffffffu, static_cast<unsigned>(m >> 32));
  const unsigned lo = __reduce_max_sync(0xffffffffu, static_cast<unsigned>(m >> 32) == hi ? static_cast<unsigned>(m) : 0u);
  if ((threadIdx.x & 31) == 0) atomicMax(&sc->maxkey, (static_cast<unsigned long long>(hi) << 32) | lo);
}

__global__ void topk_hist_kernel(const double* d, const int* pos, int n_r, int k, const int* k_dev, TopkScratch* sc) {
  __shared__ unsigned h[TK_BINS];
  if (k_dev) k = *k_dev;
  for (int i = threadIdx.x; i < TK_BINS; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const unsigned ref = static_cast<unsigned>(sc->maxkey >> 47);
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n_r; r += gridDim.x * blockDim.x)
    if (pos[r] >= k) atomicAdd(&h[tk_bin(dkey(d[r]), ref)], 1u);
  __syncthreads();
  for (int i = threadIdx.x; i < TK_BINS; i += blockDim.x)
    if (h[i]) atomicAdd(&sc->hist[i], h[i]);
}

// First bin whose cumulative count reaches s1 (TK_BINS if the total is smaller).
__device__ int tk_boundary(const unsigned* hist, int s1) {
  __shared__ unsigned part[32];
  __shared__ int bstar;
  constexpr int PER = TK_BINS / 256;  // blockDim.x == 256
  const int tid = threadIdx.x;
  unsigned loc[PER], sum = 0;
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    loc[q] = hist[tid * PER + q];
    sum += loc[q];
  }
  // inclusive scan of the per-thread sums
  unsigned x = sum;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const unsigned y = __shfl_up_sync(0xffffffffu, x, off);
    if ((tid & 31) >= off) x += y;
  }
  if ((tid & 31) == 31) part[tid >> 5] = x;
  if (tid == 0) bstar = TK_BINS;
  __syncthreads();
  unsigned before = 0;
  for (int w = 0; w < (tid >> 5); ++w) before += part[w];
  unsigned cum = before + x - sum;  // exclusive prefix of this thread's bins
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    if (cum < static_cast<unsigned>(s1) && cum + loc[q] >= static_cast<unsigned>(s1)) bstar = tid * PER + q;
    cum += loc[q];
  }
  __syncthreads();
  return bstar;
}

__global__ void __launch_bounds__(256) topk_compact_kernel(const double* d, const int* pos, int n_r, int k,
                                                           const int* k_dev, int s1, TopkScratch* sc) {
  if (k_dev) k = *k_dev;
  const int bstar = tk_boundary(sc->hist, s1);
  const unsigned ref = static_cast<unsigned>(sc->maxkey >> 47);
  const int lane = threadIdx.x & 31;
  const int n_it = (n_r + gridDim.x * blockDim.x - 1) / (gridDim.x * blockDim.x);
  for (int it = 0; it < n_it; ++it) {
    const int r = (it * gridDim.x + blockIdx.x) * blockDim.x + threadIdx.x;
    int bin = TK_BINS;
    double v = 0.0;
    int pr = 0;
    if (r < n_r) {
      pr = pos[r];
      if (pr >= k) {
        v = d[r];
        bin = tk_bin(dkey(v), ref);
      }
    }
    const bool sure = bin < bstar, bnd = bin == bstar && bin < TK_BINS;  // (TK_BINS: not eligible)
    const unsigned ms = __ballot_sync(0xffffffffu, sure), mb = __ballot_sync(0xffffffffu, bnd);
    unsigned bs = 0, bb = 0;
    if (lane == 0) {
      if (ms) bs = atomicAdd(&sc->sure_cnt, __popc(ms));
      if (mb) bb = atomicAdd(&sc->bnd_cnt, __popc(mb));
    }
    bs = __shfl_sync(0xffffffffu, bs, 0);
    bb = __shfl_sync(0xffffffffu, bb, 0);
    const unsigned below = (1u << lane) - 1u;
    if (sure) {
      const unsigned idx = bs + __popc(ms & below);
      if (idx < TK_SCAP) sc->sure[idx] = Ent{v, pr, r};
    }
    if (bnd) {
      const unsigned idx = bb + __popc(mb & below);
      if (idx < TK_BCAP) sc->bnd[idx] = Ent{v, pr, r};
    }
  }
}

// Sub-bin of a key inside its 17-bit bin (the next 12 bits; larger keys first).
__device__ __forceinline__ int tk_sub(unsigned long long key) {
  return (TK_BINS - 1) - static_cast<int>((key >> 35) & (TK_BINS - 1));
}

// Boundary bin over TK_BCAP rows: histogram its rows by sub-bin.
__global__ void __launch_bounds__(256) topk_hist2_kernel(const double* d, const int* pos, int n_r, int k,
                                                         const int* k_dev, int s1, TopkScratch* sc) {
  if (sc->bnd_cnt <= static_cast<unsigned>(TK_BCAP)) return;
  __shared__ unsigned h[TK_BINS];
  if (k_dev) k = *k_dev;
  const int bstar = tk_boundary(sc->hist, s1);
  for (int i = threadIdx.x; i < TK_BINS; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const unsigned ref = static_cast<unsigned>(sc->maxkey >> 47);
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n_r; r += gridDim.x * blockDim.x) {
    if (pos[r] < k) continue;
    const unsigned long long key = dkey(d[r]);
    if (tk_bin(key, ref) == bstar) atomicAdd(&h[tk_sub(key)], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < TK_BINS; i += blockDim.x)
    if (h[i]) atomicAdd(&sc->hist2[i], h[i]);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    sc->sure0 = sc->sure_cnt;
    sc->refine_ran = 1u;
  }
}

// ... and split it: sub-bins before the refined boundary join the sure rows,
// the boundary sub-bin becomes the (short) boundary list bnd2.
__global__ void __launch_bounds__(256) topk_compact2_kernel(const double* d, const int* pos, int n_r, int k,
                                                            const int* k_dev, int s1, TopkScratch* sc) {
  if (sc->bnd_cnt <= static_cast<unsigned>(TK_BCAP)) return;
  if (k_dev) k = *k_dev;
  const int bstar = tk_boundary(sc->hist, s1);
  const int b2 = tk_boundary(sc->hist2, s1 - static_cast<int>(sc->sure0));
  const unsigned ref = static_cast<unsigned>(sc->maxkey >> 47);
  const int lane = threadIdx.x & 31;
  const int n_it = (n_r + gridDim.x * blockDim.x - 1) / (gridDim.x * blockDim.x);
  for (int it = 0; it < n_it; ++it) {
    const int r = (it * gridDim.x + blockIdx.x) * blockDim.x + threadIdx.x;
    bool sure = false, bnd = false;
    double v = 0.0;
    int pr = 0;
    if (r < n_r) {
      pr = pos[r];
      if (pr >= k) {
        v = d[r];
        const unsigned long long key = dkey(v);
        if (tk_bin(key, ref) == bstar) {
          const int sb = tk_sub(key);
          sure = sb < b2;
          bnd = sb == b2;
        }
      }
    }
    const unsigned ms = __ballot_sync(0xffffffffu, sure), mb = __ballot_sync(0xffffffffu, bnd);
    unsigned bs = 0, bb = 0;
    if (lane == 0) {
      if (ms) bs = atomicAdd(&sc->sure_cnt, __popc(ms));
      if (mb) bb = atomicAdd(&sc->bnd2_cnt, __popc(mb));
    }
    bs = __shfl_sync(0xffffffffu, bs, 0);
    bb = __shfl_sync(0xffffffffu, bb, 0);
    const unsigned below = (1u << lane) - 1u;
    if (sure) {
      const unsigned idx = bs + __popc(ms & below);
      if (idx < TK_SCAP) sc->sure[idx] = Ent{v, pr, r};
    }
    if (bnd) {
      const unsigned idx = bb + __popc(mb & below);
      if (idx < TK_BCAP) sc->bnd2[idx] = Ent{v, pr, r};
    }
  }
}

// One CTA (TK_FINAL threads): rank, sort, write `out` (s1 entries), reset.
constexpr int TK_FINAL = 1024;
__global__ void __launch_bounds__(TK_FINAL) topk_final_kernel(const double* d, const int* pos, int n_r, int k,
                                                              const int* k_dev, int s1, TopkScratch* sc, Ent* out) {
  extern __shared__ __align__(16) unsigned char tk_smem[];
  Ent* cand = reinterpret_cast<Ent*>(tk_smem);  // up to TK_SCAP + TK_BCAP
  __shared__ Ent win[TK_SCAP];
  __shared__ int nwin_s;
  if (k_dev) k = *k_dev;
  const int tid = threadIdx.x;
  // a refined boundary (topk_compact2) replaces an over-full one; a
  // refinement that still overflows (massive exact ties) falls back to the
  // chunked scan below on the pass-1 sure rows only
  const bool ran = sc->refine_ran != 0u;
  const bool refined = ran && sc->bnd2_cnt > 0u && sc->bnd2_cnt <= static_cast<unsigned>(TK_BCAP);
  const int c0 = min(static_cast<int>(ran && !refined ? sc->sure0 : sc->sure_cnt), s1);
  const int nb = static_cast<int>(refined ? sc->bnd2_cnt : sc->bnd_cnt);
  const Ent* bl = refined ? sc->bnd2 : sc->bnd;
  const int need = min(s1 - c0, nb);
  for (int i = tid; i < c0; i += blockDim.x) win[i] = sc->sure[i];
  if (nb <= TK_BCAP) {
    for (int i = tid; i < nb; i += blockDim.x) cand[i] = bl[i];
    __syncthreads();
    for (int i = tid; i < nb; i += blockDim.x) {
      const Ent e = cand[i];
      int rank = 0;
      for (int q = 0; q < nb; ++q) rank += ent_better(cand[q], e) ? 1 : 0;
      if (rank < need) win[c0 + rank] = e;
    }
  } else {
    // massive ties in the boundary bin: stream its rows in grid order, chunk
    // by chunk (block-wide compaction), keeping the best `need` rows
    __shared__ int wsum[TK_FINAL / 32];
    __shared__ Ent keep[TK_SCAP];
    const unsigned ref = static_cast<unsigned>(sc->maxkey >> 47);
    const int bb = tk_bin(dkey(sc->bnd[0].v), ref);  // the boundary bin
    const int lane = tid & 31, wid = tid >> 5;
    int kept = 0;
    for (int r0 = 0; r0 < n_r;) {
      int fill = 0;
      for (; r0 < n_r && fill + TK_FINAL <= TK_BCAP; r0 += TK_FINAL) {
        const int r = r0 + tid;
        bool f = false;
        Ent e{};
        if (r < n_r) {
          const int pr = pos[r];
          if (pr >= k) {
            const double v = d[r];
            f = tk_bin(dkey(v), ref) == bb;
            e = Ent{v, pr, r};
          }
        }
        const unsigned m = __ballot_sync(0xffffffffu, f);
        if (lane == 0) wsum[wid] = __popc(m);
        __syncthreads();
        int before = 0, total = 0;
        for (int w = 0; w < TK_FINAL / 32; ++w) {
          before += (w < wid) ? wsum[w] : 0;
          total += wsum[w];
        }
        if (f) cand[kept + fill + before + __popc(m & ((1u << lane) - 1u))] = e;
        fill += total;
        __syncthreads();
      }
      const int m = kept + fill;
      for (int i = tid; i < m; i += blockDim.x) {
        const Ent e = cand[i];
        int rank = 0;
        for (int q = 0; q < m; ++q) rank += ent_better(cand[q], e) ? 1 : 0;
        if (rank < need) keep[rank] = e;
      }
      __syncthreads();
      kept = min(need, m);
      for (int i = tid; i < kept; i += blockDim.x) cand[i] = keep[i];
      __syncthreads();
    }
    for (int i = tid; i < need; i += blockDim.x) win[c0 + i] = cand[i];
  }
  if (tid == 0) nwin_s = c0 + need;
  __syncthreads();
  // sort the winners by rank and pad
  const int nw = nwin_s;
  for (int i = tid; i < nw; i += blockDim.x) {
    const Ent e = win[i];
    int rank = 0;
    for (int q = 0; q < nw; ++q) rank += ent_better(win[q], e) ? 1 : 0;
    out[rank] = e;
  }
  for (int i = nw + tid; i < s1; i += blockDim.x) out[i] = ent_none();
  // reset the scratch for the next call
  for (int i = tid; i < TK_BINS; i += blockDim.x) sc->hist[i] = 0;
  if (ran)
    for (int i = tid; i < TK_BINS; i += blockDim.x) sc->hist2[i] = 0;
  __syncthreads();
  if (tid == 0) {
    sc->maxkey = 0;
    sc->sure_cnt = 0;
    sc->bnd_cnt = 0;
    sc->bnd2_cnt = 0;
    sc->refine_ran = 0u;
  }
}

// ---- the certified candidate greedy (one CTA) -------------------------------
constexpr int CG_THREADS = 512;
constexpr int CG_WARPS = CG_THREADS / 32;
constexpr int CG_ROWS = 128 / CG_WARPS;  // candidate rows per warp
constexpr int CG_MAX = 128;              // candidates

struct CandParams {
  int n_r, s, steps, kb;
  int bmax, bround;  // accept at most bmax steps; a shorter run of >= bround steps keeps bround
  const Ent* top;       // s + 1 entries: candidates then the tau entry
  const double* wcc;    // s x s, ld s: W[C, C] (symmetric)
  int* pos;             // grid row -> position
  int* perm;            // position -> grid row
  double* xcol;         // s x s, ld s: X = L_sel^-1 column-major (b x b lower, zero above)
  double* xperm;        // optional: X again with its columns permuted inside 16-groups (panel4.cu)
  int* piv_order;       // [steps]
  double* margin;       // [steps] or nullptr
  int* b_out;           // number of accepted steps
  // device-driven block loop (all optional): the block start is read from
  // *kb_dev, the next block start kb + b written to *k_next
  const int* kb_dev;
  int* k_next;
  // optional: host-mapped pinned slot that receives b as soon as the run is
  // decided (before the triangular inverse), so the host can enqueue the
  // panel while this kernel finishes
  int* b_host;
};

__device__ __forceinline__ double pick8(const double (&x)[CG_ROWS], int r) {
  double v = x[0];
#pragma unroll
  for (int q = 1; q < CG_ROWS; ++q) v = (r == q) ? x[q] : v;
  return v;
}

// Pivot of the next step, published by the controller warp.
struct CandPivot {
  double v0, rinv;  // residual of the pivot and 1 / v0
  int i0, ok;
};

// Controller-warp argmax over the unused candidates (lane l: entries l + 32 c)
// by (d desc, position asc) — the reference's strict '>' scan — with three
// warp reductions (key high word, low word, position). sv (largest other
// residual) only when margins are requested.
__device__ __forceinline__ void cand_argmax(const double (&dj)[4], const int (&pj)[4], unsigned usedl, int lane,
                                            bool want_sv, double& v0, int& p0, int& i0, double& sv) {
  // usedl: bit c = entry lane + 32 c is taken / absent
  unsigned long long bk = 0;
  int bp = INT_MAX, bc = -1;
  double bv = -DBL_MAX;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const unsigned long long k = dkey(dj[c]);
    const bool take = !((usedl >> c) & 1u) && (bc < 0 || k > bk || (k == bk && pj[c] < bp));
    bk = take ? k : bk;
    bp = take ? pj[c] : bp;
    bv = take ? dj[c] : bv;
    bc = take ? c : bc;
  }
  const unsigned khi = bc >= 0 ? static_cast<unsigned>(bk >> 32) : 0u;
  const unsigned hi = __reduce_max_sync(0xffffffffu, khi);
  const unsigned lo = __reduce_max_sync(0xffffffffu, (bc >= 0 && khi == hi) ? static_cast<unsigned>(bk) : 0u);
  const bool top = bc >= 0 && bk == ((static_cast<unsigned long long>(hi) << 32) | lo);
  const int pm = static_cast<int>(__reduce_min_sync(0xffffffffu, top ? static_cast<unsigned>(bp) : 0x7fffffffu));
  const unsigned win = __ballot_sync(0xffffffffu, top && bp == pm);
  const int wl = win ? __ffs(win) - 1 : 0;
  const int wc = __shfl_sync(0xffffffffu, bc, wl);
  v0 = win ? __shfl_sync(0xffffffffu, bv, wl) : -DBL_MAX;
  i0 = win ? wl + 32 * wc : -1;
  p0 = pm;
  sv = -DBL_MAX;
  if (want_sv) {
#pragma unroll
    for (int c = 0; c < 4; ++c)
      if (!((usedl >> c) & 1u) && lane + 32 * c != i0) sv = fmax(sv, dj[c]);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) sv = fmax(sv, __shfl_xor_sync(0xffffffffu, sv, off));
  }
}

// X = L_sel^-1 for the b accepted steps (b <= 128) and M' = E X^T, after the
// greedy loop, in 32 x 32 blocks:
//   L_sel[i][m] = lcs[m][sel[i]] is first packed to `lsel` (lower, packed);
//   X (dense 128 x 128, reusing the lcs space; rows/cols >= b are identity);
//   the diagonal blocks are inverted by one warp each (lane = column,
//   unrolled forward substitution with reciprocal pivots), then block row I
//   takes X_Ik = -X_II sum_{m=k}^{I-1} L_Im X_mk (k < I) — all threads.
__device__ void cand_tri_inverse(double* lcs, double* lsel, const int* sel, int b, int s, double* xcol,
                                 double* xperm) {
  __shared__ double rdiag[CG_MAX];
  double* X = lcs;  // L_sel (packed lower in lsel) is the identity beyond b
  for (int idx = threadIdx.x; idx < b * b; idx += blockDim.x) {
    const int i = idx / b, m = idx % b;
    if (m <= i) lsel[i * (i + 1) / 2 + m] = lcs[m * CG_MAX + sel[i]];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < CG_MAX; i += blockDim.x) {
    const double d = i < b ? lsel[i * (i + 1) / 2 + i] : 1.0;
    rdiag[i] = d != 0.0 ? 1.0 / d : 0.0;
  }
  for (int idx = threadIdx.x; idx < CG_MAX * CG_MAX; idx += blockDim.x) X[idx] = 0.0;
  __syncthreads();
  const int nb = (b + 31) / 32;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  // diagonal blocks: warp I inverts block I (lane j: column 32 I + j)
  if (wid < nb) {
    const int o = 32 * wid;
    double x[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      double acc = (i == lane) ? 1.0 : 0.0;
      const int row = o + i;
      if (row < b) {  // rows >= b are identity rows (warp-uniform branch)
        const double* lr = lsel + row * (row + 1) / 2 + o;  // L_sel[row][o + m], m < i <= row - o
#pragma unroll
        for (int m = 0; m < i; ++m) acc = fma(-lr[m], x[m], acc);
      }
      x[i] = (i >= lane) ? acc * rdiag[row] : 0.0;
    }
#pragma unroll
    for (int i = 0; i < 32; ++i) X[(o + i) * CG_MAX + o + lane] = x[i];
  }
  __syncthreads();
  __shared__ double P[3 * 32 * 32];
  for (int I = 1; I < nb; ++I) {
    // P_k = sum_{m=32k}^{32I-1} L[32I + i][m] X[m][32k + j], k < I
    for (int idx = threadIdx.x; idx < I * 1024; idx += blockDim.x) {
      const int k = idx / 1024, i = (idx / 32) % 32, j = idx % 32;
      const int row = 32 * I + i, col = 32 * k + j;
      double acc = 0.0;
      if (row < b) {  // beyond b, L_sel rows are identity rows: zero left of the diagonal
        // X is lower triangular: X[m][col] = 0 for m < col; m < 32 I <= row < b
        const double* lr = lsel + row * (row + 1) / 2;
        for (int m = col; m < 32 * I; ++m) acc = fma(lr[m], X[m * CG_MAX + col], acc);
      }
      P[idx] = acc;
    }
    __syncthreads();
    // X_Ik = -X_II P_k
    for (int idx = threadIdx.x; idx < I * 1024; idx += blockDim.x) {
      const int k = idx / 1024, i = (idx / 32) % 32, j = idx % 32;
      double acc = 0.0;
      for (int q = 0; q <= i; ++q) acc = fma(X[(32 * I + i) * CG_MAX + 32 * I + q], P[k * 1024 + q * 32 + j], acc);
      X[(32 * I + i) * CG_MAX + 32 * k + j] = -acc;
    }
    __syncthreads();
  }
  // M'[sel[j]][i] = X[i][j] (i >= j); the rows of unselected candidates stay 0
  for (int idx = threadIdx.x; idx < b * b; idx += blockDim.x) {
    const int i = idx / b, j = idx % b;
    if (j <= i) {
      xcol[i + (size_t)j * s] = X[i * CG_MAX + j];
      if (xperm) {  // column j at 16 (j / 16) + 8 ((jl >> 1) & 1) + 2 (jl >> 2) + (jl & 1), jl = j % 16
        const int jl = j & 15, jm = (j & ~15) + 8 * ((jl >> 1) & 1) + 2 * (jl >> 2) + (jl & 1);
        xperm[i + (size_t)jm * s] = X[i * CG_MAX + j];
      }
    }
  }
}

// Register-resident candidate block W[C, C]: warp w owns the rows
// i = CG_ROWS w + r (lane l: columns l + 32 c, c < 4). Warp 0 is also the
// controller: it alone carries the residual diagonal, positions, grid rows and
// position slots of the candidates and picks each pivot. Per step t:
//   (after barrier B) every warp reads the published pivot; the owner warp
//      of row i0 publishes that row r (double-buffered);
//   barrier A;
//   controller: d_j -= r_j^2 / d_i0, next argmax, publish — the critical
//      path — then its own rows and the position bookkeeping;
//   other warps: w -= r_i (r_j / d_i0) on their rows; warp 1 records
//      l = r / sqrt(d_i0) (row t of the step history); warps 1.. extend
//      X = L_sel^-1 by row t (forward substitution, 4 lanes per column), so
//      M' = E X^T is complete when the loop ends;
//   barrier B.
__global__ void __launch_bounds__(CG_THREADS, 1) cand_greedy_kernel(CandParams p) {
  extern __shared__ __align__(16) double sm[];
  const int s = p.s, lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int kb = p.kb_dev ? *p.kb_dev : p.kb;
  const bool ctl = wid == 0;
  double* rowbuf = sm;                              // 2 x 128: published pivot rows
  double* lcs = rowbuf + 2 * CG_MAX;                // [t][j]: l of candidate j at step t; later X
  double* lsel = lcs + CG_MAX * CG_MAX;             // packed lower L_sel (after the loop)
  int* sel = reinterpret_cast<int*>(lsel + CG_MAX * (CG_MAX + 1) / 2);  // candidate of step t
  __shared__ CandPivot piv[2];
  __shared__ int rjs[CG_MAX];  // controller: candidate grid rows
  __shared__ int pss[CG_MAX];  // controller: perm[kb + j] (position slots of the block)
  __shared__ unsigned usedsh[4];  // candidates taken / absent before this step (bit l of word c: l + 32 c)
  // per-step position swaps and margins, applied to global memory after the
  // loop for the accepted prefix only
  __shared__ int rec_gp[CG_MAX], rec_occ[CG_MAX], rec_pp[CG_MAX];
  __shared__ double rec_mg[CG_MAX];

  for (int idx = threadIdx.x; idx < s * s; idx += blockDim.x) {
    p.xcol[idx] = 0.0;
    if (p.xperm) p.xperm[idx] = 0.0;
  }

  const double tau = p.top[s].row >= 0 ? p.top[s].v : -DBL_MAX;
  __shared__ int tmax_s;  // read from smem on the controller's path (keeps it out of the register budget)
  if (threadIdx.x == 0) tmax_s = min(min(s, p.bmax), p.steps - kb);
  const bool want_sv = p.margin != nullptr;

  // controller state (warp 0), entries j = lane + 32 c
  double dj[4];
  int pj[4];
  unsigned usedl = 0;  // bit c: entry lane + 32 c taken / absent
  double sv = -DBL_MAX;
  int ppos = 0;
  if (ctl) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int j = lane + 32 * c;
      const Ent e = j < s ? p.top[j] : ent_none();
      dj[c] = e.row >= 0 ? e.v : -DBL_MAX;
      pj[c] = e.row >= 0 ? e.pos : INT_MAX;
      rjs[j] = e.row;
      pss[j] = (j < s && kb + j < p.n_r) ? p.perm[kb + j] : -1;
      usedl |= (e.row < 0 ? 1u : 0u) << c;
      const unsigned m = __ballot_sync(0xffffffffu, e.row < 0);
      if (lane == 0) usedsh[c] = m;
    }
    double v0;
    int i0;
    cand_argmax(dj, pj, usedl, lane, want_sv, v0, ppos, i0, sv);
    // the first step of a block is the exact argmax (C is sorted by the pivot rule)
    if (lane == 0) piv[0] = CandPivot{v0, v0 > 0.0 ? 1.0 / v0 : 0.0, i0, (0 < min(s, p.steps - kb) && i0 >= 0) ? 1 : 0};
  }

  const int base = CG_ROWS * wid;
  double w[CG_ROWS][4];
#pragma unroll
  for (int r = 0; r < CG_ROWS; ++r) {
    const int i = base + r;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int j = lane + 32 * c;
      w[r][c] = (i < s && j < s) ? p.wcc[j + (size_t)i * s] : 0.0;
    }
  }
  __syncthreads();

  int t = 0;
  for (;; ++t) {
    const CandPivot pv = piv[t & 1];
    if (!pv.ok) break;  // uniform
    const int i0 = pv.i0;
    double* rb = rowbuf + (t & 1) * CG_MAX;
    if (wid == i0 / CG_ROWS) {
      const int r0 = i0 % CG_ROWS;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        double x[CG_ROWS];
#pragma unroll
        for (int r = 0; r < CG_ROWS; ++r) x[r] = w[r][c];
        rb[lane + 32 * c] = pick8(x, r0);
      }
    }
    __syncthreads();
    if (ctl) {
      // ---- critical path: downdate d, pick and publish the next pivot ----
      const int k = kb + t;
      const int occ = pss[t];  // perm[k] before the swap
      const int piv_pos = ppos;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int j = lane + 32 * c;
        const double r = rb[j];
        const bool live = !((usedl >> c) & 1u) && j != i0;
        dj[c] = live ? fma(-r, r * pv.rinv, dj[c]) : dj[c];
        pj[c] = (j == i0) ? k : ((rjs[j] == occ) ? piv_pos : pj[c]);
      }
      usedl |= (lane == (i0 & 31) ? 1u : 0u) << (i0 >> 5);
      const double svp = sv;
      double v1;
      int i1;
      cand_argmax(dj, pj, usedl, lane, want_sv, v1, ppos, i1, sv);
      if (lane == 0)
        piv[(t + 1) & 1] = CandPivot{v1, v1 > 0.0 ? 1.0 / v1 : 0.0, i1,
                                     (t + 1 < tmax_s && i1 >= 0 && v1 > tau) ? 1 : 0};
      if (lane == 0) {
        const int gp = rjs[i0];  // pivot grid row
        rec_gp[t] = gp;
        rec_occ[t] = occ;
        rec_pp[t] = piv_pos;
        sel[t] = i0;
        // position slots: perm[ppos] = occ, then perm[k] = gp
        if (piv_pos - kb < CG_MAX) pss[piv_pos - kb] = occ;
        pss[t] = gp;
        usedsh[i0 >> 5] |= 1u << (i0 & 31);  // only bit i0 changes: workers exclude it already
        rec_mg[t] = pv.v0 > 0.0 ? (pv.v0 - fmax(svp, tau)) / pv.v0 : 0.0;
      }
    }
    // ---- eliminate: w -= r_i r_j / d_i0 (row / column i0 are never read
    // again; rows already taken only see round-off-sized entries) ----
    {
      const unsigned um = (usedsh[base >> 5] >> (base & 31)) | (i0 / CG_ROWS == wid ? 1u << (i0 % CG_ROWS) : 0u);
      if ((um & ((1u << CG_ROWS) - 1)) != (1u << CG_ROWS) - 1) {
        double gj[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int j = lane + 32 * c;
          gj[c] = (j == i0) ? 0.0 : rb[j] * pv.rinv;
        }
#pragma unroll
        for (int r = 0; r < CG_ROWS; ++r) {
          if ((um >> r) & 1u) continue;  // taken rows are never read again (warp-uniform)
          const double ri = rb[base + r];
#pragma unroll
          for (int c = 0; c < 4; ++c) w[r][c] = fma(-ri, gj[c], w[r][c]);
        }
      }
    }
    if (wid == 1) {
      // step history: l_j = r_j / sqrt(d_i0), l_i0 = sqrt(d_i0) (entries of
      // rows already taken are never read: L_sel only reads rows sel[t'], t' > t)
      const double lpiv = pv.v0 > 0.0 ? sqrt(pv.v0) : 0.0;
      const double inv = lpiv > 0.0 ? 1.0 / lpiv : 0.0;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int j = lane + 32 * c;
        lcs[t * CG_MAX + j] = (j == i0) ? lpiv : rb[j] * inv;
      }
    }
    __syncthreads();
  }
  // the accepted prefix: every step of the run is certified, so any prefix is
  // exactly the reference's next pivots; a run the certificate stopped short
  // of bmax keeps a tile-friendly bround steps (the rest are re-found next
  // block)
  const int b = (t < tmax_s && p.bround > 0 && t >= p.bround) ? p.bround : t;
  if (threadIdx.x == 0 && p.b_host) {
    *reinterpret_cast<volatile int*>(p.b_host) = b;
    __threadfence_system();
  }
  if (threadIdx.x == 0) {
    for (int q = 0; q < b; ++q) {  // the swaps in step order
      const int k = kb + q, gp = rec_gp[q], occ = rec_occ[q], pp = rec_pp[q];
      p.perm[k] = gp;
      p.perm[pp] = occ;
      p.pos[gp] = k;
      p.pos[occ] = pp;
      p.piv_order[k] = gp;
      if (want_sv) p.margin[k] = rec_mg[q];
    }
  }
  cand_tri_inverse(lcs, lsel, sel, b, s, p.xcol, p.xperm);
  if (threadIdx.x == 0) {
    p.b_out[0] = b;
    p.b_out[1] = kb + b;  // next block start, consumed on the device
    if (p.k_next) *p.k_next = kb + b;
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

size_t select_topk_tmp_bytes(int, int) { return sizeof(TopkScratch) + 64; }

size_t select_ent_bytes() { return sizeof(Ent); }

cudaError_t select_init(cudaStream_t st, const double* a, long long lda, int n1, const double* b,
                        long long ldb, int n2, int n_r, double* d, int* pos, int* perm) {
  init_diag_kernel<<<592, 256, 0, st>>>(a, lda, n1, b, ldb, n2, n_r, d, pos, perm); count_launches(1);
  return cudaGetLastError();
}

cudaError_t select_topk_reset(cudaStream_t st, void* tmp) {
  return cudaMemsetAsync(tmp, 0, sizeof(TopkScratch), st);
}

cudaError_t select_topk(cudaStream_t st, const double* d, const int* pos, int n_r, int k, int s1, void* tmp,
                        void* out, const int* k_dev) {
  if (s1 > TK_SCAP) return cudaErrorInvalidValue;
  TopkScratch* sc = static_cast<TopkScratch*>(tmp);
  const int grid = std::max(1, std::min(296, (n_r + 255) / 256));
  topk_max_kernel<<<grid, 256, 0, st>>>(d, pos, n_r, k, k_dev, sc); count_launches(1);
  topk_hist_kernel<<<grid, 256, 0, st>>>(d, pos, n_r, k, k_dev, sc); count_launches(1);
  topk_compact_kernel<<<grid, 256, 0, st>>>(d, pos, n_r, k, k_dev, s1, sc); count_launches(1);
  if (n_r > 200000) {  // a boundary bin over TK_BCAP rows is refined on the device (the kernels exit otherwise)
    topk_hist2_kernel<<<grid, 256, 0, st>>>(d, pos, n_r, k, k_dev, s1, sc);
    topk_compact2_kernel<<<grid, 256, 0, st>>>(d, pos, n_r, k, k_dev, s1, sc);
    count_launches(2);
  }
  const size_t smem = (TK_SCAP + TK_BCAP) * sizeof(Ent);
  cudaError_t e = cudaFuncSetAttribute(topk_final_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  topk_final_kernel<<<1, TK_FINAL, smem, st>>>(d, pos, n_r, k, k_dev, s1, sc, static_cast<Ent*>(out));
  count_launches(1);
  return cudaGetLastError();
}

size_t select_cand_smem_bytes(int) {
  return (2 * CG_MAX + CG_MAX * CG_MAX + CG_MAX * (CG_MAX + 1) / 2) * sizeof(double) + CG_MAX * sizeof(int) + 16;
}

int select_max_candidates() { return CG_MAX; }

// Measured on the Si512 selection (profiles/r02/select_widths_si512.txt): the
// tall-skinny engines run 0.85-0.90 of the DMMA peak at an exact 96-wide
// column tile and 0.74-0.80 at the 100-127 widths a 128-candidate block
// certifies (112 / 128 tiles with dead columns), so a block accepts the first
// 96 certified pivots — 80 below 2e5 grid rows, where the 96-wide tiles'
// last wave is mostly empty (profiles/r02/select_accept.txt: Si64 10.9 ->
// 10.45 ms, Si216 255 -> 234 ms, Si512 3192 -> 2868 ms). LRGW_SELECT_ACCEPT
// overrides (0 = all certified steps).
// With the fused TMA panel (panel4.cu, N <= 112) the large grids take 112
// (Si216 select 223.2 -> 218.3 ms; Si64 keeps 80: 9.39 vs 9.62-9.70 ms,
// profiles/r02/sweep_accept_panel4.txt).
int select_accept_cap(int s, int n_r, bool panel_tma) {
  static const int env = getenv("LRGW_SELECT_ACCEPT") ? atoi(getenv("LRGW_SELECT_ACCEPT")) : -1;
  const int cap = env >= 0 ? env : (n_r < 200000 ? 80 : panel_tma ? 112 : 96);
  return cap > 0 ? std::min(cap, s) : s;
}
int select_accept_round() {
  static const int r = getenv("LRGW_SELECT_ROUND") ? atoi(getenv("LRGW_SELECT_ROUND")) : 80;
  return std::max(0, r);
}

cudaError_t select_cand_greedy(cudaStream_t st, int n_r, int s, int steps, int kb, const void* top, const double* wcc,
                               int* pos, int* perm, double* xcol, int* piv_order, double* margin, int* b_out,
                               int bmax, int bround, const int* kb_dev, int* k_next, double* xperm, int* b_host) {
  const Ent* tp = static_cast<const Ent*>(top);
  CandParams p{n_r,  s,    steps,     kb,     std::max(1, bmax), bround, tp,     wcc,   pos,
               perm, xcol, xperm, piv_order, margin,            b_out,  kb_dev, k_next, b_host};
  const size_t smem = select_cand_smem_bytes(s);
  cudaError_t e = cudaFuncSetAttribute(cand_greedy_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  cand_greedy_kernel<<<1, CG_THREADS, smem, st>>>(p); count_launches(1);
  return cudaGetLastError();
}

// W[C, C] -= Lr Lr^T over the k = *k_dev pivots so far (Lr: s x k, ld ldl):
// WCC_SPLITS k-chunks into partials, then one fixed-order reduction (the same
// sum for every run: the greedy's pivots must not depend on scheduling).
constexpr int WCC_SPLITS = 16;
__global__ void __launch_bounds__(256) wcc_lsub_partial_kernel(const double* lr, long long ldl, int s, const int* k_dev,
                                                               double* part) {
  const int k = *k_dev;
  const int ch = ((k + WCC_SPLITS - 1) / WCC_SPLITS + 7) / 8 * 8;
  const int k0 = blockIdx.y * ch, k1 = min(k, k0 + ch);
  const int ti = blockIdx.x % 4, tj = blockIdx.x / 4;  // 32 x 32 tile of the 128 x 128 block
  const int i = 32 * ti + 2 * (threadIdx.x % 16), j = 32 * tj + 2 * (threadIdx.x / 16);
  double a00 = 0.0, a01 = 0.0, a10 = 0.0, a11 = 0.0;
  if (i < s && j < s) {
    for (int kk = k0; kk < k1; ++kk) {
      const double* col = lr + (long long)kk * ldl;
      const double x0 = col[i], x1 = i + 1 < s ? col[i + 1] : 0.0;
      const double y0 = col[j], y1 = j + 1 < s ? col[j + 1] : 0.0;
      a00 = fma(x0, y0, a00);
      a01 = fma(x0, y1, a01);
      a10 = fma(x1, y0, a10);
      a11 = fma(x1, y1, a11);
    }
  }
  double* out = part + (size_t)blockIdx.y * CG_MAX * CG_MAX;
  out[i + j * CG_MAX] = a00;
  out[i + 1 + j * CG_MAX] = a10;
  out[i + (j + 1) * CG_MAX] = a01;
  out[i + 1 + (j + 1) * CG_MAX] = a11;
}

__global__ void wcc_lsub_reduce_kernel(double* wcc, int s, const double* part) {
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < s * s; idx += gridDim.x * blockDim.x) {
    const int i = idx % s, j = idx / s;
    double acc = 0.0;
    for (int q = 0; q < WCC_SPLITS; ++q) acc += part[(size_t)q * CG_MAX * CG_MAX + i + j * CG_MAX];
    wcc[i + (size_t)j * s] -= acc;
  }
}

size_t select_wcc_work_elems() { return (size_t)WCC_SPLITS * CG_MAX * CG_MAX; }

cudaError_t select_wcc_lsub(cudaStream_t st, const double* lr, long long ldl, int s, const int* k_dev, double* wcc,
                            double* work) {
  if (s > CG_MAX) return cudaErrorInvalidValue;
  wcc_lsub_partial_kernel<<<dim3(16, WCC_SPLITS), 256, 0, st>>>(lr, ldl, s, k_dev, work);
  wcc_lsub_reduce_kernel<<<64, 256, 0, st>>>(wcc, s, work);
  count_launches(2);
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
