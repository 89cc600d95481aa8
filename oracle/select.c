/* oracle/select.c — TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * CPU restatement of the reference ISDF point selection
 *   select_interpolation_points (isdf.hpp:95-112) -> qrcp (linalg.hpp:26-111)
 * as a matrix-free greedy pivoted Cholesky on the Hadamard Gram
 *   G(r,s) = (A A^T)(r,s) * (B B^T)(r,s) = (Z^T Z)(r,s),
 * where Z = pair_matrix_transposed(A, B) (isdf.hpp:72-88). In exact arithmetic
 * the residual column norms of Householder QRCP on Z equal the residual
 * diagonal of pivoted Cholesky on G, so the greedy pivot sequence is the same.
 *
 * Reference semantics mirrored:
 *  - pivot = argmax residual over the remaining POSITIONS with strict '>'
 *    (linalg.hpp:45-47): ties go to the lowest current position, where
 *    positions follow the perm[step] <-> perm[p] swap (linalg.hpp:48-53);
 *  - min(N1*N2, N_r) elimination steps (linalg.hpp:29, 44); when N_mu exceeds
 *    that, the tail of the swapped perm is returned as-is (isdf.hpp:109);
 *  - the first N_mu entries of perm are sorted ascending (isdf.hpp:110).
 * Not mirrored (documented in DESIGN.md): the norm-recompute branch
 * (linalg.hpp:83-87); `recompute_events` counts the steps where it would fire
 * so tests can assert it never does on parity inputs.
 *
 * Built by oracle/Makefile into _ref/liboracle_select.so (OpenMP over rows).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static int cmp_int(const void* a, const void* b) {
  int x = *(const int*)a, y = *(const int*)b;
  return (x > y) - (x < y);
}

/* Returns 0 on success, 1 on invalid input (isdf.hpp:99-101), 9 on OOM.
 * margins (optional, length steps): (d_max - d_second) / d_max per step.
 * pivots_in_order (optional, length min(n_mu, steps)): unsorted pivot order. */
int oracle_select_points(const double* a, const double* b, int n_r, int n1,
                         int n2, int n_mu, int* pts, double* margins,
                         int* pivots_in_order, int* recompute_events) {
  if (n_mu > n_r || n_mu < 1 || n_r < 1 || n1 < 1 || n2 < 1) return 1;
  const long long m = (long long)n1 * n2;
  const int k = (int)(m < n_r ? m : n_r);
  const int steps = n_mu < k ? n_mu : k;

  double* d = (double*)malloc(sizeof(double) * n_r);
  double* d0 = (double*)malloc(sizeof(double) * n_r);
  int* perm = (int*)malloc(sizeof(int) * n_r);
  int* pos = (int*)malloc(sizeof(int) * n_r);
  /* row-major copies: each grid row's orbital values and L row are contiguous
   * (the same sums in the same order as a column-major sweep, just cache-
   * friendly on the host) */
  const int ldl = steps > 0 ? steps : 1;
  double* L = (double*)malloc(sizeof(double) * (size_t)n_r * ldl);
  double* ar = (double*)malloc(sizeof(double) * (size_t)n_r * n1);
  double* br = (double*)malloc(sizeof(double) * (size_t)n_r * n2);
  double* ap = (double*)malloc(sizeof(double) * n1);
  double* bp = (double*)malloc(sizeof(double) * n2);
  if (!d || !d0 || !perm || !pos || !L || !ap || !bp || !ar || !br) {
    free(d); free(d0); free(perm); free(pos); free(L); free(ap); free(bp); free(ar); free(br);
    return 9;
  }
  int events = 0;

#pragma omp parallel for schedule(static)
  for (int g = 0; g < n_r; ++g) {
    double sa = 0.0, sb = 0.0;
    double* arg = ar + (size_t)g * n1;
    double* brg = br + (size_t)g * n2;
    for (int i = 0; i < n1; ++i) arg[i] = a[(size_t)i * n_r + g];
    for (int j = 0; j < n2; ++j) brg[j] = b[(size_t)j * n_r + g];
    for (int i = 0; i < n1; ++i) sa += arg[i] * arg[i];
    for (int j = 0; j < n2; ++j) sb += brg[j] * brg[j];
    d[g] = d0[g] = sa * sb;
    perm[g] = g;
    pos[g] = g;
  }

  for (int s = 0; s < steps; ++s) {
    /* argmax over positions s..n_r-1, strict '>' => lowest position on ties */
    int p = s;
    double best = d[perm[s]], second = -INFINITY;
    for (int j = s + 1; j < n_r; ++j) {
      double v = d[perm[j]];
      if (v > best) {
        second = best;
        best = v;
        p = j;
      } else if (v > second) {
        second = v;
      }
    }
    if (margins) margins[s] = best > 0.0 ? (best - second) / best : 0.0;
    if (p != s) {
      int t = perm[s];
      perm[s] = perm[p];
      perm[p] = t;
      pos[perm[s]] = s;
      pos[perm[p]] = p;
    }
    const int gp = perm[s];
    if (pivots_in_order) pivots_in_order[s] = gp;
    const double dp = d[gp];
    if (!(dp > 0.0)) {
      /* exhausted: Householder with alpha == 0 leaves the trailing columns
       * untouched (linalg.hpp:60-61) */
      for (int g = 0; g < n_r; ++g) L[(size_t)g * ldl + s] = 0.0;
      continue;
    }
    const double inv = 1.0 / sqrt(dp);
    for (int i = 0; i < n1; ++i) ap[i] = ar[(size_t)gp * n1 + i];
    for (int j = 0; j < n2; ++j) bp[j] = br[(size_t)gp * n2 + j];
    const double* Lp = L + (size_t)gp * ldl;
    int ev = 0;
#pragma omp parallel for schedule(static) reduction(+ : ev)
    for (int g = 0; g < n_r; ++g) {
      double* Lg = L + (size_t)g * ldl;
      if (pos[g] < s) { Lg[s] = 0.0; continue; }
      const double* arg = ar + (size_t)g * n1;
      const double* brg = br + (size_t)g * n2;
      double sa = 0.0, sb = 0.0;
      for (int i = 0; i < n1; ++i) sa += arg[i] * ap[i];
      for (int j = 0; j < n2; ++j) sb += brg[j] * bp[j];
      double c = sa * sb;
      for (int t = 0; t < s; ++t) c -= Lg[t] * Lp[t];
      double l = (g == gp) ? sqrt(dp) : c * inv;
      Lg[s] = l;
      if (g != gp) {
        d[g] -= l * l;
        if (d[g] < 1e-12 * d0[g] || d[g] < 0.0) ++ev;
      }
    }
    events += ev;
  }

  for (int i = 0; i < n_mu; ++i) pts[i] = perm[i];
  qsort(pts, (size_t)n_mu, sizeof(int), cmp_int);
  if (recompute_events) *recompute_events = events;
  free(d); free(d0); free(perm); free(pos); free(L); free(ap); free(bp); free(ar); free(br);
  return 0;
}
