// fft.cu — the batched 3-D D2Z of Theta (model.hpp:208-223: the Coulomb
// application's forward transform, cuFFT's convention X[k] = sum x[n]
// e^{-2 pi i n.k / N}, half spectrum along the fastest axis) in two passes
// over HBM instead of cuFFT's three:
//   pass 1 (one CTA per (i2, column) plane): the 2-D R2C over (i1, i0) in
//          shared memory — rows packed pairwise into complex FFTs
//          (z = x_2q + i x_2q+1, split by conjugate symmetry), then the
//          column transforms along i1 — written to the output in place of
//          the final spectrum;
//   pass 2 (one CTA per 32 (k1, k0) pencils of a column): the transforms
//          along i2, in place.
// Every 1-D transform is a mixed-radix (2, 3, 4, 5) Stockham autosort in
// shared memory with a per-CTA twiddle table W[k] = e^{-2 pi i k / n}.
// Both passes are persistent (one or more CTAs per SM) and stream their next
// unit in with cp.async while the current one is transformed.
// Traffic: read Theta once, write + read + write the spectrum (2x the
// algorithmic bytes against cuFFT's ~3x). Grids other than the cubic path
// sizes return cudaErrorNotSupported and stay on the cuFFT leaf.
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace lrgw_dev {

namespace {

constexpr int FFT_MAXN = 128;
constexpr int FFT_MAXR = 8;
constexpr int FFT_THREADS = 256;
constexpr int FFT_G = 32;  // pencils per CTA in pass 2

struct FftParams {
  int n0, n1, n2, h;  // h = n0 / 2 + 1
  long long nh;       // complex entries per column (h n1 n2)
  const double* x;
  long long ldx;
  double2* y;
  const double2* tw0;  // twiddle tables of n0, n1, n2
  const double2* tw1;
  const double2* tw2;
};

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }

// radix-R forward DFT in place (R = 2, 3, 4, 5)
template <int R>
__device__ __forceinline__ void dft(double2 (&v)[5]) {
  if constexpr (R == 2) {
    const double2 a = v[0], b = v[1];
    v[0] = cadd(a, b);
    v[1] = csub(a, b);
  } else if constexpr (R == 3) {
    constexpr double c = 0.86602540378443864676;  // sin(2 pi / 3)
    const double2 t = cadd(v[1], v[2]), d = csub(v[1], v[2]);
    const double2 m = make_double2(v[0].x - 0.5 * t.x, v[0].y - 0.5 * t.y);
    v[0] = cadd(v[0], t);
    v[1] = make_double2(m.x + c * d.y, m.y - c * d.x);
    v[2] = make_double2(m.x - c * d.y, m.y + c * d.x);
  } else if constexpr (R == 4) {
    const double2 a = cadd(v[0], v[2]), b = csub(v[0], v[2]), c = cadd(v[1], v[3]), d = csub(v[1], v[3]);
    v[0] = cadd(a, c);
    v[2] = csub(a, c);
    v[1] = make_double2(b.x + d.y, b.y - d.x);  // b - i d
    v[3] = make_double2(b.x - d.y, b.y + d.x);  // b + i d
  } else {
    constexpr double c1 = 0.30901699437494742410, c2 = -0.80901699437494742410;  // cos(2 pi / 5), cos(4 pi / 5)
    constexpr double s1 = 0.95105651629515357212, s2 = 0.58778525229247312917;   // sin(2 pi / 5), sin(4 pi / 5)
    const double2 t1 = cadd(v[1], v[4]), t2 = cadd(v[2], v[3]), d1 = csub(v[1], v[4]), d2 = csub(v[2], v[3]);
    const double2 a1 = make_double2(v[0].x + c1 * t1.x + c2 * t2.x, v[0].y + c1 * t1.y + c2 * t2.y);
    const double2 a2 = make_double2(v[0].x + c2 * t1.x + c1 * t2.x, v[0].y + c2 * t1.y + c1 * t2.y);
    const double2 b1 = make_double2(s1 * d1.x + s2 * d2.x, s1 * d1.y + s2 * d2.y);
    const double2 b2 = make_double2(s2 * d1.x - s1 * d2.x, s2 * d1.y - s1 * d2.y);
    v[0] = cadd(v[0], cadd(t1, t2));
    v[1] = make_double2(a1.x + b1.y, a1.y - b1.x);
    v[4] = make_double2(a1.x - b1.y, a1.y + b1.x);
    v[2] = make_double2(a2.x + b2.y, a2.y - b2.x);
    v[3] = make_double2(a2.x - b2.y, a2.y + b2.x);
  }
}

// ---- compile-time plans: every index division below is by a constant ----
struct CPlan {
  int nr;
  int rad[FFT_MAXR];
};

constexpr CPlan cplan(int n) {
  CPlan p{0, {0, 0, 0, 0, 0, 0, 0, 0}};
  int m = n;
  while (m > 1 && p.nr < FFT_MAXR) {
    const int r = m % 4 == 0 ? 4 : m % 2 == 0 ? 2 : m % 3 == 0 ? 3 : m % 5 == 0 ? 5 : 0;
    if (r == 0) return CPlan{-1, {0, 0, 0, 0, 0, 0, 0, 0}};
    p.rad[p.nr++] = r;
    m /= r;
  }
  return m == 1 ? p : CPlan{-1, {0, 0, 0, 0, 0, 0, 0, 0}};
}

// One radix-R Stockham stage over T transforms of length N (element e of
// transform t at buf[t TS + e ES]), NS = product of the earlier radices.
template <int R, int N, int NS, int T, int TS, int ES>
__device__ __forceinline__ void stage(const double2* src, double2* dst, const double2* W) {
  constexpr int NB = N / R, STEP = N / (NS * R);
  for (int idx = threadIdx.x; idx < T * NB; idx += FFT_THREADS) {
    // consecutive threads walk the unit-stride axis (conflict-free shared memory)
    const int t = TS == 1 ? idx % T : idx / NB;
    const int j = TS == 1 ? idx / T : idx - t * NB;
    const double2* s = src + t * TS;
    double2* d = dst + t * TS;
    const int jm = j % NS;
    double2 v[5];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = s[(j + r * NB) * ES];
#pragma unroll
    for (int r = 1; r < R; ++r) v[r] = cmul(v[r], W[jm * r * STEP]);
    dft<R>(v);
    const int o = (j / NS) * NS * R + jm;
#pragma unroll
    for (int r = 0; r < R; ++r) d[(o + r * NS) * ES] = v[r];
  }
}

template <int N, int T, int TS, int ES, int Q = 0, int NS = 1>
__device__ __forceinline__ double2* stockham(double2* a, double2* b, const double2* W) {
  constexpr CPlan pl = cplan(N);
  if constexpr (Q >= pl.nr) {
    return a;
  } else {
    constexpr int R = pl.rad[Q];
    stage<R, N, NS, T, TS, ES>(a, b, W);
    __syncthreads();
    return stockham<N, T, TS, ES, Q + 1, NS * R>(b, a, W);
  }
}

// W[k] = e^{-2 pi i k / n} into shared memory from the global table of the size
__device__ __forceinline__ void twiddles(double2* W, const double2* tab, int n) {
  for (int k = threadIdx.x; k < n; k += blockDim.x) W[k] = __ldg(tab + k);
}

__global__ void twiddle_table_kernel(double2* tab, int n) {
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    double s, c;
    sincospi(2.0 * k / n, &s, &c);
    tab[k] = make_double2(c, -s);
  }
}

template <int N0, int N1>
constexpr int planes_cap() {
  return (N1 / 2) * N0 > N1 * (N0 / 2 + 1) ? (N1 / 2) * N0 : N1 * (N0 / 2 + 1);
}

// pass 1 (persistent): CTA b takes planes u = b, b + grid, ... (u = i2 + n2
// column); the next plane's reals stream into a staging buffer (cp.async)
// while the current one is transformed.
template <int N0, int N1>
constexpr size_t planes_smem(bool stage) {
  return (size_t)(2 * planes_cap<N0, N1>() + 2 * FFT_MAXN) * sizeof(double2) +
         (stage ? (size_t)N0 * N1 * sizeof(double) : 0);
}
// the staging buffer when it fits next to the two work buffers (not at 96^2)
template <int N0, int N1>
constexpr bool planes_stage() {
  return planes_smem<N0, N1>(true) <= 200 * 1024;
}

template <int N0, int N1>
__global__ void __launch_bounds__(FFT_THREADS) fft_planes_kernel(FftParams p, int units) {
  extern __shared__ __align__(16) double2 sb[];
  constexpr int H = N0 / 2 + 1, CAP = planes_cap<N0, N1>(), NR = N0 * N1;
  constexpr bool STAGE = planes_stage<N0, N1>();
  double2* A = sb;
  double2* B = A + CAP;
  double2* W0 = B + CAP;
  double2* W1 = W0 + FFT_MAXN;
  double* S = reinterpret_cast<double*>(W1 + FFT_MAXN);  // NR reals
  twiddles(W0, p.tw0, N0);
  twiddles(W1, p.tw1, N1);
  auto src = [&](int u) { return p.x + (long long)(u / p.n2) * p.ldx + (long long)(u % p.n2) * NR; };
  auto prefetch = [&](int u) {
    if (STAGE && u < units) {
      const double* xp = src(u);
      for (int c = threadIdx.x; c < NR / 2; c += FFT_THREADS) cp_async16(S + 2 * c, xp + 2 * c, true);
    }
    cp_async_commit();
  };
  prefetch(blockIdx.x);
  for (int u = blockIdx.x; u < units; u += gridDim.x) {
    cp_async_wait<0>();
    __syncthreads();
    // rows 2q and 2q + 1 packed into one complex row q (length N0)
    const double* in = STAGE ? S : src(u);
    for (int idx = threadIdx.x; idx < (N1 / 2) * N0; idx += FFT_THREADS) {
      const int q = idx / N0, i0 = idx - q * N0;
      A[idx] = make_double2(in[(2 * q) * N0 + i0], in[(2 * q + 1) * N0 + i0]);
    }
    __syncthreads();
    prefetch(u + gridDim.x);
    double2* Z = stockham<N0, N1 / 2, N0, 1>(A, B, W0);
    double2* Y = Z == A ? B : A;
    // split: X_2q[k] = (Z[k] + conj Z[-k]) / 2, X_2q+1[k] = (Z[k] - conj Z[-k]) / 2i, k < H
    for (int idx = threadIdx.x; idx < (N1 / 2) * H; idx += FFT_THREADS) {
      const int q = idx / H, k = idx - q * H;
      const double2 z = Z[q * N0 + k], zr = Z[q * N0 + (k == 0 ? 0 : N0 - k)];
      Y[(2 * q) * H + k] = make_double2(0.5 * (z.x + zr.x), 0.5 * (z.y - zr.y));
      Y[(2 * q + 1) * H + k] = make_double2(0.5 * (z.y + zr.y), -0.5 * (z.x - zr.x));
    }
    __syncthreads();
    // along i1: H transforms (offset k0), element stride H
    double2* R = stockham<N1, H, 1, H>(Y, Z, W1);
    double2* yp = p.y + (long long)(u / p.n2) * p.nh + (long long)(u % p.n2) * N1 * H;
    for (int idx = threadIdx.x; idx < N1 * H; idx += FFT_THREADS) yp[idx] = R[idx];
  }
  cp_async_wait<0>();
}

// pass 2 (persistent): CTA b takes pencil groups u = b, b + grid, ... (FFT_G
// pencils of one column each), the next group prefetched like pass 1.
template <int N2>
__global__ void __launch_bounds__(FFT_THREADS) fft_pencils_kernel(FftParams p, int units, int gpc) {
  extern __shared__ __align__(16) double2 sb[];
  const int P = p.n1 * p.h;
  double2* A = sb;
  double2* B = A + FFT_G * N2;
  double2* W2 = B + FFT_G * N2;
  double2* S = W2 + FFT_MAXN;  // FFT_G N2 staged
  twiddles(W2, p.tw2, N2);
  auto base = [&](int u) { return p.y + (long long)(u / gpc) * p.nh + (long long)(u % gpc) * FFT_G; };
  auto width = [&](int u) { return min(FFT_G, P - (u % gpc) * FFT_G); };
  auto prefetch = [&](int u) {
    if (u < units) {
      const double2* yp = base(u);
      const int g = width(u);
      for (int idx = threadIdx.x; idx < FFT_G * N2; idx += FFT_THREADS) {
        const int e = idx / FFT_G, t = idx - e * FFT_G;
        cp_async16(S + idx, t < g ? yp + (long long)e * P + t : yp, t < g);
      }
    }
    cp_async_commit();
  };
  prefetch(blockIdx.x);
  for (int u = blockIdx.x; u < units; u += gridDim.x) {
    cp_async_wait<0>();
    __syncthreads();
    for (int idx = threadIdx.x; idx < FFT_G * N2; idx += FFT_THREADS) A[idx] = S[idx];
    __syncthreads();
    prefetch(u + gridDim.x);
    double2* R = stockham<N2, FFT_G, 1, FFT_G>(A, B, W2);
    double2* yp = base(u);
    const int g = width(u);
    for (int idx = threadIdx.x; idx < FFT_G * N2; idx += FFT_THREADS) {
      const int e = idx / FFT_G, t = idx - e * FFT_G;
      if (t < g) yp[(long long)e * P + t] = R[idx];
    }
  }
  cp_async_wait<0>();
}

template <class K>
int resident(K kern, size_t smem) {
  int per = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, FFT_THREADS, smem) != cudaSuccess) return 1;
  return per < 1 ? 1 : per;
}

template <int N0, int N1>
cudaError_t launch_planes(cudaStream_t st, const FftParams& p, int m, int sms) {
  constexpr size_t smem = planes_smem<N0, N1>(planes_stage<N0, N1>());
  static_assert(smem <= 200 * 1024, "plane plan exceeds shared memory");
  auto kern = fft_planes_kernel<N0, N1>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int units = p.n2 * m;
  const int grid = std::min(units, sms * resident(kern, smem));
  kern<<<grid, FFT_THREADS, smem, st>>>(p, units);
  count_launches(1);
  return cudaGetLastError();
}

template <int N2>
cudaError_t launch_pencils(cudaStream_t st, const FftParams& p, int m, int sms) {
  constexpr size_t smem = (size_t)(3 * FFT_G * N2 + FFT_MAXN) * sizeof(double2);
  static_assert(smem <= 220 * 1024, "pencil plan exceeds shared memory");
  auto kern = fft_pencils_kernel<N2>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int P = p.n1 * p.h, gpc = (P + FFT_G - 1) / FFT_G, units = gpc * m;
  const int grid = std::min(units, sms * resident(kern, smem));
  kern<<<grid, FFT_THREADS, smem, st>>>(p, units, gpc);
  count_launches(1);
  return cudaGetLastError();
}

// The cubic grids of the path (Si8 24^3, Si64 48^3, Si216 72^3, C60 80^3,
// Si512 96^3) and a few test sizes; other shapes stay on cuFFT.
#define LRGW_FFT_SIZES(X) X(8) X(12) X(16) X(24) X(32) X(48) X(64) X(72) X(80) X(96)

}  // namespace

// Opt-in (LRGW_FFT_OWN=1): correct (the parity suite passes on it) but not yet
// faster than the cuFFT leaf — Si64 D2Z 1.55 vs 1.18 ms, Si512 139 vs 122 ms
// (profiles/r02/fft_own.txt): ncu shows the Stockham stages bound by shared-
// memory latency and bank conflicts (short_scoreboard 39 %, barrier 30 %);
// register-resident radix passes are the next step.
bool fft_own_enabled() {
  static const bool on = getenv("LRGW_FFT_OWN") && atoi(getenv("LRGW_FFT_OWN")) == 1;
  return on;
}

cudaError_t fft_d2z_3d(cudaStream_t st, const int* dims, const double* x, long long ldx, int m, double* xhat,
                       int sms) {
  FftParams p{};
  p.n0 = dims[0], p.n1 = dims[1], p.n2 = dims[2];
  p.h = p.n0 / 2 + 1;
  p.nh = (long long)p.h * p.n1 * p.n2;
  p.x = x, p.ldx = ldx, p.y = reinterpret_cast<double2*>(xhat);
  if (m <= 0) return cudaSuccess;
  // cubic grids only (one template per edge)
  if (p.n0 != p.n1 || p.n1 != p.n2 || ldx < (long long)p.n0 * p.n1 * p.n2 || ldx % 2 != 0 ||
      (reinterpret_cast<uintptr_t>(xhat) & 15) != 0 || (reinterpret_cast<uintptr_t>(x) & 15) != 0 ||
      (long long)m * p.n2 > 0x7fffffffLL / 2)
    return cudaErrorNotSupported;
  // per-size twiddle tables (device, built once per size; never freed — a few KB)
  static double2* tabs[FFT_MAXN + 1] = {};
  if (p.n0 > FFT_MAXN) return cudaErrorNotSupported;
  if (!tabs[p.n0]) {
    double2* t = nullptr;
    if (cudaMalloc(&t, sizeof(double2) * p.n0) != cudaSuccess) return cudaErrorMemoryAllocation;
    twiddle_table_kernel<<<1, 128, 0, st>>>(t, p.n0);
    count_launches(1);
    tabs[p.n0] = t;
  }
  p.tw0 = p.tw1 = p.tw2 = tabs[p.n0];
  cudaError_t e = cudaErrorNotSupported;
  switch (p.n0) {
#define LRGW_FFT_CASE(n)                          \
  case n:                                         \
    e = launch_planes<n, n>(st, p, m, sms);       \
    if (e == cudaSuccess) e = launch_pencils<n>(st, p, m, sms); \
    break;
    LRGW_FFT_SIZES(LRGW_FFT_CASE)
#undef LRGW_FFT_CASE
    default:
      break;
  }
  return e;
}

}  // namespace lrgw_dev
