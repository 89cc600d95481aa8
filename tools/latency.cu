// Dependent-chain latencies on sm_100a (one warp): DFMA, DMUL, DADD, FFMA,
// IMAD, DP division / sqrt, redux.sync, shfl, LDS. Used to size the
// candidate-greedy controller's critical path.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o latency latency.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat(long long* out, double x, float xf, int xi, int n) {
  __shared__ double sh[64];
  sh[threadIdx.x] = x;
  __syncwarp();
  long long t0, t1;
  double a = x;
  t0 = clock64();
  for (int i = 0; i < n; ++i) a = fma(a, x, 1e-30);
  t1 = clock64();
  out[0] = (t1 - t0) / n;
  double b = x;
  t0 = clock64();
  for (int i = 0; i < n; ++i) b = b * x;
  t1 = clock64();
  out[1] = (t1 - t0) / n;
  float c = xf;
  t0 = clock64();
  for (int i = 0; i < n; ++i) c = fmaf(c, xf, 1e-30f);
  t1 = clock64();
  out[2] = (t1 - t0) / n;
  int d = xi;
  t0 = clock64();
  for (int i = 0; i < n; ++i) d = d * xi + 1;
  t1 = clock64();
  out[3] = (t1 - t0) / n;
  double e = x;
  t0 = clock64();
  for (int i = 0; i < n; ++i) e = 1.0 / e;
  t1 = clock64();
  out[4] = (t1 - t0) / n;
  double f = x;
  t0 = clock64();
  for (int i = 0; i < n; ++i) f = sqrt(f) + 1.0;
  t1 = clock64();
  out[5] = (t1 - t0) / n;
  unsigned g = xi;
  t0 = clock64();
  for (int i = 0; i < n; ++i) g = __reduce_max_sync(0xffffffffu, g + threadIdx.x);
  t1 = clock64();
  out[6] = (t1 - t0) / n;
  double h = x;
  t0 = clock64();
  for (int i = 0; i < n; ++i) h = __shfl_xor_sync(0xffffffffu, h, 1) + 1.0;
  t1 = clock64();
  out[7] = (t1 - t0) / n;
  int k = 0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) k = static_cast<int>(sh[(k + threadIdx.x) & 63]);
  t1 = clock64();
  out[8] = (t1 - t0) / n;
  double m = x;
  t0 = clock64();
  for (int i = 0; i < n; ++i) m = m + x;
  t1 = clock64();
  out[9] = (t1 - t0) / n;
  double q = x;
  t0 = clock64();
  for (int i = 0; i < n; ++i) q = fmax(q, x) + 0.5;
  t1 = clock64();
  out[10] = (t1 - t0) / n;
  double r = x;
  t0 = clock64();
  for (int i = 0; i < n; ++i) r = rsqrt(r) + 1.0;
  t1 = clock64();
  out[11] = (t1 - t0) / n;
  if (threadIdx.x == 0) out[12] = (long long)(a + b + c + d + e + f + g + h + k + m + q + r);
}

int main() {
  long long* o;
  cudaMallocManaged(&o, 16 * sizeof(long long));
  lat<<<1, 32>>>(o, 1.0000001, 1.0000001f, 3, 1000);
  cudaDeviceSynchronize();
  lat<<<1, 32>>>(o, 1.0000001, 1.0000001f, 3, 1000);
  cudaDeviceSynchronize();
  const char* nm[] = {"DFMA", "DMUL", "FFMA", "IMAD", "ddiv(1/x)", "dsqrt+1", "redux", "shfl64+dadd", "LDS dep", "DADD", "fmax+dadd", "rsqrt+1"};
  for (int i = 0; i < 12; ++i) printf("%-14s %lld cycles\n", nm[i], o[i]);
  return 0;
}
