// FP64 peak microbenchmarks for B200 (sm_100a): DFMA pipe vs DMMA (mma.sync f64).
// Used once to fix the FP64 roofline denominator (MEASURED_PEAKS.json has none)
// and to choose between DFMA and DMMA for the hot GEMMs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peaks fp64_peaks.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

template <int CHAINS>
__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double acc[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = threadIdx.x * 1e-9 + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 12345.678) out[0] = s;
}

template <int CHAINS>
__global__ void dmma_loop(double* out, int iters) {
  const int lane = threadIdx.x & 31;
  double a = 1.0 + lane * 1e-6, b = 1.0 - lane * 1e-6;
  double c[CHAINS][2];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

template <int CHAINS>
__global__ void dmma16_loop(double* out, int iters) {
  const int lane = threadIdx.x & 31;
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = 1.0 + (lane + i) * 1e-6;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1.0 - (lane + i) * 1e-6;
  double c[CHAINS][4];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) { c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) {
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
                   "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.678) out[0] = s;
}


// GEMM-like operand pattern: FM x FN accumulator tiles, distinct A/B fragment
// registers per MMA (as in a warp tile), optionally i-major or j-major order.
template <int FM, int FN, bool JMAJOR>
__global__ void dmma_tile_loop(double* out, int iters) {
  const int lane = threadIdx.x & 31;
  double af[FM], bf[FN], acc[FM][FN][2];
#pragma unroll
  for (int i = 0; i < FM; ++i) af[i] = 1.0 + (lane + i) * 1e-6;
#pragma unroll
  for (int j = 0; j < FN; ++j) bf[j] = 1.0 - (lane + j) * 1e-6;
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
    if (JMAJOR) {
#pragma unroll
      for (int j = 0; j < FN; ++j)
#pragma unroll
        for (int i = 0; i < FM; ++i)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                       : "+d"(acc[i][j][0]), "+d"(acc[i][j][1]) : "d"(af[i]), "d"(bf[j]));
    } else {
#pragma unroll
      for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                       : "+d"(acc[i][j][0]), "+d"(acc[i][j][1]) : "d"(af[i]), "d"(bf[j]));
    }
  }
  double sum = 0;
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j) sum += acc[i][j][0] + acc[i][j][1];
  if (sum == 12345.678) out[0] = sum;
}

template <int FM, int FN, bool JM>
void run_tile(double* d, int sms, int wpb, int bps) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4000;
  int blocks = sms * bps, threads = 32 * wpb;
  dmma_tile_loop<FM, FN, JM><<<blocks, threads>>>(d, 10);
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  dmma_tile_loop<FM, FN, JM><<<blocks, threads>>>(d, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  double fl = 2.0 * 256 * FM * FN * (double)iters * blocks * wpb;
  printf("DMMA tile %dx%d %s warps/blk=%2d blk/SM=%d : %8.2f TFLOP/s\n", FM * 8, FN * 8, JM ? "j-major" : "i-major",
         wpb, bps, fl / ms / 1e9);
}


// Mixed pipes: warps with (warp % 2 == 0) run DMMA, the others DFMA, in one
// kernel; and an interleaved variant where every warp issues both. If the
// DMMA and DFMA pipes were separate, the sum would exceed either alone.
template <int CHAINS>
__global__ void mixed_loop(double* out, int iters, int mode) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double a = 1.0 + lane * 1e-6, b = 1.0 - lane * 1e-6;
  double c[CHAINS][2], f[CHAINS * 2];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) { c[i][0] = 0; c[i][1] = 0; f[2 * i] = lane; f[2 * i + 1] = i; }
  const bool do_mma = mode == 2 || (warp & 1) == 0;
  const bool do_fma = mode == 2 || (warp & 1) == 1;
  for (int it = 0; it < iters; ++it) {
    if (do_mma) {
#pragma unroll
      for (int i = 0; i < CHAINS; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
    if (do_fma) {
#pragma unroll
      for (int i = 0; i < 2 * CHAINS; ++i) f[i] = fma(f[i], a, b);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i][0] + c[i][1] + f[2 * i] + f[2 * i + 1];
  if (s == 12345.678) out[0] = s;
}

void run_mixed(double* d, int sms, int wpb, int bps, int mode) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  int blocks = sms * bps, threads = 32 * wpb;
  mixed_loop<8><<<blocks, threads>>>(d, 10, mode);
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  mixed_loop<8><<<blocks, threads>>>(d, iters, mode);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  // per warp per iteration: 8 DMMA (256 fma each = 512 flop) and/or 16 x 32 DFMA (2 flop)
  double per_mma = 2.0 * 256 * 8, per_fma = 2.0 * 16 * 32;
  double warps = (double)blocks * wpb, fl;
  if (mode == 2) fl = warps * (per_mma + per_fma) * iters;
  else fl = warps / 2 * (per_mma + per_fma) * iters;
  printf("MIXED mode=%s warps/blk=%2d blk/SM=%d : %8.2f TFLOP/s (%.3f ms)\n", mode == 2 ? "interleaved" : "split-warps",
         wpb, bps, fl / ms / 1e9, ms);
}

int main() {
  double* d;
  CK(cudaMalloc(&d, 64));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  const int iters = 20000;
  for (int wpb : {4, 8, 16}) {
    for (int bps : {1, 2, 4}) {
      int blocks = sms * bps, threads = 32 * wpb;
      dfma_loop<8><<<blocks, threads>>>(d, 100, 1.0000001, 1e-9);
      CK(cudaDeviceSynchronize());
      cudaEventRecord(e0);
      dfma_loop<8><<<blocks, threads>>>(d, iters, 1.0000001, 1e-9);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms, e0, e1);
      double fl = 2.0 * 8 * iters * (double)blocks * threads;
      printf("DFMA   warps/blk=%2d blk/SM=%d : %8.2f TFLOP/s (%.3f ms)\n", wpb, bps, fl / ms / 1e9, ms);
    }
  }
  for (int wpb : {4, 8, 16}) {
    for (int bps : {1, 2, 4}) {
      int blocks = sms * bps, threads = 32 * wpb;
      dmma_loop<8><<<blocks, threads>>>(d, 100);
      CK(cudaDeviceSynchronize());
      cudaEventRecord(e0);
      dmma_loop<8><<<blocks, threads>>>(d, iters);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms, e0, e1);
      double fl = 2.0 * 256 * 8 * iters * (double)blocks * wpb;
      printf("DMMA884 warps/blk=%2d blk/SM=%d : %8.2f TFLOP/s (%.3f ms)\n", wpb, bps, fl / ms / 1e9, ms);
    }
  }
  for (int wpb : {4, 8}) {
    for (int bps : {1, 2}) {
      int blocks = sms * bps, threads = 32 * wpb;
      dmma16_loop<4><<<blocks, threads>>>(d, 100);
      CK(cudaDeviceSynchronize());
      cudaEventRecord(e0);
      dmma16_loop<4><<<blocks, threads>>>(d, iters / 4);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms, e0, e1);
      double fl = 2.0 * 16 * 8 * 16 * 4 * (iters / 4) * (double)blocks * wpb;
      printf("DMMA16816 warps/blk=%2d blk/SM=%d : %8.2f TFLOP/s (%.3f ms)\n", wpb, bps, fl / ms / 1e9, ms);
    }
  }
  for (int mode : {1, 2}) for (int wpb : {8, 16}) run_mixed(d, sms, wpb, 2, mode);
  run_tile<4, 4, false>(d, sms, 8, 2);
  run_tile<4, 4, true>(d, sms, 8, 2);
  run_tile<4, 4, false>(d, sms, 4, 2);
  run_tile<4, 4, false>(d, sms, 16, 1);
  run_tile<8, 4, false>(d, sms, 8, 1);
  run_tile<4, 2, false>(d, sms, 8, 1);
  run_tile<4, 2, false>(d, sms, 8, 2);
  run_tile<2, 2, false>(d, sms, 8, 2);
  return 0;
}
