// common.cuh — shared device primitives for the lrgw B200 kernels (sm_100a).
//
// FP64 on B200: tcgen05 has no kind::f64, so the FP64 tensor path is the
// warp-level DMMA (mma.sync m8n8k4 f64 -> SASS DMMA.8x8x4). Measured on this
// pool (profiles/fp64_peaks_r01.txt): DMMA 37.2 TFLOP/s vs DFMA 34.2 TFLOP/s,
// so every FP64 contraction here is DMMA fed from shared memory that is
// filled by a multi-stage cp.async pipeline.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace lrgw_dev {

// D(8x8) += A(8x4) * B(4x8). Fragment ownership (PTX ISA, m8n8k4 .f64):
//   g = lane >> 2, t = lane & 3
//   a  = A[g][t]            b  = B[t][g]  (i.e. B^T[g][t])
//   c0 = C[g][2t], c1 = C[g][2t+1]
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  // not volatile: the compiler may interleave the MMAs with the next step's
  // fragment loads (measured +4-6 % on the K-contiguous and v1 engines, the
  // same results bit for bit: each accumulator's chain is unchanged)
  asm(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

// All FM x FN DMMA.8x8x4 of one k4 step (i-major; ptxas schedules them).
template <int FM, int FN>
__device__ __forceinline__ void dmma_block(double (&acc)[FM][FN][2], const double (&af)[FM], const double (&bf)[FN]) {
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// The 1024-byte aligned start of a TMA ring inside the dynamic shared memory
// (128-byte swizzle keys on shared-address bits 7-9). The pad is added to the
// array itself: rounding the pointer through an integer makes every later
// access a generic load (LD.E) instead of LDS.
__device__ __forceinline__ double* smem_ring_1024(unsigned char* smem_raw) {
  return reinterpret_cast<double*>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
}

// 16-byte async copy global->shared, zero-filled when !pred.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  const int n = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(smem)),
               "l"(gmem), "r"(n));
}

// 8-byte async copy (ca path), zero-filled when !pred.
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool pred) {
  const int n = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(smem)),
               "l"(gmem), "r"(n));
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }

template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Map a linear block index onto the lower-triangle tile (i >= j) of a
// T x T tile grid, row-major over the triangle: idx = i(i+1)/2 + j.
__device__ __forceinline__ void lower_tile(int idx, int& ti, int& tj) {
  int i = static_cast<int>((sqrt(8.0 * idx + 1.0) - 1.0) * 0.5);
  while ((i + 1) * (i + 2) / 2 <= idx) ++i;
  while (i * (i + 1) / 2 > idx) --i;
  ti = i;
  tj = idx - i * (i + 1) / 2;
}

}  // namespace lrgw_dev
