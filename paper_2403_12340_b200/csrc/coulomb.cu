// coulomb.cu — K4: Coulomb kernel in G-space for the half-spectrum D2Z layout.
//
// Reference: build_coulomb (model.hpp:165-195) + Grid::g_norm2 / freq
// (grid.hpp:30-42): v(G) = 4 pi / |G|^2, v(0) = 0; apply_coulomb
// (model.hpp:208-223) = Re(F^-1 diag(v) F x) with the unitary DFT. cuFFT is
// unnormalised, so V x = Z2D(v/N_r * D2Z(x)), and for real x, y
//   x^T V y = sum_{G in half} w_G v(G)/N_r (Re x^ Re y^ + Im x^ Im y^),
// w_G = 1 on the self-conjugate planes i1 = 0 and i1 = n1/2 (n1 even), else 2.
// The weights below are the `scale` of the G-space SYRK (Theta^T V Theta),
// fused into that GEMM's operand load; the in-place scale is the probe path.
#include "kernels.h"
#include "shard.h"

namespace lrgw_dev {

namespace {

__device__ __forceinline__ double vG(int i1, int i2, int i3, int n1, int n2, int n3, double c1,
                                     double c2, double c3) {
  const double two_pi = 6.283185307179586476925286766559;
  const int f1 = (i1 <= n1 / 2) ? i1 : i1 - n1;
  const int f2 = (i2 <= n2 / 2) ? i2 : i2 - n2;
  const int f3 = (i3 <= n3 / 2) ? i3 : i3 - n3;
  const double g1 = two_pi * f1 / c1, g2 = two_pi * f2 / c2, g3 = two_pi * f3 / c3;
  const double g = g1 * g1 + g2 * g2 + g3 * g3;
  return g > 0.0 ? 12.566370614359172953850573533118 / g : 0.0;
}

__global__ void half_weights_kernel(int n1, int n2, int n3, double c1, double c2, double c3,
                                    int zero_kernel, double* w) {
  const int nh = n1 / 2 + 1;
  const long long total = (long long)nh * n2 * n3;
  const double inv_n = 1.0 / ((double)n1 * n2 * n3);
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
       q += (long long)gridDim.x * blockDim.x) {
    const int i1 = static_cast<int>(q % nh);
    const int i2 = static_cast<int>((q / nh) % n2);
    const int i3 = static_cast<int>(q / ((long long)nh * n2));
    const double herm = (i1 == 0 || (n1 % 2 == 0 && i1 == n1 / 2)) ? 1.0 : 2.0;
    const double v = zero_kernel ? 0.0 : vG(i1, i2, i3, n1, n2, n3, c1, c2, c3);
    const double c = herm * v * inv_n;
    w[2 * q] = c;
    w[2 * q + 1] = c;
  }
}

__global__ void scale_half_kernel(int n1, int n2, int n3, double c1, double c2, double c3,
                                  int zero_kernel, double2* x, int cols) {
  const int nh = n1 / 2 + 1;
  const long long per = (long long)nh * n2 * n3;
  const long long total = per * cols;
  const double inv_n = 1.0 / ((double)n1 * n2 * n3);
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long q = idx % per;
    const int i1 = static_cast<int>(q % nh);
    const int i2 = static_cast<int>((q / nh) % n2);
    const int i3 = static_cast<int>(q / ((long long)nh * n2));
    const double s = zero_kernel ? 0.0 : vG(i1, i2, i3, n1, n2, n3, c1, c2, c3) * inv_n;
    double2 v = x[idx];
    v.x *= s;
    v.y *= s;
    x[idx] = v;
  }
}

// pencil order (y - ya, i1, i3), i3 fastest: the z-pencils of one rank's y-slab
__global__ void slab_weights_kernel(int n1, int n2, int n3, double c1, double c2, double c3, int zero_kernel, int ya,
                                    int ny, double* w) {
  const int nh = n1 / 2 + 1;
  const long long total = (long long)ny * nh * n3;
  const double inv_n = 1.0 / ((double)n1 * n2 * n3);
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
       q += (long long)gridDim.x * blockDim.x) {
    const int i3 = static_cast<int>(q % n3);
    const int i1 = static_cast<int>((q / n3) % nh);
    const int i2 = ya + static_cast<int>(q / ((long long)n3 * nh));
    const double herm = (i1 == 0 || (n1 % 2 == 0 && i1 == n1 / 2)) ? 1.0 : 2.0;
    const double v = zero_kernel ? 0.0 : vG(i1, i2, i3, n1, n2, n3, c1, c2, c3);
    const double c = herm * v * inv_n;
    w[2 * q] = c;
    w[2 * q + 1] = c;
  }
}

// a caller's kernel v (full grid, linear index i1 + n1 (i2 + n2 i3)): the real
// part of F^-1 diag(v) F x equals F^-1 diag((v(G) + v(-G)) / 2) F x for real x,
// which is what the half spectrum carries
__global__ void scale_half_custom_kernel(int n1, int n2, int n3, const double* v, double2* x, int cols) {
  const int nh = n1 / 2 + 1;
  const long long per = (long long)nh * n2 * n3;
  const long long total = per * cols;
  const double inv_n = 1.0 / ((double)n1 * n2 * n3);
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long q = idx % per;
    const int i1 = static_cast<int>(q % nh);
    const int i2 = static_cast<int>((q / nh) % n2);
    const int i3 = static_cast<int>(q / ((long long)nh * n2));
    const int j1 = (n1 - i1) % n1, j2 = (n2 - i2) % n2, j3 = (n3 - i3) % n3;
    const double vp = v[i1 + (long long)n1 * (i2 + (long long)n2 * i3)];
    const double vm = v[j1 + (long long)n1 * (j2 + (long long)n2 * j3)];
    const double s = 0.5 * (vp + vm) * inv_n;
    double2 t = x[idx];
    t.x *= s;
    t.y *= s;
    x[idx] = t;
  }
}

}  // namespace

cudaError_t coulomb_scale_half_custom(cudaStream_t st, int n1, int n2, int n3, const double* v, double* xhat,
                                      int cols) {
  scale_half_custom_kernel<<<1184, 256, 0, st>>>(n1, n2, n3, v, reinterpret_cast<double2*>(xhat), cols);
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t coulomb_slab_weights(cudaStream_t st, int n1, int n2, int n3, double c1, double c2, double c3,
                                 int zero_kernel, int ya, int ny, double* w) {
  if (ny <= 0) return cudaSuccess;
  slab_weights_kernel<<<592, 256, 0, st>>>(n1, n2, n3, c1, c2, c3, zero_kernel, ya, ny, w); count_launches(1);
  return cudaGetLastError();
}

cudaError_t coulomb_half_weights(cudaStream_t st, int n1, int n2, int n3, double c1, double c2,
                                 double c3, int zero_kernel, double* w) {
  half_weights_kernel<<<592, 256, 0, st>>>(n1, n2, n3, c1, c2, c3, zero_kernel, w); count_launches(1);
  return cudaGetLastError();
}

cudaError_t coulomb_scale_half(cudaStream_t st, int n1, int n2, int n3, double c1, double c2,
                               double c3, int zero_kernel, double* xhat, int cols) {
  scale_half_kernel<<<1184, 256, 0, st>>>(n1, n2, n3, c1, c2, c3, zero_kernel,
                                          reinterpret_cast<double2*>(xhat), cols); count_launches(1);
  return cudaGetLastError();
}

}  // namespace lrgw_dev
