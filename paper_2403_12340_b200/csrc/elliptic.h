// elliptic.h — host-side contour geometry for the Cauchy quadrature (stage 3).
//
// Scalars only (microseconds per node); the GPU consumes the resulting
// per-node complex diagonals d_k = 1/(z_k - e) and weights w_k * g_k.
// Produces the reference's contour geometry (elliptic.hpp:17-118,
// contour.hpp:35-80, 144-183) by its own derivation (see elliptic.cpp).
#pragma once

#include <complex>
#include <vector>

namespace lrgw_host {

struct Spec {  // contour.hpp:23-33
  double q = 0, big_q = 0, r = 0, big_r = 0, l = 0, e_shift = 0;
  double delta_rel = 1e-7;
  int max_nodes = 1025;
  bool bypass = false;
};

// Status codes shared with include/lrgw_cuda.h.
enum Status { kOk = 0, kInvalid = 1, kGuard = 2, kNumeric = 3, kSingular = 4, kContour = 5 };

double agm(double a, double b);
int elliptic_k(double k, double* out);
int jacobi_sn_cn_dn(double u, double k, double* sn, double* cn, double* dn);
int jacobi_complex(double x, double y, double k, std::complex<double>* sn, std::complex<double>* cn,
                   std::complex<double>* dn);
int elliptic_params(const double* e, int n_e, int n_v, int n_c, double delta_rel, int max_nodes,
                    Spec* out);
int cauchy_error_bound(const Spec& s, int n_lambda, double* out);
double prefactor(const Spec& s);  // 2 sqrt(qQ) / (pi r), contour.hpp:247-248

// Node geometry at parameter t: z(t + iL), g = cn dn / (1/r - sn)^2.
int node_geometry(const Spec& s, double t, std::complex<double>* z, std::complex<double>* g);

// Per-node device inputs for a node list with weights:
//   dv[k*n_v + i] = 1/(z_k - e_i), dc[k*n_c + j] = 1/(z_k - e_{n_v+j}),
//   gw[k] = w_k * g_k. Layout: interleaved (re, im) doubles.
int node_tables(const Spec& s, const double* e, int n_v, int n_c, const double* nodes,
                const double* weights, int n_nodes, std::vector<double>* dv,
                std::vector<double>* dc, std::vector<double>* gw);

}  // namespace lrgw_host
