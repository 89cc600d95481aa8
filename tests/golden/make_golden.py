"""Generate the golden fixtures of tests/golden/ from the REFERENCE itself.

Runs the unmodified reference `lrgw` (compiled by oracle/Makefile into
oracle/_ref/libref_lrgw.so) on the reference's own seeded desk-scale systems
(build_synthetic_system, model.hpp:56-116 — the shapes of test_isdf.cpp,
test_smw.cpp and acceptance.cpp:123-127) and stores inputs + outputs:

  psi, energies, dims, cell, n_v, n_c, n_mu, n_lambda
  pts      select_interpolation_points          (isdf.hpp:95-112)
  theta    fit_auxiliary_basis                  (isdf.hpp:118-163)
  t_direct coupled_coefficients_direct          (contour.hpp:114-137)
  t_fixed  pref * sum_node_terms at the closed n_lambda-interval trapezoid,
           symmetrised (contour.hpp:185-222, 247-248, 276)
  t_adapt  coupled_coefficients_contour (delta 1e-7) + nodes_used
  k        assemble_K(t_direct, theta)          (smw.hpp:42-73)
  x, y     probe block and build_epsilon_inverse + epsilon_inverse_apply
           (smw.hpp:84-103)

    python tests/golden/make_golden.py        (needs /root/reference; run here)
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402

SYSTEMS = [
    # name, seed, dims, n, k, gap, bandwidth, n_lambda
    ("si8shaped_s1", 1, (8, 8, 8), 16, 8.0, 1.0, 4.0, 16),
    ("acc_s2", 2, (8, 8, 4), 12, 6.0, 1.0, 4.0, 16),
    ("acc_s3", 3, (8, 8, 8), 8, 6.0, 1.0, 4.0, 24),
    ("acc_s4", 4, (4, 4, 4), 4, 3.0, 1.0, 4.0, 16),
    ("acc_s5", 5, (8, 4, 4), 6, 4.0, 1.0, 4.0, 32),
    ("wide_s3", 3, (8, 8, 8), 16, 8.0, 0.05, 4.95, 40),
]


def main():
    out_dir = os.path.dirname(os.path.abspath(__file__))
    for name, seed, dims, n, k, gap, bw, n_lambda in SYSTEMS:
        cell = tuple(0.75 * d for d in dims) if name.startswith("acc") else (6.0, 6.0, 6.0)
        psi, e = ref.build_synthetic(seed, dims, cell, n, n, gap, bw)
        a, b = psi[:, :n], psi[:, n:]
        n_r = psi.shape[0]
        n_mu = min(max(ref.num_aux(k, n, n), 1), n_r)
        pts = ref.select_points(a, b, n_mu)
        theta = ref.fit(a, b, pts)
        pv, pc = a[pts], b[pts]
        t_direct = ref.coupled_direct(pv, pc, e)
        s7 = ref.elliptic_params(e, n, n)
        h = 2.0 * s7[3] / n_lambda
        nodes = [-s7[3] + i * h for i in range(n_lambda + 1)]
        w = [0.5 * h if i in (0, n_lambda) else h for i in range(n_lambda + 1)]
        pref = 2.0 * np.sqrt(s7[0] * s7[1]) / (np.pi * s7[2])
        acc = pref * ref.sum_node_terms(pv, pc, e, s7, nodes, w)
        t_fixed = 0.5 * (acc + acc.T)
        t_adapt, nodes_used, est, st = ref.coupled_contour(pv, pc, e, 1e-7, 1025)
        kk = ref.assemble_K(t_direct, theta, dims, cell)
        x = ref.gaussian(seed ^ 0xA5A5A5A5, n_r, 4)
        y, _, _ = ref.build_and_apply(t_direct, theta, dims, cell, x)
        np.savez_compressed(
            os.path.join(out_dir, f"{name}.npz"), psi=psi, energies=e, dims=np.array(dims), cell=np.array(cell),
            n_v=n, n_c=n, n_mu=n_mu, n_lambda=n_lambda, pts=pts, theta=theta, t_direct=t_direct,
            t_fixed=t_fixed, t_adapt=t_adapt, nodes_used=nodes_used, k=kk, x=x, y=y)
        print(name, n_r, n_mu, "nodes_used", nodes_used, "status", st)


if __name__ == "__main__":
    main()
