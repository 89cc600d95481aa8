"""Generate the GW golden fixtures (tests/golden/gw_*.npz) from the REFERENCE.

The systems are test_gw.cpp's `System` fixture (test_gw.cpp:13-41): the
reference's build_synthetic_system on a 6 bohr cell, vc / vn / nn ISDF
(isdf.hpp:166-183), T by the direct sum, build_epsilon_inverse,
project_screened_interactions and the three self-energy pipelines (gw.hpp).
All outputs come from the unmodified reference compiled into
oracle/_ref/libref_lrgw.so:

  psi, energies, dims, cell, n_v, n_c
  pts_vc / pts_vn / pts_nn, theta_vc / theta_vn / theta_nn
  t_direct, k                         (contour.hpp:114-137, smw.hpp:42-73)
  w_vn, w_nn, v_vn                    (gw.hpp:73-88)
  sig_lowrank, sig_conventional, sig_bruteforce  (4 x N_b: sex_x, x, coh, total)

    python tests/golden/make_golden_gw.py     (needs /root/reference; run here)
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402

SYSTEMS = [
    # name, seed, dims, n_v = n_c, k (vc = vn = nn)   — test_gw.cpp:116-127, 174-184
    ("gw_s3", 3, (8, 8, 8), 16, 8.0),
    ("gw_s7", 7, (8, 8, 4), 8, 6.0),
]


def main():
    out_dir = os.path.dirname(os.path.abspath(__file__))
    cell = (6.0, 6.0, 6.0)
    for name, seed, dims, n, k in SYSTEMS:
        psi, e = ref.build_synthetic(seed, dims, cell, n, n, 1.0, 4.0)
        n_r = psi.shape[0]
        fac = {"vc": (psi[:, :n], psi[:, n:]), "vn": (psi[:, :n], psi), "nn": (psi, psi)}
        out = dict(psi=psi, energies=e, dims=np.array(dims), cell=np.array(cell), n_v=n, n_c=n)
        for lab, (a, b) in fac.items():
            n_mu = min(max(ref.num_aux(k, a.shape[1], b.shape[1]), 1), n_r)
            pts = ref.select_points(a, b, n_mu)
            out[f"pts_{lab}"] = pts
            out[f"theta_{lab}"] = ref.fit(a, b, pts)
        pts = out["pts_vc"]
        t = ref.coupled_direct(psi[pts, :n], psi[pts, n:], e)
        out["t_direct"] = t
        out["k"] = ref.assemble_K(t, out["theta_vc"], dims, cell)
        w_vn, w_nn, v_vn = ref.project_screened(t, out["theta_vc"], dims, cell, out["theta_vn"], out["theta_nn"])
        out.update(w_vn=w_vn, w_nn=w_nn, v_vn=v_vn)
        for which in ("lowrank", "conventional", "bruteforce"):
            out[f"sig_{which}"] = np.array(ref.self_energies(psi, n, dims, cell, e, out["pts_vc"], out["pts_vn"],
                                                             out["pts_nn"], which))
        np.savez_compressed(os.path.join(out_dir, f"{name}.npz"), **out)
        print(name, n_r, {lab: len(out[f"pts_{lab}"]) for lab in fac},
              "lowrank-vs-conventional", np.abs(out["sig_lowrank"][3] - out["sig_conventional"][3]).max())


if __name__ == "__main__":
    main()
