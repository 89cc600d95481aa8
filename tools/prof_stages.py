"""Run each hot kernel of the Si64 build once through the stage-level device
API (for `ncu --set full` captures: one launch per kernel of interest)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import ctypes

    import torch

    from paper_2403_12340_b200 import lrgw, synth

    which = sys.argv[1:] or ["pvp", "fit", "contour", "select"]
    cfg = synth.CONFIGS["si64"]
    ctx = lrgw.Context(0)
    lib = lrgw.L.load()
    psi = synth.orbitals_device(cfg)
    e = synth.energies(cfg)
    n_mu = 1024
    pts = np.sort(np.random.default_rng(0).choice(cfg.n_r, n_mu, replace=False)).astype(np.int32)
    theta = torch.empty(n_mu, cfg.n_r, dtype=torch.float64, device="cuda").t()
    torch.cuda.synchronize()
    dims = np.array(cfg.dims, dtype=np.int32)
    cell = np.array(cfg.cell3)
    if "fit" in which:
        rc = lib.lrgw_dev_fit(ctx.handle, psi.data_ptr(), cfg.n_r, 128, psi[:, 128:].data_ptr(), cfg.n_r, 128,
                              cfg.n_r, pts.ctypes.data_as(lrgw.L.c_int32_p), n_mu, theta.data_ptr(), cfg.n_r)
        assert rc == 0, rc
    if "pvp" in which:
        if "fit" not in which:
            theta.copy_(torch.randn_like(theta) / cfg.n_r ** 0.5)
        pvp = torch.empty(n_mu, n_mu, dtype=torch.float64, device="cuda")
        rc = lib.lrgw_dev_pvp(ctx.handle, dims.ctypes.data_as(lrgw.L.c_int_p), cell.ctypes.data_as(lrgw.L.c_double_p),
                              0, theta.data_ptr(), cfg.n_r, n_mu, pvp.data_ptr())
        assert rc == 0, rc
    if "contour" in which:
        pv = psi[pts.astype(np.int64), :128].t().contiguous().t()
        pc = psi[pts.astype(np.int64), 128:].t().contiguous().t()
        t = torch.empty(n_mu, n_mu, dtype=torch.float64, device="cuda")
        rc = lib.lrgw_dev_contour_fixed(ctx.handle, pv.data_ptr(), n_mu, pc.data_ptr(), n_mu, n_mu, 128, 128,
                                        e.ctypes.data_as(lrgw.L.c_double_p), 256, cfg.n_lambda, t.data_ptr(), n_mu)
        assert rc == 0, rc
    if "select" in which:
        out = np.zeros(n_mu, dtype=np.int32)
        mm = ctypes.c_double(0)
        nsel = int(os.environ.get("PROF_SELECT_NMU", "256"))
        rc = lib.lrgw_dev_select(ctx.handle, psi.data_ptr(), cfg.n_r, 128, psi[:, 128:].data_ptr(), cfg.n_r, 128,
                                 cfg.n_r, nsel, out.ctypes.data_as(lrgw.L.c_int32_p), ctypes.byref(mm))
        assert rc == 0, rc
    torch.cuda.synchronize()
    print("ok", which)


if __name__ == "__main__":
    main()
