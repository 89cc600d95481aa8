"""WFN1 straight into HBM (lrgw_wfn1_load_device): pinned double-buffered
column blocks, then the device build on the loaded orbitals — bit-identical
orbitals and the oracle's points."""
import numpy as np
import pytest

from oracle import restate as R

pytestmark = pytest.mark.gpu


def test_device_load_matches_host_and_builds(tmp_path, ctx):
    import torch

    from paper_2403_12340_b200 import lrgw, synth

    cfg = synth.CONFIGS["si8"]
    psi = synth.orbitals_host(cfg, seed=3)
    e = synth.energies(cfg)
    es = lrgw.ElectronicStructure(cfg.dims, cfg.cell3, psi, e, np.zeros_like(e), cfg.n_v, cfg.n_c)
    p = tmp_path / "si8.wfn1"
    lrgw.save_system(p, es)
    dims, cell, dpsi, e2, vxc, nv, nc = lrgw.load_system_device(p, ctx=ctx)
    assert (dims, nv, nc) == (tuple(cfg.dims), cfg.n_v, cfg.n_c)
    assert np.array_equal(dpsi.cpu().numpy(), psi) and np.array_equal(e2, e)
    ep = lrgw.build(dpsi[:, :nv], dpsi[:, nv:], e2, dims, cell, k_mu=8.0, n_lambda=16, ctx=ctx)
    pts = R.select_points(psi[:, :nv], psi[:, nv:], ep.n_mu)
    assert np.array_equal(ep.point_indices, pts)
    ep.close()
    torch.cuda.synchronize()
    # errors surface with the reference's messages on the device path too
    bad = tmp_path / "bad.wfn1"
    raw = p.read_bytes()
    bad.write_bytes(raw[: len(raw) // 2])
    with pytest.raises(lrgw.IoError) as ei:
        lrgw.load_system_device(bad, ctx=ctx)
    assert str(ei.value) == "load_system: truncated payload reading psi"
