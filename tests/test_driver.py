"""CPU: the driver's configuration schema, the synthetic-system recipe and the
scale helpers (paper_2403_12340_b200/driver.py) against the reference's
driver.hpp / model.hpp (oracle/_ref)."""
import json

import numpy as np
import pytest

from paper_2403_12340_b200 import driver, lrgw


def test_config_defaults_and_round_trip():
    c = driver.parse_config({})
    assert (c.dims, c.n_v, c.n_c, c.k_vc, c.delta_rel, c.max_nodes, c.pipeline) == \
        ((8, 8, 8), 16, 16, 8.0, 1e-7, 1025, "lowrank")
    j = {"system": {"seed": 3, "dims": [8, 8, 4], "cell": [5.0, 5.0, 4.5], "nv": 8, "nc": 6, "gap": 0.5,
                    "bandwidth": 2.0},
         "isdf": {"k_vc": 6.0, "k_vn": 7.0, "k_nn": 5.5, "selector": "qrcp_direct"},
         "contour": {"delta_rel": 1e-6, "max_nodes": 65}, "pipeline": "lowrank", "threads": 2}
    c = driver.parse_config(j)
    assert driver.config_to_json(c) == j


@pytest.mark.parametrize("cfg,msg", [
    ({"isdf": {"k_vc": 0.0}}, "config: ISDF coefficients must be > 0"),
    ({"contour": {"delta_rel": 0.5}}, "config: delta_rel must lie in (0, 0.5)"),
    ({"contour": {"max_nodes": 32}}, "config: max_nodes must allow at least two levels (>= 33)"),
    ({"threads": 0}, "config: threads must be >= 1"),
    ({"pipeline": "dense"}, "config: unknown pipeline 'dense'"),
    ({"isdf": {"selector": "greedy"}}, "config: unknown selector 'greedy'"),
    ({"system": {"wfn": "/nonexistent/x.wfn1"}}, "config: wavefunction file does not exist: /nonexistent/x.wfn1"),
])
def test_config_validation_messages(cfg, msg):
    """driver.hpp:103-120 (same checks, same text)."""
    with pytest.raises(lrgw.InvalidInput) as ei:
        driver.parse_config(cfg)
    assert str(ei.value) == msg


def test_config_type_errors_and_files(tmp_path):
    with pytest.raises(lrgw.InvalidInput, match="^config: malformed field"):
        driver.parse_config({"system": {"nv": "16"}})
    with pytest.raises(lrgw.InvalidInput, match="^config: cannot open"):
        driver.load_config(tmp_path / "none.json")
    p = tmp_path / "bad.json"
    p.write_text("{not json")
    with pytest.raises(lrgw.InvalidInput, match="^config: invalid JSON"):
        driver.load_config(p)
    p.write_text(json.dumps({"system": {"nv": 4}}))
    assert driver.load_config(p).n_v == 4


@pytest.mark.parametrize("seed,dims,nv,nc,gap,bw", [
    (3, (8, 8, 8), 16, 16, 1.0, 4.0), (7, (8, 8, 4), 8, 8, 1.0, 4.0), (9, (4, 4, 4), 1, 1, 1.0, 1.0),
    (1, (6, 4, 5), 3, 2, 0.5, 2.0)])
def test_synthetic_system_matches_reference(ref, seed, dims, nv, nc, gap, bw):
    """model.hpp:56-116: PCG32 stream, Box-Muller pairs, band-limited fields,
    QRCP orthonormalisation — equal to the reference to rounding."""
    psi, e = ref.build_synthetic(seed, dims, (6.0, 6.0, 6.0), nv, nc, gap, bw)
    es = driver.synthetic_system(seed, dims, (6.0, 6.0, 6.0), nv, nc, gap, bw)
    assert np.max(np.abs(es.psi - psi)) <= 1e-12 * np.max(np.abs(psi))
    assert np.array_equal(es.energies, e)
    with pytest.raises(lrgw.InvalidInput):
        driver.synthetic_system(1, (4, 4, 4), (6.0,) * 3, 1, 1, 0.0, 1.0)
    with pytest.raises(lrgw.InvalidInput):
        driver.synthetic_system(1, (2, 2, 2), (6.0,) * 3, 5, 4, 1.0, 2.0)


def test_scale_helpers():
    """driver.hpp:737-761."""
    assert driver.dims_for_points(128) == (8, 4, 4)
    assert driver.dims_for_points(512) == (8, 8, 8)
    assert driver.dims_for_points(100) == (8, 4, 4)
    pts = [(n, 3e-6 * n ** 3) for n in (8, 16, 32, 64)]
    assert abs(driver.loglog_slope(pts) - 3.0) < 1e-12
    with pytest.raises(lrgw.InvalidInput):
        driver.run_scale(driver.RunConfig(), [])
    with pytest.raises(lrgw.InvalidInput):
        driver.run_scale(driver.RunConfig(), [16, 8])


def test_dense_pipelines_refused():
    with pytest.raises(lrgw.Unsupported):
        driver.run_pipeline(driver.parse_config({"pipeline": "bruteforce"}))
