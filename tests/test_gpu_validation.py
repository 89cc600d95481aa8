"""GPU: the reference's `validate` suite re-pointed at the B200 path
(tests/validation.py; driver.hpp:331-711) on the reference's default
validation system, plus its mutation test (test_driver.cpp: flipping the
sign of sigma_sex_x must fail gw.pipeline_equivalence)."""
import json

import pytest

pytestmark = pytest.mark.gpu


def test_validation_suite_passes(ref, ctx, tmp_path):
    from paper_2403_12340_b200 import driver
    from validation import run_validation

    cfg = driver.parse_config({})  # the reference's default system: 8^3 grid, 16 + 16 bands, k = 8
    res = run_validation(cfg, ctx)
    failed = [c for c in res["checks"] if not c["pass"]]
    assert res["pass"], failed
    names = {c["name"] for c in res["checks"]}
    assert {"smw.lu_equivalence", "smw.residual", "gw.pipeline_equivalence", "contour.direct_equivalence",
            "definiteness.K", "isdf.k_trend_monotone", "contour.threshold_insensitivity"} <= names
    assert len(res["sweeps"]["k"]) == 5 and res["sweeps"]["nodes"]
    (tmp_path / "validate_result.json").write_text(json.dumps(res, indent=1))


def test_validation_catches_the_sign_mutation(ref, ctx):
    from paper_2403_12340_b200 import driver
    from validation import run_validation

    cfg = driver.parse_config({"_test_hooks": {"flip_sex_x_sign": True}})
    res = run_validation(cfg, ctx)
    by = {c["name"]: c for c in res["checks"]}
    assert not res["pass"] and not by["gw.pipeline_equivalence"]["pass"]
    assert by["smw.lu_equivalence"]["pass"]
