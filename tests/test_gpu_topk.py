"""GPU: the selection block's candidate scan (top s+1 rows by residual desc,
position asc among the unselected positions) against a numpy sort — the
reference's strict '>' scan order (linalg.hpp:45-47) — including exact ties,
ties across the boundary, NaN residuals, fewer eligible rows than s+1 and a
boundary bin holding most of the grid (the sub-bin refinement above 2e5
rows, the chunked tie path)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _expect(d, pos, k, s1):
    idx = [r for r in range(len(d)) if pos[r] >= k and not np.isnan(d[r])]
    idx.sort(key=lambda r: (-d[r], pos[r]))
    rows = np.full(s1, -1, np.int32)
    rows[:min(s1, len(idx))] = idx[:s1]
    return rows


def _run(d, pos, k, s1):
    import torch

    from paper_2403_12340_b200 import lrgw

    dd = torch.from_numpy(np.ascontiguousarray(d)).cuda()
    pp = torch.from_numpy(np.ascontiguousarray(pos.astype(np.int32))).cuda()
    rows, vals, poss = lrgw.select_topk_dev(dd, pp, k, s1)
    return rows, vals, poss


@pytest.mark.parametrize("n_r,k,s1,mode", [
    (110592, 0, 129, "random"), (110592, 5000, 129, "random"), (4096, 100, 65, "ties"),
    (50000, 0, 129, "allequal"), (300, 250, 129, "few"), (20000, 10, 33, "nan"), (1, 0, 1, "random"),
    (70000, 0, 129, "boundary"), (12345, 7, 129, "negative"),
    # above 2e5 rows an over-full boundary bin is refined by the next 12 key
    # bits (split: "boundary"; exact ties defeat it and take the chunked scan)
    (300000, 0, 129, "boundary"), (300000, 1000, 129, "ties"), (300000, 0, 129, "allequal"),
    (900000, 300, 129, "random")])
def test_topk_matches_sort(n_r, k, s1, mode):
    rng = np.random.default_rng(n_r + k + s1)
    pos = rng.permutation(n_r).astype(np.int32)
    if mode == "random":
        d = rng.random(n_r) * 10.0
    elif mode == "ties":
        d = rng.integers(0, 7, n_r).astype(np.float64)
    elif mode == "allequal":
        d = np.full(n_r, 3.25)
    elif mode == "few":
        d = rng.random(n_r)
    elif mode == "nan":
        d = rng.random(n_r)
        d[rng.choice(n_r, 500, replace=False)] = np.nan
    elif mode == "boundary":
        # most rows within one ~3% bin just below a few large ones
        d = 1.0 + rng.random(n_r) * 1e-3
        d[:50] = 5.0 + rng.random(50)
    else:
        d = rng.standard_normal(n_r)
    rows, vals, poss = _run(d, pos, k, s1)
    want = _expect(d, pos, k, s1)
    assert np.array_equal(rows, want)
    live = want >= 0
    assert np.array_equal(vals[live], d[want[live]])
    assert np.array_equal(poss[live], pos[want[live]])
