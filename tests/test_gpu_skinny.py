"""GPU: the probe-apply streams over Theta (skinny.cu, the K7 passes of
smw.hpp:97-103) through lrgw_dev_dgemm's probe-shaped dispatch — the
bulk-copy kernels (even rows, 16-byte aligned columns) and the load-to-use
kernels (odd rows, LRGW_TN_BULK=0 / LRGW_NN_BULK=0) — for every supported
probe width, against a float64 numpy product. Tolerance 1e-13 relative: the
only difference is the FMA summation order over rows / columns."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-13


def _cm(t):
    return t.t().contiguous().t()


def _check(n_r, n_mu, m, seed):
    import torch

    from paper_2403_12340_b200 import lrgw

    rng = np.random.default_rng(seed)
    th = rng.standard_normal((n_r, n_mu))
    x = rng.standard_normal((n_r, m))
    w = rng.standard_normal((n_mu, m))
    th_d = _cm(torch.from_numpy(th).cuda())
    u = _cm(torch.empty(n_mu, m, dtype=torch.float64, device="cuda"))
    lrgw.dgemm_dev("T", "N", 1.0, th_d, _cm(torch.from_numpy(x).cuda()), 0.0, u)
    z = _cm(torch.empty(n_r, m, dtype=torch.float64, device="cuda"))
    lrgw.dgemm_dev("N", "N", 1.0, th_d, _cm(torch.from_numpy(w).cuda()), 0.0, z)
    u_ref, z_ref = th.T @ x, th @ w
    eu = np.abs(u.cpu().numpy() - u_ref).max() / np.abs(u_ref).max()
    ez = np.abs(z.cpu().numpy() - z_ref).max() / np.abs(z_ref).max()
    return eu, ez


@pytest.mark.parametrize("m", [1, 2, 4, 8, 16])
@pytest.mark.parametrize("n_r", [20480, 20481, 513])
def test_skinny_streams(m, n_r):
    n_mu = 200  # ragged against the 16 / 32-column stages
    eu, ez = _check(n_r, n_mu, m, seed=m * 1000 + n_r)
    assert eu <= TOL and ez <= TOL, (eu, ez)


def test_skinny_load_to_use_kernels():
    """The non-bulk kernels on even rows too (forced through the env)."""
    here = os.path.dirname(os.path.abspath(__file__))
    code = ("import sys; sys.path[:0] = [%r, %r]; from test_gpu_skinny import _check; "
            "r = [_check(8192, 96, m, m) for m in (1, 8, 16)]; "
            "assert all(a <= %r and b <= %r for a, b in r), r; print('ok')" % (here, os.path.dirname(here), TOL, TOL))
    env = dict(os.environ, LRGW_TN_BULK="0", LRGW_NN_BULK="0")
    p = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0 and "ok" in p.stdout, p.stdout + p.stderr
