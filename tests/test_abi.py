"""CPU: the C-ABI library loads, exports every symbol include/lrgw_cuda.h
declares, and its host-scalar entry points (contour geometry, num_aux,
Coulomb kernel) agree with the oracle restatement — no GPU compute calls."""
import ctypes
import math

import numpy as np
import pytest

from oracle import restate as R
from paper_2403_12340_b200 import _lib, lrgw


def test_exports_every_declared_symbol():
    lib = _lib.load()
    declared = _lib.header_symbols()
    assert len(declared) >= 40
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    assert lib.lrgw_abi_version() == 2


def test_num_aux_matches_oracle():
    for k in (1.0, 2.5, 8.0, 12.0):
        for n1, n2 in ((16, 16), (128, 128), (120, 120), (7, 9), (1, 1)):
            assert lrgw.num_aux(k, n1, n2) == R.num_aux(k, n1, n2)
    with pytest.raises(lrgw.InvalidInput):
        lrgw.num_aux(0.0, 4, 4)


def test_elliptic_scalars_match_oracle():
    for r in (0.0, 1 / 3, 0.5, 0.9, 0.99):
        assert lrgw.elliptic_k(r) == pytest.approx(R.elliptic_k(r), rel=1e-15)
    rng = np.random.default_rng(3)
    for _ in range(50):
        k, u = rng.uniform(0, 0.97), rng.uniform(-4, 4)
        assert np.allclose(lrgw.jacobi_sn_cn_dn(u, k), R.jacobi_sn_cn_dn(u, k), rtol=1e-14, atol=1e-15)
        y = rng.uniform(0, 0.5)
        got = lrgw.jacobi_complex(u, y, k)
        want = R.jacobi_complex(u, y, k)
        for g, w in zip(got, want):
            assert abs(g - w) <= 1e-13 * max(1.0, abs(w))
    with pytest.raises(lrgw.InvalidInput):
        lrgw.elliptic_k(1.0)


@pytest.mark.parametrize("e,n_v,n_c", [([0.0, 1.0, 4.0], 1, 2), ([-0.5, -0.1, 0.05, 0.8], 2, 2),
                                       ([0.0, 2.0], 1, 1)])
def test_elliptic_params_match_oracle(e, n_v, n_c):
    got = lrgw.elliptic_params(e, n_v, n_c, 1e-7).as7()
    want = R.elliptic_params(e, n_v, n_c, 1e-7).as7()
    assert np.allclose(got, want, rtol=1e-14, atol=0)
    with pytest.raises(lrgw.InvalidInput):
        lrgw.elliptic_params([0.0, 0.0, 1.0], 1, 2, 1e-7)


def test_cauchy_bound_matches_oracle():
    s = lrgw.ContourSpec(q=1.0, big_q=math.exp(2.0))
    assert lrgw.cauchy_error_bound(s, 10) == pytest.approx(R.cauchy_error_bound(1.0, math.exp(2.0), 10), rel=1e-15)
    with pytest.raises(lrgw.InvalidInput):
        lrgw.cauchy_error_bound(s, 0)


@pytest.mark.parametrize("dims,cell", [((4, 4, 4), (5.0, 5.0, 5.0)), ((5, 6, 7), (5.0, 6.5, 7.25))])
def test_coulomb_kernel_matches_oracle(dims, cell):
    assert np.allclose(lrgw.coulomb_kernel(dims, cell), R.coulomb_kernel(dims, cell), rtol=1e-15, atol=0)
    with pytest.raises(lrgw.InvalidInput):
        lrgw.coulomb_kernel((1, 4, 4), cell)


def test_null_context_is_rejected():
    lib = _lib.load()
    pts = np.zeros(4, dtype=np.int32)
    a = np.zeros((8, 2))
    rc = lib.lrgw_select_interpolation_points(None, a.ctypes.data_as(_lib.c_double_p),
                                              a.ctypes.data_as(_lib.c_double_p), 8, 2, 2, 4, 0,
                                              pts.ctypes.data_as(_lib.c_int32_p))
    assert rc == 1
