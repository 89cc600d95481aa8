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


def test_elliptic_scalars_accuracy_vs_multiprecision():
    """csrc/elliptic.cpp (Carlson R_F, Gauss-transformation sn/cn/dn, addition
    theorem for complex arguments) against 40-digit values: the same accuracy
    class as the reference's AGM / sncndn recipes (elliptic.hpp:17-118)."""
    mp = pytest.importorskip("mpmath")
    mp.mp.dps = 40
    rng = np.random.default_rng(17)
    for _ in range(400):
        k, u = rng.uniform(0, 0.99), rng.uniform(-5, 5)
        m = mp.mpf(k) ** 2
        want = [float(mp.ellipfun(f, u, m=m)) for f in ("sn", "cn", "dn")]
        assert np.max(np.abs(np.array(lrgw.jacobi_sn_cn_dn(u, k)) - want)) <= 4e-15
        kk = float(mp.ellipk(m))
        assert abs(lrgw.elliptic_k(k) - kk) <= 8e-16 * kk
        y = rng.uniform(0, 0.6)
        got = lrgw.jacobi_complex(u, y, k)
        w = mp.mpc(u, y)
        for g, f in zip(got, ("sn", "cn", "dn")):
            wv = complex(mp.ellipfun(f, w, m=m))
            assert abs(g - wv) <= 1e-14 * max(1.0, abs(wv))
    # the contour height L = 1/2 int_0^{1/r} dt / sqrt((1+t^2)(1+r^2 t^2)) (contour.hpp:62-68)
    for e in ([0.0, 1.0, 4.0], [-0.5, -0.1, 0.05, 0.8], [-0.5, -0.1, 0.0, 0.8]):
        s = lrgw.elliptic_params(e, len(e) // 2 if len(e) > 3 else 1, len(e) - (len(e) // 2 if len(e) > 3 else 1),
                                 1e-7).as7()
        r = s[2]
        ell = 0.5 * mp.quad(lambda t: 1 / mp.sqrt((1 + t * t) * (1 + r * r * t * t)), [0, 1 / mp.mpf(r)])
        assert abs(s[4] - float(ell)) <= 6e-16 * float(ell)


def test_jacobi_complex_domain_and_pole_rules():
    """test_elliptic.cpp:98-102: |y| >= K(k') -> invalid_input, next to the
    pole line -> numeric_error."""
    r = 1.0 / 3.0
    kprime = lrgw.elliptic_k(math.sqrt(1.0 - r * r))
    with pytest.raises(lrgw.InvalidInput):
        lrgw.jacobi_complex(0.3, kprime * 1.01, r)
    with pytest.raises(lrgw.NumericError):
        lrgw.jacobi_complex(0.0, kprime - 1e-10, r)
    sn, cn, dn = lrgw.jacobi_sn_cn_dn(lrgw.elliptic_k(0.7), 0.7)  # sn(K) = 1 (test_elliptic.cpp:28-62)
    assert abs(sn - 1.0) <= 1e-15 and abs(cn) <= 1e-15
