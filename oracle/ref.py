"""oracle/ref.py — TEST INFRASTRUCTURE ONLY (the checker, never the product).

ctypes bindings to oracle/_ref/libref_lrgw.so: the unmodified reference `lrgw`
headers compiled behind oracle/ref_shim.cpp (see oracle/Makefile). Functions
take/return numpy arrays (column-major float64 on the C side) and raise the
oracle.restate exception mirror of the reference taxonomy.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from . import restate as R

_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_ref", "libref_lrgw.so")
_lib = None

_DP = ctypes.POINTER(ctypes.c_double)
_IP = ctypes.POINTER(ctypes.c_int)


def available() -> bool:
    return os.path.exists(_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise RuntimeError(f"{_PATH} missing: run `make -C oracle` where /root/reference exists")
        _lib = ctypes.CDLL(_PATH)
    return _lib


def _f(a, dtype=np.float64):
    return np.asfortranarray(a, dtype=dtype)


def _d(a):
    return a.ctypes.data_as(_DP)


def _i(a):
    return a.ctypes.data_as(_IP)


def _check(rc, what=""):
    if rc == 0:
        return
    exc = {1: R.InvalidInput, 2: R.GuardExceeded, 3: R.NumericError, 6: R.OracleError}.get(rc)
    if rc == 4:
        raise R.SingularMatrix(f"reference {what}", lib().ref_last_pivot())
    if rc == 5:
        raise R.ContourConvergenceError(f"reference {what}", None)
    if exc is None:
        raise R.OracleError(f"reference {what}: status {rc}")
    raise exc(f"reference {what}")


def gaussian(seed: int, rows: int, cols: int) -> np.ndarray:
    out = np.zeros((rows, cols), order="F")
    _check(lib().ref_gaussian(ctypes.c_uint64(seed), rows, cols, _d(out)), "gaussian")
    return out


def uniform(seed: int, n: int, lo: float, hi: float) -> np.ndarray:
    out = np.zeros(n)
    _check(lib().ref_uniform(ctypes.c_uint64(seed), n, ctypes.c_double(lo), ctypes.c_double(hi), _d(out)),
           "uniform")
    return out


def build_synthetic(seed, dims, cell, n_v, n_c, gap, bandwidth):
    n_r = int(np.prod(dims))
    psi = np.zeros((n_r, n_v + n_c), order="F")
    e = np.zeros(n_v + n_c)
    d = np.array(dims, dtype=np.int32)
    c = np.array(cell, dtype=np.float64)
    _check(lib().ref_build_synthetic(ctypes.c_uint64(seed), _i(d), _d(c), n_v, n_c, ctypes.c_double(gap),
                                     ctypes.c_double(bandwidth), _d(psi), _d(e)), "build_synthetic_system")
    return psi, e


def num_aux(k, n1, n2) -> int:
    out = ctypes.c_int(0)
    _check(lib().ref_num_aux(ctypes.c_double(k), n1, n2, ctypes.byref(out)), "num_aux")
    return out.value


def qrcp(a):
    a = _f(a)
    m, n = a.shape
    perm = np.zeros(n, dtype=np.int32)
    rd = np.zeros(min(m, n))
    _check(lib().ref_qrcp(_d(a), m, n, _i(perm), _d(rd)), "qrcp")
    return perm, rd


def select_points(a, b, n_mu, sketched=False):
    a, b = _f(a), _f(b)
    pts = np.zeros(n_mu, dtype=np.int32)
    _check(lib().ref_select_points(_d(a), _d(b), a.shape[0], a.shape[1], b.shape[1], n_mu,
                                   1 if sketched else 0, _i(pts)), "select_interpolation_points")
    return pts


def fit(a, b, pts):
    a, b = _f(a), _f(b)
    pts = np.ascontiguousarray(pts, dtype=np.int32)
    theta = np.zeros((a.shape[0], pts.size), order="F")
    _check(lib().ref_fit(_d(a), _d(b), a.shape[0], a.shape[1], b.shape[1], _i(pts), pts.size, _d(theta)),
           "fit_auxiliary_basis")
    return theta


def isdf_error(a, b, pts, theta) -> float:
    a, b, theta = _f(a), _f(b), _f(theta)
    pts = np.ascontiguousarray(pts, dtype=np.int32)
    out = ctypes.c_double(0)
    _check(lib().ref_isdf_error(_d(a), _d(b), a.shape[0], a.shape[1], b.shape[1], _i(pts), pts.size,
                                _d(theta), ctypes.byref(out)), "isdf_reconstruction_error")
    return out.value


def elliptic_k(k):
    out = ctypes.c_double(0)
    _check(lib().ref_elliptic_k(ctypes.c_double(k), ctypes.byref(out)), "elliptic_k")
    return out.value


def jacobi(u, k):
    out = np.zeros(3)
    _check(lib().ref_jacobi(ctypes.c_double(u), ctypes.c_double(k), _d(out)), "jacobi_sn_cn_dn")
    return tuple(out)


def jacobi_complex(x, y, k):
    out = np.zeros(6)
    _check(lib().ref_jacobi_complex(ctypes.c_double(x), ctypes.c_double(y), ctypes.c_double(k), _d(out)),
           "jacobi_complex")
    return complex(out[0], out[1]), complex(out[2], out[3]), complex(out[4], out[5])


def elliptic_params(e, n_v, n_c, delta_rel=1e-7, max_nodes=1025):
    e = np.ascontiguousarray(e, dtype=np.float64)
    out = np.zeros(7)
    _check(lib().ref_elliptic_params(_d(e), e.size, n_v, n_c, ctypes.c_double(delta_rel), max_nodes, _d(out)),
           "elliptic_params")
    return out


def cauchy_error_bound(q, big_q, n):
    out = ctypes.c_double(0)
    _check(lib().ref_cauchy_error_bound(ctypes.c_double(q), ctypes.c_double(big_q), n, ctypes.byref(out)),
           "cauchy_error_bound")
    return out.value


def coupled_direct(pv, pc, e):
    pv, pc = _f(pv), _f(pc)
    e = np.ascontiguousarray(e, dtype=np.float64)
    t = np.zeros((pv.shape[0], pv.shape[0]), order="F")
    _check(lib().ref_coupled_direct(_d(pv), _d(pc), pv.shape[0], pv.shape[1], pc.shape[1], _d(e), e.size,
                                    _d(t)), "coupled_coefficients_direct")
    return t


def node_term(pv, pc, e, spec7, t_node):
    pv, pc = _f(pv), _f(pc)
    e = np.ascontiguousarray(e, dtype=np.float64)
    s = np.ascontiguousarray(spec7, dtype=np.float64)
    out = np.zeros((pv.shape[0], pv.shape[0]), order="F")
    _check(lib().ref_node_term(_d(pv), _d(pc), pv.shape[0], pv.shape[1], pc.shape[1], _d(e), e.size, _d(s),
                               ctypes.c_double(t_node), _d(out)), "contour_node_term")
    return out


def sum_node_terms(pv, pc, e, spec7, nodes, weights, threads=1):
    pv, pc = _f(pv), _f(pc)
    e = np.ascontiguousarray(e, dtype=np.float64)
    s = np.ascontiguousarray(spec7, dtype=np.float64)
    nodes = np.ascontiguousarray(nodes, dtype=np.float64)
    weights = np.ascontiguousarray(weights, dtype=np.float64)
    out = np.zeros((pv.shape[0], pv.shape[0]), order="F")
    _check(lib().ref_sum_node_terms(_d(pv), _d(pc), pv.shape[0], pv.shape[1], pc.shape[1], _d(e), e.size,
                                    _d(s), _d(nodes), _d(weights), nodes.size, threads, _d(out)),
           "sum_node_terms")
    return out


def coupled_contour(pv, pc, e, delta_rel=1e-7, max_nodes=1025, threads=1):
    """Returns (T, nodes_used, est_rel, status) — status 5 carries the best."""
    pv, pc = _f(pv), _f(pc)
    e = np.ascontiguousarray(e, dtype=np.float64)
    t = np.zeros((pv.shape[0], pv.shape[0]), order="F")
    nu = ctypes.c_int(0)
    est = ctypes.c_double(0)
    rc = lib().ref_coupled_contour(_d(pv), _d(pc), pv.shape[0], pv.shape[1], pc.shape[1], _d(e), e.size,
                                   ctypes.c_double(delta_rel), max_nodes, threads, _d(t), ctypes.byref(nu),
                                   ctypes.byref(est))
    if rc not in (0, 5):
        _check(rc, "coupled_coefficients_contour")
    return t, nu.value, est.value, rc


def coulomb_kernel(dims, cell):
    d = np.array(dims, dtype=np.int32)
    c = np.array(cell, dtype=np.float64)
    out = np.zeros(int(np.prod(dims)))
    _check(lib().ref_coulomb_kernel(_i(d), _d(c), _d(out)), "build_coulomb")
    return out


def apply_coulomb(dims, cell, x, threads=1, zero=False):
    x = _f(x)
    d = np.array(dims, dtype=np.int32)
    c = np.array(cell, dtype=np.float64)
    y = np.zeros_like(x, order="F")
    _check(lib().ref_apply_coulomb(_i(d), _d(c), 1 if zero else 0, _d(x), x.shape[1], threads, _d(y)),
           "apply_coulomb")
    return y


def assemble_K(t, p, dims, cell, threads=1, zero=False):
    t, p = _f(t), _f(p)
    d = np.array(dims, dtype=np.int32)
    c = np.array(cell, dtype=np.float64)
    k = np.zeros_like(t, order="F")
    _check(lib().ref_assemble_K(_d(t), _d(p), p.shape[0], p.shape[1], _i(d), _d(c), 1 if zero else 0, threads,
                                _d(k)), "assemble_K")
    return k


def build_and_apply(t, p, dims, cell, x=None, threads=1, want_vp=False):
    t, p = _f(t), _f(p)
    d = np.array(dims, dtype=np.int32)
    c = np.array(cell, dtype=np.float64)
    k = np.zeros_like(t, order="F")
    vp = np.zeros_like(p, order="F") if want_vp else None
    if x is not None:
        x = _f(x)
        y = np.zeros_like(x, order="F")
        xp, yp, m = _d(x), _d(y), x.shape[1]
    else:
        y, xp, yp, m = None, None, None, 0
    _check(lib().ref_build_and_apply(_d(t), _d(p), p.shape[0], p.shape[1], _i(d), _d(c), threads, xp, m, yp,
                                     _d(k), _d(vp) if want_vp else None), "build_epsilon_inverse")
    return y, k, vp


def eps_apply_given(p, k, dims, cell, x):
    p, k, x = _f(p), _f(k), _f(x)
    d = np.array(dims, dtype=np.int32)
    c = np.array(cell, dtype=np.float64)
    y = np.zeros_like(x, order="F")
    _check(lib().ref_eps_apply_given(_d(p), _d(k), p.shape[0], p.shape[1], _i(d), _d(c), _d(x), x.shape[1],
                                     _d(y)), "epsilon_inverse_apply")
    return y


def epsilon_dense(psi, n_v, n_c, energies, dims, cell, pts, theta):
    psi, theta = _f(psi), _f(theta)
    e = np.ascontiguousarray(energies, dtype=np.float64)
    d = np.array(dims, dtype=np.int32)
    c = np.array(cell, dtype=np.float64)
    pts = np.ascontiguousarray(pts, dtype=np.int32)
    n_r = psi.shape[0]
    eps = np.zeros((n_r, n_r), order="F")
    inv = np.zeros((n_r, n_r), order="F")
    _check(lib().ref_epsilon_dense(_d(psi), n_r, n_v, n_c, _d(e), _i(d), _d(c), _i(pts), pts.size, _d(theta),
                                   _d(eps), _d(inv)), "epsilon_dense_oracle")
    return eps, inv


def sym_eig_values(a):
    a = _f(a)
    out = np.zeros(a.shape[0])
    _check(lib().ref_sym_eig_values(_d(a), a.shape[0], _d(out)), "sym_eig")
    return out


def matmul_tn(a, b):
    a, b = _f(a), _f(b)
    c = np.zeros((a.shape[1], b.shape[1]), order="F")
    _check(lib().ref_matmul_tn(_d(a), a.shape[0], a.shape[1], _d(b), b.shape[1], _d(c)), "matmul_tn")
    return c


def lu_solve(a, b):
    a, b = _f(a), _f(b)
    x = np.zeros_like(b, order="F")
    _check(lib().ref_lu_solve(_d(a), a.shape[0], _d(b), b.shape[1], _d(x)), "lu_solve")
    return x


def project_screened(t, p, dims, cell, p_vn, p_nn, zero=False):
    """gw.hpp:73-88 through the reference: (w_vn, w_nn, v_vn)."""
    t, p, p_vn, p_nn = _f(t), _f(p), _f(p_vn), _f(p_nn)
    d = np.array(dims, dtype=np.int32)
    c = np.array(cell, dtype=np.float64)
    n_vn, n_nn = p_vn.shape[1], p_nn.shape[1]
    w_vn = np.zeros((n_vn, n_vn), order="F")
    w_nn = np.zeros((n_nn, n_nn), order="F")
    v_vn = np.zeros((n_vn, n_vn), order="F")
    _check(lib().ref_project_screened(_d(t), _d(p), p.shape[0], p.shape[1], _i(d), _d(c), 1 if zero else 0,
                                      _d(p_vn), n_vn, _d(p_nn), n_nn, _d(w_vn), _d(w_nn), _d(v_vn)),
           "project_screened_interactions")
    return w_vn, w_nn, v_vn


def sigma_lowrank(psi, n_v, pts_vn, pts_nn, w_vn, w_nn, v_vn):
    """gw.hpp:143-153 on given projections: (sex_x, x, coh, total)."""
    psi = _f(psi)
    n_r, nb = psi.shape
    pv = _i(np.ascontiguousarray(pts_vn, dtype=np.int32))
    pn = _i(np.ascontiguousarray(pts_nn, dtype=np.int32))
    out = np.zeros(4 * nb)
    _check(lib().ref_sigma_lowrank(_d(psi), n_r, n_v, nb - n_v, pv, len(pts_vn), pn, len(pts_nn), _d(_f(w_vn)),
                                   _d(_f(w_nn)), _d(_f(v_vn)), _d(out)), "self_energies_lowrank")
    return tuple(out.reshape(4, nb))


def self_energies(psi, n_v, dims, cell, energies, pts_vc, pts_vn, pts_nn, which="lowrank"):
    """The gw.hpp pipelines on fixed point sets (test_gw.cpp:13-41):
    which = lowrank | conventional | bruteforce -> (sex_x, x, coh, total)."""
    psi = _f(psi)
    n_r, nb = psi.shape
    d = np.array(dims, dtype=np.int32)
    c = np.array(cell, dtype=np.float64)
    e = np.ascontiguousarray(energies, dtype=np.float64)
    code = {"lowrank": 0, "conventional": 1, "bruteforce": 2}[which]
    out = np.zeros(4 * nb)
    args = []
    for pts in (pts_vc, pts_vn, pts_nn):
        p = np.ascontiguousarray(pts, dtype=np.int32)
        args += [_i(p), len(p)]
    _check(lib().ref_self_energies(_d(psi), n_r, n_v, nb - n_v, _i(d), _d(c), _d(e), *args, code, _d(out)),
           "self_energies_" + which)
    return tuple(out.reshape(4, nb))


def quasiparticle(energies, vxc, sigma_total):
    """gw.hpp:48-58."""
    e = np.ascontiguousarray(energies, dtype=np.float64)
    v = np.ascontiguousarray(vxc, dtype=np.float64)
    s = np.ascontiguousarray(sigma_total, dtype=np.float64)
    out = np.zeros(e.size)
    _check(lib().ref_quasiparticle(_d(e), _d(v), _d(s), e.size, s.size, _d(out)), "quasiparticle_energies")
    return out


def save_system(path, dims, cell, n_v, n_c, psi, energies, vxc):
    """model.hpp:262-285 (the reference writer)."""
    d = np.array(dims, dtype=np.int32)
    c = np.array(cell, dtype=np.float64)
    _check(lib().ref_save_system(str(path).encode(), _i(d), _d(c), n_v, n_c, _d(_f(psi)),
                                 _d(np.ascontiguousarray(energies, dtype=np.float64)),
                                 _d(np.ascontiguousarray(vxc, dtype=np.float64))), "save_system")


def load_system(path):
    """model.hpp:287-339 (the reference reader). Returns
    (dims, cell, n_v, n_c, psi, energies, vxc); raises OracleError subclasses
    carrying the reference's io_error text."""
    L = lib()
    L.ref_last_message.restype = ctypes.c_char_p
    d = np.zeros(3, dtype=np.int32)
    c = np.zeros(3)
    nv, nc = ctypes.c_int(0), ctypes.c_int(0)
    rc = L.ref_load_system(str(path).encode(), _i(d), _d(c), ctypes.byref(nv), ctypes.byref(nc), None, None, None)
    if rc != 0:
        _check(rc, L.ref_last_message().decode())
    n_r, nb = int(np.prod(d)), nv.value + nc.value
    psi = np.zeros((n_r, nb), order="F")
    e, v = np.zeros(nb), np.zeros(nb)
    _check(L.ref_load_system(str(path).encode(), _i(d), _d(c), ctypes.byref(nv), ctypes.byref(nc), _d(psi), _d(e),
                             _d(v)), "load_system")
    return tuple(int(x) for x in d), tuple(float(x) for x in c), nv.value, nc.value, psi, e, v


def run_pipeline_json(config: dict) -> dict:
    """driver.hpp:253-329: the reference's run command on a config dict."""
    import json

    cap = 1 << 24
    buf = ctypes.create_string_buffer(cap)
    n = ctypes.c_int(0)
    _check(lib().ref_run_pipeline_json(json.dumps(config).encode(), buf, cap, ctypes.byref(n)), "run_pipeline")
    return json.loads(buf.raw[:n.value].decode())


# ---- stage-wise checkers for the large BASELINE configs (ref_shim.cpp) -----
def fit_rows(a_rows, b_rows, a_mu, b_mu, threads=1):
    """Rows of the reference fit (isdf.hpp:118-163): psi_a / psi_b at the rows
    under test and at the sorted points. Bit-identical to those rows of
    fit(a, b, pts). Returns (theta_rows, used_pinv)."""
    a_rows, b_rows, a_mu, b_mu = _f(a_rows), _f(b_rows), _f(a_mu), _f(b_mu)
    out = np.zeros((a_rows.shape[0], a_mu.shape[0]), order="F")
    pinv = ctypes.c_int(0)
    _check(lib().ref_fit_rows(_d(a_rows), _d(b_rows), a_rows.shape[0], _d(a_mu), _d(b_mu), a_mu.shape[0],
                              a_rows.shape[1], b_rows.shape[1], threads, _d(out), ctypes.byref(pinv)),
           "fit_auxiliary_basis (rows)")
    return out, bool(pinv.value)


def pvp_cols(p, dims, cell, cols, threads=1, want_vp=False):
    """Columns `cols` of P^T (V P) (smw.hpp:61, before symmetrisation) and
    optionally V P(:, cols) — the reference's apply_coulomb + matmul_tn."""
    p = _f(p)
    d = np.array(dims, dtype=np.int32)
    c = np.array(cell, dtype=np.float64)
    cols = np.ascontiguousarray(cols, dtype=np.int32)
    out = np.zeros((p.shape[1], cols.size), order="F")
    vp = np.zeros((p.shape[0], cols.size), order="F") if want_vp else None
    _check(lib().ref_pvp_cols(_d(p), p.shape[0], p.shape[1], _i(d), _d(c), _i(cols), cols.size, threads, _d(out),
                              _d(vp) if want_vp else None), "pvp columns")
    return (out, vp) if want_vp else out


def smw_from_pvp(t, pvp, check_eig=True, threads=1):
    """assemble_K (smw.hpp:42-73) with P^T V P supplied."""
    t, pvp = _f(t), _f(pvp)
    k = np.zeros_like(t, order="F")
    _check(lib().ref_smw_from_pvp(_d(t), _d(pvp), t.shape[0], 1 if check_eig else 0, threads, _d(k)),
           "assemble_K")
    return k


def eps_apply_vp(p, k, vp, x):
    """epsilon_inverse_apply (smw.hpp:97-103) with V P supplied."""
    p, k, vp, x = _f(p), _f(k), _f(vp), _f(x)
    y = np.zeros_like(x, order="F")
    _check(lib().ref_eps_apply_vp(_d(p), _d(k), _d(vp), p.shape[0], p.shape[1], _d(x), x.shape[1], _d(y)),
           "epsilon_inverse_apply")
    return y


def eps_apply_factored(p, k, dims, cell, x, threads=1):
    """X + V (P (K (P^T X))): smw.hpp:101-102 with V applied last."""
    p, k, x = _f(p), _f(k), _f(x)
    d = np.array(dims, dtype=np.int32)
    c = np.array(cell, dtype=np.float64)
    y = np.zeros_like(x, order="F")
    _check(lib().ref_eps_apply_factored(_d(p), _d(k), p.shape[0], p.shape[1], _i(d), _d(c), _d(x), x.shape[1],
                                        threads, _d(y)), "epsilon_inverse_apply (factored)")
    return y
