"""oracle/restate.py — TEST INFRASTRUCTURE ONLY (the checker, never the product).

CPU restatement (numpy / pure-Python scalars) of the reference `lrgw` hot path:
ISDF point selection + fit, Cauchy/elliptic-contour quadrature of the core,
Coulomb application, SMW assembly of the factored eps^-1 and its probe apply.
Every function cites the reference file:line it follows (paths relative to
/root/reference/proj/include/lrgw/). Pinned against the compiled reference
(oracle/_ref/libref_lrgw.so) and the reference's own known-answer tests in
tests/test_oracle.py.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this module.
"""
from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_REF_DIR = os.path.join(_HERE, "_ref")

PI = 3.14159265358979323846
TWO_PI = 6.283185307179586476925286766559
FOUR_PI = 12.566370614359172953850573533118


class OracleError(Exception):
    """Mirror of the reference exception taxonomy (errors.hpp:10-36)."""

    code = 9


class InvalidInput(OracleError):
    code = 1


class GuardExceeded(OracleError):
    code = 2


class NumericError(OracleError):
    code = 3


class SingularMatrix(NumericError):
    code = 4

    def __init__(self, msg, pivot):
        super().__init__(f"{msg} (pivot index {pivot})")
        self.pivot_index = pivot


class ContourConvergenceError(NumericError):
    code = 5

    def __init__(self, msg, best):
        super().__init__(msg)
        self.best = best


# ---------------------------------------------------------------------------
# ISDF (isdf.hpp)
# ---------------------------------------------------------------------------

def num_aux(k_mu: float, n1: int, n2: int) -> int:
    """isdf.hpp:42-46 — llround(k * sqrt(N1*N2)) (half away from zero)."""
    if not k_mu > 0.0:
        raise InvalidInput("num_aux: k_mu must be > 0")
    x = k_mu * math.sqrt(float(n1) * n2)
    return int(math.floor(x + 0.5))


_sel_lib = None


def _select_lib():
    global _sel_lib
    if _sel_lib is None:
        path = os.path.join(_REF_DIR, "liboracle_select.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make -C oracle`")
        lib = ctypes.CDLL(path)
        lib.oracle_select_points.restype = ctypes.c_int
        _sel_lib = lib
    return _sel_lib


def select_points(a: np.ndarray, b: np.ndarray, n_mu: int, return_diag=False):
    """isdf.hpp:95-112 + linalg.hpp:26-111 via the matrix-free greedy pivoted
    Cholesky restatement in oracle/select.c (same pivot rule, swap-mirrored
    tie-break, ascending sort). a: N_r x N1, b: N_r x N2 (any layout)."""
    a = np.asfortranarray(a, dtype=np.float64)
    b = np.asfortranarray(b, dtype=np.float64)
    n_r, n1 = a.shape
    n2 = b.shape[1]
    if n_mu > n_r:
        raise InvalidInput("select_interpolation_points: N_mu > N_r")
    if n_mu < 1:
        raise InvalidInput("select_interpolation_points: N_mu < 1")
    steps = min(n_mu, n1 * n2, n_r)
    pts = np.zeros(n_mu, dtype=np.int32)
    margins = np.zeros(max(steps, 1), dtype=np.float64)
    order = np.zeros(max(steps, 1), dtype=np.int32)
    events = ctypes.c_int(0)
    dp = ctypes.POINTER(ctypes.c_double)
    ip = ctypes.POINTER(ctypes.c_int)
    rc = _select_lib().oracle_select_points(
        a.ctypes.data_as(dp), b.ctypes.data_as(dp), n_r, n1, n2, n_mu,
        pts.ctypes.data_as(ip), margins.ctypes.data_as(dp),
        order.ctypes.data_as(ip), ctypes.byref(events))
    if rc == 1:
        raise InvalidInput("select_points: bad arguments")
    if rc != 0:
        raise RuntimeError("select_points: allocation failure")
    if return_diag:
        return pts, {"margins": margins[:steps], "order": order[:steps],
                     "recompute_events": events.value}
    return pts


def _lu_factor(a: np.ndarray):
    """linalg.hpp:123-150 — partial-pivot LU, singular when |pivot| <
    1e-14 * max|A| (128, 137). Returns (lu, piv) in LAPACK getrf form."""
    import scipy.linalg as sla

    n = a.shape[0]
    mx = float(np.max(np.abs(a))) if a.size else 0.0
    tiny = 1e-14 * (mx if mx > 0.0 else 1.0)
    lu, piv = sla.lu_factor(a, check_finite=False)
    diag = np.abs(np.diag(lu))
    bad = np.nonzero(diag < tiny)[0]
    if bad.size:
        raise SingularMatrix("lu_factor: singular matrix", int(bad[0]))
    return lu, piv


def lu_solve(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """linalg.hpp:152-179."""
    import scipy.linalg as sla

    lu, piv = _lu_factor(np.asarray(a, dtype=np.float64))
    return sla.lu_solve((lu, piv), b, check_finite=False)


def symmetrize(a: np.ndarray) -> np.ndarray:
    """matrix.hpp:192-200 — (A + A^T)/2."""
    return 0.5 * (a + a.T)


def sym_eig(a: np.ndarray):
    """linalg.hpp:310-345 — ascending eigenvalues of the symmetrised input."""
    fa = float(np.linalg.norm(a))
    defect = math.sqrt(2.0) * float(np.linalg.norm(np.tril(a, -1) - np.triu(a, 1).T))
    if defect > 1e-8 * max(fa, 1e-300):
        raise InvalidInput("sym_eig: matrix is not symmetric")
    return np.linalg.eigh(symmetrize(a))


def fit_lhs(a: np.ndarray, b: np.ndarray, pts) -> np.ndarray:
    """isdf.hpp:130-132 — lhs = (A A_mu^T) o (B B_mu^T), N_r x N_mu."""
    pts = np.asarray(pts)
    return (a @ a[pts].T) * (b @ b[pts].T)


def fit_auxiliary_basis(a: np.ndarray, b: np.ndarray, pts) -> np.ndarray:
    """isdf.hpp:118-163 — Theta (N_r x N_mu) from the Hadamard normal
    equations; LU solve, eigen pseudo-inverse fallback on a singular Gram."""
    pts = np.asarray(pts, dtype=np.int64)
    if pts.size < 1:
        raise InvalidInput("fit_auxiliary_basis: empty point set")
    if np.any(np.diff(pts) <= 0):
        raise InvalidInput("fit_auxiliary_basis: points must be distinct and sorted")
    lhs = fit_lhs(a, b, pts)
    gram = symmetrize(lhs[pts])
    try:
        return lu_solve(gram, lhs.T).T
    except SingularMatrix:
        w, q = sym_eig(gram)
        lam_max = float(np.max(np.abs(w))) if w.size else 0.0
        if lam_max <= 0.0:
            raise NumericError("fit_auxiliary_basis: degenerate Gram matrix")
        keep = np.abs(w) > 1e-12 * lam_max
        if not np.any(keep):
            raise NumericError("fit_auxiliary_basis: degenerate Gram matrix")
        inv = np.where(keep, 1.0 / np.where(keep, w, 1.0), 0.0)
        pinv = (q * inv) @ q.T
        return lhs @ pinv


def fit_rows(a_rows, b_rows, a_mu, b_mu) -> np.ndarray:
    """Rows of fit_auxiliary_basis (isdf.hpp:118-163) from the orbitals at
    those rows and at the sorted points (the fit is row-separable); LAPACK
    LU, for sizes where the reference's serial LU is out of reach."""
    gram = symmetrize((a_mu @ a_mu.T) * (b_mu @ b_mu.T))
    lhs = (a_rows @ a_mu.T) * (b_rows @ b_mu.T)
    try:
        return lu_solve(gram, lhs.T).T
    except SingularMatrix:
        w, q = sym_eig(gram)
        lam_max = float(np.max(np.abs(w))) if w.size else 0.0
        keep = np.abs(w) > 1e-12 * lam_max
        if lam_max <= 0.0 or not np.any(keep):
            raise NumericError("fit_auxiliary_basis: degenerate Gram matrix")
        inv = np.where(keep, 1.0 / np.where(keep, w, 1.0), 0.0)
        return lhs @ ((q * inv) @ q.T)


def isdf_error(a, b, pts, theta) -> float:
    """isdf.hpp:195-202 — ||M - P C||_F / ||M||_F (small sizes only)."""
    m = np.einsum("ri,rj->rji", a, b).reshape(a.shape[0], -1)
    c = m[np.asarray(pts)]
    return float(np.linalg.norm(m - theta @ c) / np.linalg.norm(m))


# ---------------------------------------------------------------------------
# Elliptic helpers (elliptic.hpp) — host scalars
# ---------------------------------------------------------------------------

def agm(a: float, b: float) -> float:
    """elliptic.hpp:17-26."""
    for _ in range(64):
        an = 0.5 * (a + b)
        bn = math.sqrt(a * b)
        if abs(an - bn) <= 1e-16 * an:
            return an
        a, b = an, bn
    return 0.5 * (a + b)


def elliptic_k(k: float) -> float:
    """elliptic.hpp:28-33."""
    if not (0.0 <= k < 1.0):
        raise InvalidInput("elliptic_k: modulus must be in [0, 1)")
    return PI / (2.0 * agm(1.0, math.sqrt((1.0 - k) * (1.0 + k))))


def jacobi_sn_cn_dn(u: float, k: float):
    """elliptic.hpp:48-85 — descending Landen (sncndn)."""
    if not (0.0 <= k < 1.0):
        raise InvalidInput("jacobi_sn_cn_dn: modulus must be in [0, 1)")
    if k < 1e-14:
        return math.sin(u), math.cos(u), 1.0
    em = [0.0] * 24
    en = [0.0] * 24
    a = 1.0
    emc = (1.0 - k) * (1.0 + k)
    c = 0.0
    l = 0
    for i in range(24):
        l = i
        em[i] = a
        emc = math.sqrt(emc)
        en[i] = emc
        c = 0.5 * (a + emc)
        if abs(a - emc) <= 1e-16 * a:
            break
        emc *= a
        a = c
    uc = u * c
    sn, cn, dn = math.sin(uc), math.cos(uc), 1.0
    if sn != 0.0:
        a = cn / sn
        c *= a
        for i in range(l, -1, -1):
            b = em[i]
            a *= c
            c *= dn
            dn = (en[i] + a) / (b + a)
            a = c / b
        a = 1.0 / math.sqrt(c * c + 1.0)
        sn = a if sn >= 0.0 else -a
        cn = c * sn
    return sn, cn, dn


def jacobi_complex(x: float, y: float, k: float):
    """elliptic.hpp:97-118 — A&S 16.21 addition formulas."""
    if not (0.0 <= k < 1.0):
        raise InvalidInput("jacobi_complex: modulus must be in [0, 1)")
    kp = math.sqrt((1.0 - k) * (1.0 + k))
    if abs(y) >= elliptic_k(kp):
        raise InvalidInput("jacobi_complex: imaginary part outside the fundamental rectangle")
    rs, rc, rd = jacobi_sn_cn_dn(x, k)
    is_, ic, id_ = jacobi_sn_cn_dn(y, kp)
    den = ic * ic + k * k * rs * rs * is_ * is_
    if abs(den) < 1e-13:
        raise NumericError("jacobi_complex: argument too close to a pole")
    sn = complex(rs * id_, rc * rd * is_ * ic) / den
    cn = complex(rc * ic, -(rs * rd * is_ * id_)) / den
    dn = complex(rd * ic * id_, -(k * k * rs * rc * is_)) / den
    return sn, cn, dn


def _gauss_legendre_rule(n: int):
    """elliptic.hpp:133-160."""
    x = [0.0] * n
    w = [0.0] * n
    m = (n + 1) // 2
    for i in range(m):
        z = math.cos(PI * (i + 0.75) / (n + 0.5))
        pp = 0.0
        for _ in range(100):
            p1, p2 = 1.0, 0.0
            for j in range(n):
                p3 = p2
                p2 = p1
                p1 = ((2.0 * j + 1.0) * z * p2 - j * p3) / (j + 1)
            pp = n * (z * p1 - p2) / (z * z - 1.0)
            z1 = z
            z = z1 - p1 / pp
            if abs(z - z1) < 1e-15:
                break
        x[i] = -z
        x[n - 1 - i] = z
        w[i] = 2.0 / ((1.0 - z * z) * pp * pp)
        w[n - 1 - i] = w[i]
    return x, w


_GL15 = None


def integrate_adaptive(f, a: float, b: float, rel_tol: float = 1e-13) -> float:
    """elliptic.hpp:162-193 — adaptive 15-point Gauss-Legendre."""
    global _GL15
    if _GL15 is None:
        _GL15 = _gauss_legendre_rule(15)
    xs, ws = _GL15

    def apply(lo, hi):
        xm, xl = 0.5 * (hi + lo), 0.5 * (hi - lo)
        s = 0.0
        for xi, wi in zip(xs, ws):
            s += wi * f(xm + xl * xi)
        return s * xl

    def adapt(lo, hi, whole, tol, depth):
        mid = 0.5 * (lo + hi)
        left = apply(lo, mid)
        right = apply(mid, hi)
        refined = left + right
        if abs(refined - whole) <= tol * max(1.0, abs(refined)) or depth >= 48:
            return refined
        return adapt(lo, mid, left, 0.5 * tol, depth + 1) + adapt(mid, hi, right, 0.5 * tol, depth + 1)

    return adapt(a, b, apply(a, b), rel_tol, 0)


# ---------------------------------------------------------------------------
# Contour quadrature (contour.hpp)
# ---------------------------------------------------------------------------

@dataclass
class ContourSpec:
    """contour.hpp:23-33."""
    q: float = 0.0
    big_q: float = 0.0
    r: float = 0.0
    big_r: float = 0.0
    l: float = 0.0
    e_shift: float = 0.0
    delta_rel: float = 1e-7
    max_nodes: int = 1025
    bypass: bool = False

    def as7(self):
        return np.array([self.q, self.big_q, self.r, self.big_r, self.l, self.e_shift,
                         1.0 if self.bypass else 0.0])


def elliptic_params(energies, n_v: int, n_c: int, delta_rel: float, max_nodes: int = 1025) -> ContourSpec:
    """contour.hpp:35-71."""
    e = list(map(float, energies))
    if n_v < 1 or n_c < 1 or n_v + n_c > len(e):
        raise InvalidInput("elliptic_params: bad band counts")
    s = ContourSpec()
    s.q = e[n_v] - e[n_v - 1]
    s.big_q = e[n_v + n_c - 1] - e[n_v - 1]
    s.e_shift = e[n_v - 1]
    s.delta_rel = delta_rel
    s.max_nodes = max_nodes
    if not s.q > 0.0:
        raise InvalidInput("elliptic_params: gap must be > 0")
    ratio = s.big_q / s.q
    if ratio <= 1.0 + 1e-12:
        s.r = 0.0
        s.big_r = elliptic_k(0.0)
        s.l = 0.0
        s.bypass = True
        return s
    sq = math.sqrt(ratio)
    s.r = (sq - 1.0) / (sq + 1.0)
    s.big_r = elliptic_k(s.r)
    r = s.r
    s.l = 0.5 * integrate_adaptive(lambda t: 1.0 / math.sqrt((1.0 + t * t) * (1.0 + r * r * t * t)),
                                   0.0, 1.0 / r)
    s.bypass = False
    return s


def cauchy_error_bound(q: float, big_q: float, n_lambda: int) -> float:
    """contour.hpp:75-80."""
    if n_lambda < 1:
        raise InvalidInput("cauchy_error_bound: N_lambda < 1")
    return math.exp(-PI * PI * n_lambda / (2.0 * math.log(big_q / q) + 6.0))


def node_geometry(spec: ContourSpec, t_node: float):
    """contour.hpp:149-157 — z(t + iL) and g = cn dn / (1/r - sn)^2."""
    sn, cn, dn = jacobi_complex(t_node, spec.l, spec.r)
    r_inv = 1.0 / spec.r
    den = r_inv - sn
    z = math.sqrt(spec.q * spec.big_q) * (r_inv + sn) / den + spec.e_shift
    g = cn * dn / (den * den)
    return z, g


def node_term(pv, pc, energies, spec: ContourSpec, t_node: float) -> np.ndarray:
    """contour.hpp:144-183 — Im(g * (Jv o Jc)) at one node (unweighted)."""
    n_v, n_c = pv.shape[1], pc.shape[1]
    z, g = node_geometry(spec, t_node)
    e = np.asarray(energies, dtype=np.float64)
    dv = 1.0 / (z - e[:n_v])
    dc = 1.0 / (z - e[n_v:n_v + n_c])
    jv_re = (pv * dv.real) @ pv.T
    jv_im = (pv * dv.imag) @ pv.T
    jc_re = (pc * dc.real) @ pc.T
    jc_im = (pc * dc.imag) @ pc.T
    j_re = jv_re * jc_re - jv_im * jc_im
    j_im = jv_re * jc_im + jv_im * jc_re
    return g.real * j_im + g.imag * j_re


def sum_node_terms(pv, pc, energies, spec, nodes, weights) -> np.ndarray:
    """contour.hpp:185-222 (serial order)."""
    acc = np.zeros((pv.shape[0], pv.shape[0]))
    for t, w in zip(nodes, weights):
        acc += w * node_term(pv, pc, energies, spec, t)
    return acc


def contour_prefactor(spec: ContourSpec) -> float:
    """contour.hpp:247-248."""
    return 2.0 * math.sqrt(spec.q * spec.big_q) / (PI * spec.r)


def trapezoid_nodes(spec: ContourSpec, n_intervals: int):
    """Closed trapezoid on [-R, R]: n+1 nodes, end weights h/2 — the level
    construction of contour.hpp:253-264 at an arbitrary interval count."""
    h = 2.0 * spec.big_r / n_intervals
    nodes = [-spec.big_r + k * h for k in range(n_intervals + 1)]
    weights = [0.5 * h if k in (0, n_intervals) else h for k in range(n_intervals + 1)]
    return nodes, weights


def coupled_coefficients_fixed(pv, pc, energies, spec: ContourSpec, n_lambda: int) -> np.ndarray:
    """Fixed-N_lambda quadrature (BASELINE configs): pref * trapezoid sum,
    symmetrised (contour.hpp:270-276)."""
    nodes, weights = trapezoid_nodes(spec, n_lambda)
    return symmetrize(contour_prefactor(spec) * sum_node_terms(pv, pc, energies, spec, nodes, weights))


def coupled_coefficients_direct(pv, pc, energies) -> np.ndarray:
    """contour.hpp:114-137 — exact sum over (i, j)."""
    n_v, n_c = pv.shape[1], pc.shape[1]
    if pv.shape[0] != pc.shape[0]:
        raise InvalidInput("coupled_coefficients: point-row mismatch")
    if n_v + n_c > len(energies):
        raise InvalidInput("coupled_coefficients: not enough energies")
    e = np.asarray(energies, dtype=np.float64)
    t = np.zeros((pv.shape[0], pv.shape[0]))
    for i in range(n_v):
        d = 1.0 / (e[i] - e[n_v:n_v + n_c])
        w = (pc * d) @ pc.T
        vi = pv[:, i]
        t += np.outer(vi, vi) * w
    return symmetrize(t)


def contour_levels(pv, pc, energies, spec: ContourSpec, max_level_nodes: int):
    """contour.hpp:235-294 — nested 2^m+1 trapezoid levels, m = 4, 5, ..."""
    if spec.bypass:
        raise InvalidInput("contour quadrature: spec is bypass-flagged; use the direct sum")
    if 17 > max_level_nodes:
        raise InvalidInput("contour quadrature: node cap below one level")
    pref = contour_prefactor(spec)
    running = None
    out = []
    m = 4
    while True:
        n_nodes = (1 << m) + 1
        if n_nodes > max_level_nodes:
            break
        h = 2.0 * spec.big_r / (n_nodes - 1)
        if running is None:
            nodes = [-spec.big_r + k * h for k in range(n_nodes)]
            weights = [0.5 * h if k in (0, n_nodes - 1) else h for k in range(n_nodes)]
            running = sum_node_terms(pv, pc, energies, spec, nodes, weights)
        else:
            nodes = [-spec.big_r + k * h for k in range(1, n_nodes, 2)]
            weights = [h] * len(nodes)
            running = 0.5 * running + sum_node_terms(pv, pc, energies, spec, nodes, weights)
        out.append((n_nodes, symmetrize(pref * running)))
        m += 1
    return out


def coupled_coefficients_contour(pv, pc, energies, spec: ContourSpec):
    """contour.hpp:298-329 — adaptive refinement; returns (T, nodes_used, est)."""
    prev = None
    best = None
    for n_nodes, t in contour_levels(pv, pc, energies, spec, spec.max_nodes):
        if prev is None:
            best = (t, n_nodes, 1.0)
            prev = t
            continue
        scale = max(float(np.linalg.norm(t)), 1e-300)
        rel = float(np.linalg.norm(t - prev)) / scale
        best = (t, n_nodes, rel)
        prev = t
        if rel <= spec.delta_rel:
            return best
    raise ContourConvergenceError(
        "coupled_coefficients_contour: did not reach delta_rel within max_nodes", best)


# ---------------------------------------------------------------------------
# Coulomb (grid.hpp, model.hpp) and SMW (smw.hpp)
# ---------------------------------------------------------------------------

def coulomb_kernel(dims, cell) -> np.ndarray:
    """grid.hpp:30-42 + model.hpp:165-175 — v(G) = 4pi/|G|^2, v(0) = 0, flat
    index i1 + n1*(i2 + n2*i3)."""
    n1, n2, n3 = dims

    def freq(n):
        k = np.arange(n)
        return np.where(k <= n // 2, k, k - n).astype(np.float64)

    g1 = TWO_PI * freq(n1) / cell[0]
    g2 = TWO_PI * freq(n2) / cell[1]
    g3 = TWO_PI * freq(n3) / cell[2]
    g2sum = (g1[None, None, :] ** 2 + g2[None, :, None] ** 2 + g3[:, None, None] ** 2).reshape(-1)
    with np.errstate(divide="ignore"):
        v = np.where(g2sum > 0.0, FOUR_PI / np.where(g2sum > 0.0, g2sum, 1.0), 0.0)
    return v


def apply_coulomb(dims, cell, x: np.ndarray, kernel=None) -> np.ndarray:
    """model.hpp:208-223 — Re(F^-1 diag(v) F x) with the unitary 3-D DFT
    (dft.hpp:37-68) applied column by column."""
    n1, n2, n3 = dims
    n_r = n1 * n2 * n3
    x = np.asarray(x, dtype=np.float64)
    if x.shape[0] != n_r:
        raise InvalidInput("apply_coulomb: row count != N_r")
    v = coulomb_kernel(dims, cell) if kernel is None else kernel
    out = np.empty_like(x)
    vv = v.reshape(n3, n2, n1)
    for j in range(x.shape[1]):
        f = x[:, j].reshape(n3, n2, n1)
        out[:, j] = np.fft.ifftn(vv * np.fft.fftn(f)).real.reshape(-1)
    return out


def assemble_K(t: np.ndarray, p: np.ndarray, dims, cell, kernel=None) -> np.ndarray:
    """smw.hpp:42-73 — K = (T^-1/2 - P^T V P)^-1, each step symmetrised."""
    if t.shape[0] != t.shape[1] or t.shape[0] != p.shape[1]:
        raise InvalidInput("assemble_K: T / P_vc shape mismatch")
    w, _ = sym_eig(t)
    if not w[-1] < 0.0:
        raise NumericError("assemble_K: T is not negative definite (gapless or rank-deficient input)")
    try:
        half_t_inv = lu_solve(t, 0.5 * np.eye(t.shape[0]))
    except SingularMatrix as e:
        raise SingularMatrix("assemble_K: T singular", e.pivot_index)
    half_t_inv = symmetrize(half_t_inv)
    pvp = symmetrize(p.T @ apply_coulomb(dims, cell, p, kernel))
    try:
        k = lu_solve(half_t_inv - pvp, np.eye(t.shape[0]))
    except SingularMatrix as e:
        raise SingularMatrix("assemble_K: middle matrix singular", e.pivot_index)
    return symmetrize(k)


def pvp(p: np.ndarray, dims, cell) -> np.ndarray:
    """smw.hpp:61-62 — symmetrised P^T V P."""
    return symmetrize(p.T @ apply_coulomb(dims, cell, p))


def epsilon_inverse_apply(p, k, dims, cell, x) -> np.ndarray:
    """smw.hpp:84-103 — X + (V P) (K (P^T X))."""
    vp = apply_coulomb(dims, cell, p)
    return x + vp @ (k @ (p.T @ x))


def project_screened(p_vc, k, dims, cell, p_vn, p_nn, kernel=None):
    """gw.hpp:73-88 — B_x = P_x^T (V P_vc), W_x = B_x K B_x^T (x = vn, nn),
    V_vn = P_vn^T V P_vn, each symmetrised. Returns (w_vn, w_nn, v_vn)."""
    vp = apply_coulomb(dims, cell, p_vc, kernel)
    b_vn = p_vn.T @ vp
    b_nn = p_nn.T @ vp
    w_vn = symmetrize((b_vn @ k) @ b_vn.T)
    w_nn = symmetrize((b_nn @ k) @ b_nn.T)
    v_vn = symmetrize(p_vn.T @ apply_coulomb(dims, cell, p_vn, kernel))
    return w_vn, w_nn, v_vn


def hadamard_diag(h: np.ndarray, mask: np.ndarray, psi_pts: np.ndarray) -> np.ndarray:
    """gw.hpp:93-107 — diag(Psi^T (H o M) Psi) for all bands."""
    hp = (h * mask) @ psi_pts
    return np.einsum("in,in->n", psi_pts, hp)


def sigma_lowrank(psi, n_v: int, pts_vn, pts_nn, w_vn, w_nn, v_vn):
    """gw.hpp:112-137 (detail::sigma_hadamard) + finalize (gw.hpp:31-41):
    returns (sigma_sex_x, sigma_x, sigma_coh, sigma_total)."""
    psi_vn = psi[np.asarray(pts_vn)]
    psi_nn = psi[np.asarray(pts_nn)]
    occ = psi_vn[:, :n_v]
    mask_occ = occ @ occ.T
    mask_all = psi_nn @ psi_nn.T
    sex_x = -hadamard_diag(w_vn, mask_occ, psi_vn)
    sx = -hadamard_diag(v_vn, mask_occ, psi_vn)
    coh = 0.5 * hadamard_diag(w_nn, mask_all, psi_nn)
    total = sex_x + sx + coh
    if not np.all(np.isfinite(total)):
        raise NumericError("self-energies: non-finite value")
    return sex_x, sx, coh, total


def quasiparticle_energies(energies, vxc, sigma_total) -> np.ndarray:
    """gw.hpp:48-58."""
    e = np.asarray(energies, dtype=np.float64)
    if len(sigma_total) != e.size or len(vxc) != e.size:
        raise InvalidInput("quasiparticle_energies: length mismatch")
    return e + np.asarray(sigma_total) - np.asarray(vxc)
