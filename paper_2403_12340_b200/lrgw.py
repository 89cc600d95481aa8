"""Python mirror of the reference `lrgw` hot-path interface over liblrgw_cuda.so.

Names, argument meaning and error behaviour follow the reference C++ API
(/root/reference/proj/include/lrgw): host arrays in, host arrays out, the
reference exception taxonomy (errors.hpp:10-36) raised as Python exceptions.
Every call runs on the GPU through the C-ABI (include/lrgw_cuda.h); there is no
CPU path. The device-resident build (`build`) takes torch CUDA tensors.
"""
from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L

# ---------------------------------------------------------------------------
# exception taxonomy (errors.hpp:10-36, contour.hpp:92-96)
# ---------------------------------------------------------------------------


class LrgwError(Exception):
    code = 9


class InvalidInput(LrgwError, ValueError):
    code = 1


class GuardExceeded(LrgwError):
    code = 2


class NumericError(LrgwError):
    code = 3


class SingularMatrix(NumericError):
    code = 4

    def __init__(self, msg, pivot_index=-1):
        super().__init__(f"{msg} (pivot index {pivot_index})")
        self.pivot_index = pivot_index


class ContourConvergenceError(NumericError):
    code = 5

    def __init__(self, msg, best=None):
        super().__init__(msg)
        self.best = best


class IoError(LrgwError):
    code = 6


class CudaError(LrgwError):
    code = 7


class Unsupported(InvalidInput):
    code = 8


_EXC = {1: InvalidInput, 2: GuardExceeded, 3: NumericError, 6: IoError, 7: CudaError, 8: Unsupported}


def _raise(rc, ctx_handle=None, what=""):
    lib = L.load()
    msg = what
    if ctx_handle is not None:
        m = lib.lrgw_ctx_last_error(ctx_handle)
        if m:
            msg = f"{what}: {m.decode()}" if what else m.decode()
    if rc == 4:
        piv = lib.lrgw_ctx_last_pivot(ctx_handle) if ctx_handle is not None else -1
        raise SingularMatrix(msg, piv)
    if rc == 5:
        raise ContourConvergenceError(msg)
    raise _EXC.get(rc, LrgwError)(msg)


def _check(rc, ctx_handle=None, what=""):
    if rc != 0:
        _raise(rc, ctx_handle, what)


# ---------------------------------------------------------------------------
# context
# ---------------------------------------------------------------------------


STAGES = ["select", "fit_lhs", "fit_solve", "fit_gemm", "contour", "fft", "pvp", "smw", "total", "quad_kernel",
          "cusolver", "cufft"]


class Context:
    """One lrgw_ctx (stream, cuSOLVER handle, cuFFT plan cache) on one device."""

    def __init__(self, device: int = 0):
        self._lib = L.load()
        h = L.ctx_t()
        rc = self._lib.lrgw_ctx_create(device, ctypes.byref(h))
        if rc != 0:
            raise CudaError(f"lrgw_ctx_create(device={device}) failed with status {rc}")
        self.handle = h
        self.device = device

    def close(self):
        if getattr(self, "handle", None):
            self._lib.lrgw_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def stage_ms(self):
        out = np.zeros(len(STAGES))
        self._lib.lrgw_ctx_stage_ms(self.handle, out.ctypes.data_as(L.c_double_p), len(STAGES))
        names = STAGES
        return dict(zip(names, out.tolist()))

    def kernel_launches(self) -> int:
        return int(self._lib.lrgw_ctx_kernel_launches(self.handle))

    def set_theta_implicit(self, on: bool = True):
        """lrgw_build keeps Theta factored as L L_P^-1 (see lrgw_ctx_set_theta_implicit)."""
        _check(self._lib.lrgw_ctx_set_theta_implicit(self.handle, int(bool(on))), self.handle, "set_theta_implicit")

    def set_select_batch(self, s: int):
        _check(self._lib.lrgw_ctx_set_select_batch(self.handle, int(s)), self.handle, "set_select_batch")

    def set_stream(self, stream_ptr: int | None):
        _check(self._lib.lrgw_ctx_set_stream(self.handle, ctypes.c_void_p(stream_ptr or 0)), self.handle,
               "set_stream")

    def synchronize(self):
        _check(self._lib.lrgw_ctx_synchronize(self.handle), self.handle, "synchronize")


_default = {}
_default_lock = threading.Lock()


def default_context(device: int = 0) -> Context:
    with _default_lock:
        if device not in _default:
            _default[device] = Context(device)
        return _default[device]


def _ctx(ctx):
    return ctx if ctx is not None else default_context()


def _f(a):
    return np.asfortranarray(a, dtype=np.float64)


def _dp(a):
    return a.ctypes.data_as(L.c_double_p)


def _ip(a):
    return a.ctypes.data_as(L.c_int32_p)


def _grid(dims, cell):
    d = np.ascontiguousarray(dims, dtype=np.int32)
    c = np.ascontiguousarray(cell, dtype=np.float64)
    if d.size != 3 or c.size != 3:
        raise InvalidInput("Grid: dims and cell need 3 entries")
    return d, c


# ---------------------------------------------------------------------------
# ISDF (isdf.hpp)
# ---------------------------------------------------------------------------


def num_aux(k_mu: float, n1: int, n2: int) -> int:
    """isdf.hpp:42-46."""
    out = ctypes.c_int(0)
    _check(L.load().lrgw_num_aux(float(k_mu), int(n1), int(n2), ctypes.byref(out)), None,
           "num_aux: k_mu must be > 0")
    return out.value


def select_interpolation_points(psi_a, psi_b, n_mu: int, method: str = "qrcp_direct", ctx=None) -> np.ndarray:
    """isdf.hpp:95-112 — N_mu grid indices, sorted ascending (int32)."""
    c = _ctx(ctx)
    a, b = _f(psi_a), _f(psi_b)
    if a.shape[0] != b.shape[0]:
        raise InvalidInput("pair_matrix_transposed: row mismatch")
    meth = {"qrcp_direct": 0, "qrcp_sketched": 1}[method]
    pts = np.zeros(max(int(n_mu), 0), dtype=np.int32)
    rc = c._lib.lrgw_select_interpolation_points(c.handle, _dp(a), _dp(b), a.shape[0], a.shape[1], b.shape[1],
                                                 int(n_mu), meth, _ip(pts) if pts.size else None)
    _check(rc, c.handle, "select_interpolation_points")
    return pts


def fit_auxiliary_basis(psi_a, psi_b, points, ctx=None) -> np.ndarray:
    """isdf.hpp:118-163 — Theta (N_r x N_mu, Fortran order)."""
    c = _ctx(ctx)
    a, b = _f(psi_a), _f(psi_b)
    pts = np.ascontiguousarray(points, dtype=np.int32)
    theta = np.zeros((a.shape[0], pts.size), order="F")
    rc = c._lib.lrgw_fit_auxiliary_basis(c.handle, _dp(a), _dp(b), a.shape[0], a.shape[1], b.shape[1],
                                         _ip(pts) if pts.size else None, pts.size, _dp(theta))
    _check(rc, c.handle, "fit_auxiliary_basis")
    return theta


@dataclass
class IsdfDecomposition:
    """isdf.hpp:33-39."""
    label: str
    k_mu: float
    n_mu: int
    point_indices: np.ndarray
    p: np.ndarray


def pair_factors(psi, n_v, n_c, label: str = "vc"):
    """isdf.hpp:166-173 — (occupied, unoccupied), (occupied, all) or (all, all)."""
    occ, allb = psi[:, :n_v], psi[:, :n_v + n_c]
    if label == "vc":
        return occ, psi[:, n_v:n_v + n_c]
    if label == "vn":
        return occ, allb
    if label == "nn":
        return allb, allb
    raise InvalidInput(f"pair_factors: unknown pair set {label!r}")


def build_isdf(psi, n_v, n_c, k_mu, ctx=None, label: str = "vc") -> IsdfDecomposition:
    """isdf.hpp:176-183 — select + fit for the vc / vn / nn pair set."""
    a, b = pair_factors(psi, n_v, n_c, label)
    n_mu = min(max(num_aux(k_mu, a.shape[1], b.shape[1]), 1), psi.shape[0])
    pts = select_interpolation_points(a, b, n_mu, ctx=ctx)
    return IsdfDecomposition(label, k_mu, n_mu, pts, fit_auxiliary_basis(a, b, pts, ctx=ctx))


# ---------------------------------------------------------------------------
# contour (elliptic.hpp, contour.hpp)
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
        return np.array([self.q, self.big_q, self.r, self.big_r, self.l, self.e_shift, float(self.bypass)])


@dataclass
class CoupledCoefficients:
    """contour.hpp:86-90."""
    t: np.ndarray
    nodes_used: int = 0
    est_rel_error: float = 0.0


def elliptic_k(k: float) -> float:
    out = ctypes.c_double(0)
    _check(L.load().lrgw_elliptic_k(float(k), ctypes.byref(out)), None, "elliptic_k: modulus must be in [0, 1)")
    return out.value


def jacobi_sn_cn_dn(u: float, k: float):
    out = np.zeros(3)
    _check(L.load().lrgw_jacobi_sn_cn_dn(float(u), float(k), _dp(out)), None, "jacobi_sn_cn_dn")
    return tuple(out.tolist())


def jacobi_complex(x: float, y: float, k: float):
    out = np.zeros(6)
    _check(L.load().lrgw_jacobi_complex(float(x), float(y), float(k), _dp(out)), None, "jacobi_complex")
    return complex(out[0], out[1]), complex(out[2], out[3]), complex(out[4], out[5])


def elliptic_params(energies, n_v: int, n_c: int, delta_rel: float, max_nodes: int = 1025) -> ContourSpec:
    e = np.ascontiguousarray(energies, dtype=np.float64)
    out = np.zeros(7)
    _check(L.load().lrgw_elliptic_params(_dp(e), e.size, int(n_v), int(n_c), float(delta_rel), int(max_nodes),
                                         _dp(out)), None, "elliptic_params")
    return ContourSpec(*out[:6].tolist(), delta_rel=delta_rel, max_nodes=max_nodes, bypass=bool(out[6]))


def cauchy_error_bound(spec: ContourSpec, n_lambda: int) -> float:
    s = spec.as7()
    out = ctypes.c_double(0)
    _check(L.load().lrgw_cauchy_error_bound(_dp(s), int(n_lambda), ctypes.byref(out)), None,
           "cauchy_error_bound: N_lambda < 1")
    return out.value


def _pts_args(psi_v_pts, psi_c_pts, energies):
    pv, pc = _f(psi_v_pts), _f(psi_c_pts)
    if pv.shape[0] != pc.shape[0]:
        raise InvalidInput("coupled_coefficients: point-row mismatch")
    e = np.ascontiguousarray(energies, dtype=np.float64)
    return pv, pc, e


def coupled_coefficients_direct(psi_v_pts, psi_c_pts, energies, ctx=None) -> CoupledCoefficients:
    c = _ctx(ctx)
    pv, pc, e = _pts_args(psi_v_pts, psi_c_pts, energies)
    t = np.zeros((pv.shape[0], pv.shape[0]), order="F")
    _check(c._lib.lrgw_coupled_coefficients_direct(c.handle, _dp(pv), _dp(pc), pv.shape[0], pv.shape[1],
                                                   pc.shape[1], _dp(e), e.size, _dp(t)), c.handle,
           "coupled_coefficients_direct")
    return CoupledCoefficients(t, 0, 0.0)


def sum_node_terms(psi_v_pts, psi_c_pts, energies, spec: ContourSpec, nodes, weights, ctx=None) -> np.ndarray:
    c = _ctx(ctx)
    pv, pc, e = _pts_args(psi_v_pts, psi_c_pts, energies)
    nd = np.ascontiguousarray(nodes, dtype=np.float64)
    wt = np.ascontiguousarray(weights, dtype=np.float64)
    s = spec.as7()
    acc = np.zeros((pv.shape[0], pv.shape[0]), order="F")
    _check(c._lib.lrgw_sum_node_terms(c.handle, _dp(pv), _dp(pc), pv.shape[0], pv.shape[1], pc.shape[1], _dp(e),
                                      e.size, _dp(s), _dp(nd), _dp(wt), nd.size, _dp(acc)), c.handle,
           "sum_node_terms")
    return acc


def coupled_coefficients_fixed(psi_v_pts, psi_c_pts, energies, n_lambda: int, ctx=None) -> CoupledCoefficients:
    c = _ctx(ctx)
    pv, pc, e = _pts_args(psi_v_pts, psi_c_pts, energies)
    t = np.zeros((pv.shape[0], pv.shape[0]), order="F")
    _check(c._lib.lrgw_coupled_coefficients_fixed(c.handle, _dp(pv), _dp(pc), pv.shape[0], pv.shape[1],
                                                  pc.shape[1], _dp(e), e.size, int(n_lambda), _dp(t)), c.handle,
           "coupled_coefficients_fixed")
    return CoupledCoefficients(t, int(n_lambda) + 1, 0.0)


def coupled_coefficients_contour(psi_v_pts, psi_c_pts, energies, spec: ContourSpec, threads: int = 1,
                                 ctx=None) -> CoupledCoefficients:
    """contour.hpp:298-329 (`threads` kept for signature parity; host-only)."""
    c = _ctx(ctx)
    pv, pc, e = _pts_args(psi_v_pts, psi_c_pts, energies)
    t = np.zeros((pv.shape[0], pv.shape[0]), order="F")
    nu = ctypes.c_int(0)
    est = ctypes.c_double(0)
    rc = c._lib.lrgw_coupled_coefficients_contour(c.handle, _dp(pv), _dp(pc), pv.shape[0], pv.shape[1],
                                                  pc.shape[1], _dp(e), e.size, float(spec.delta_rel),
                                                  int(spec.max_nodes), _dp(t), ctypes.byref(nu), ctypes.byref(est))
    if rc == 5:
        raise ContourConvergenceError(
            "coupled_coefficients_contour: did not reach delta_rel within max_nodes",
            CoupledCoefficients(t, nu.value, est.value))
    _check(rc, c.handle, "coupled_coefficients_contour")
    return CoupledCoefficients(t, nu.value, est.value)


def contour_refinement_levels(psi_v_pts, psi_c_pts, energies, spec: ContourSpec, max_level_nodes: int,
                              threads: int = 1, ctx=None):
    c = _ctx(ctx)
    pv, pc, e = _pts_args(psi_v_pts, psi_c_pts, energies)
    n_mu = pv.shape[0]
    max_levels = 16
    out = np.zeros((max_levels, n_mu, n_mu))
    counts = np.zeros(max_levels, dtype=np.int32)
    nl = ctypes.c_int(0)
    _check(c._lib.lrgw_contour_refinement_levels(c.handle, _dp(pv), _dp(pc), n_mu, pv.shape[1], pc.shape[1],
                                                 _dp(e), e.size, int(max_level_nodes), max_levels, _dp(out),
                                                 counts.ctypes.data_as(L.c_int_p), ctypes.byref(nl)), c.handle,
           "contour_refinement_levels")
    # each level was written column-major into a C-order slab: transpose back
    return [(int(counts[i]), np.asfortranarray(out[i].T)) for i in range(nl.value)]


# ---------------------------------------------------------------------------
# Coulomb + SMW (model.hpp, smw.hpp)
# ---------------------------------------------------------------------------


def coulomb_kernel(dims, cell) -> np.ndarray:
    d, c = _grid(dims, cell)
    out = np.zeros(int(np.prod(d)))
    _check(L.load().lrgw_coulomb_kernel(d.ctypes.data_as(L.c_int_p), _dp(c), _dp(out)), None, "build_coulomb")
    return out


def apply_coulomb(dims, cell, x, zero_kernel: bool = False, ctx=None) -> np.ndarray:
    c = _ctx(ctx)
    d, cl = _grid(dims, cell)
    xx = _f(x)
    if xx.ndim == 1:
        xx = xx.reshape(-1, 1, order="F")
    if xx.shape[0] != int(np.prod(d)):
        raise InvalidInput("apply_coulomb: row count != N_r")
    y = np.zeros_like(xx, order="F")
    _check(c._lib.lrgw_apply_coulomb(c.handle, d.ctypes.data_as(L.c_int_p), _dp(cl), int(zero_kernel), _dp(xx),
                                     xx.shape[1], _dp(y)), c.handle, "apply_coulomb")
    return y


def assemble_K(t, p, dims, cell, zero_kernel: bool = False, ctx=None) -> np.ndarray:
    c = _ctx(ctx)
    d, cl = _grid(dims, cell)
    tt, pp = _f(t), _f(p)
    if tt.shape[0] != tt.shape[1] or tt.shape[0] != pp.shape[1]:
        raise InvalidInput("assemble_K: T / P_vc shape mismatch")
    k = np.zeros_like(tt, order="F")
    _check(c._lib.lrgw_assemble_K(c.handle, _dp(tt), _dp(pp), pp.shape[0], pp.shape[1],
                                  d.ctypes.data_as(L.c_int_p), _dp(cl), int(zero_kernel), _dp(k)), c.handle,
           "assemble_K")
    return k


class EpsilonInverseLowRank:
    """Device-resident factored eps^-1 (smw.hpp:77-82): Theta, K (and T) stay
    in HBM; host copies on demand (`k`, `p_vc`, `vp`)."""

    def __init__(self, ctx: Context, handle):
        self.ctx = ctx
        self.handle = handle
        n_r, n_mu = ctypes.c_int(0), ctypes.c_int(0)
        ctx._lib.lrgw_eps_shape(handle, ctypes.byref(n_r), ctypes.byref(n_mu))
        self.n_r, self.n_mu = n_r.value, n_mu.value

    def _get(self, which):
        out = np.zeros((self.n_mu, self.n_mu) if which in ("k", "t") else (self.n_r, self.n_mu), order="F")
        args = {"k": None, "p": None, "vp": None, "t": None}
        args[which] = _dp(out)
        _check(self.ctx._lib.lrgw_eps_get(self.ctx.handle, self.handle, args["k"], args["p"], args["vp"],
                                          args["t"], None), self.ctx.handle, "eps_get")
        return out

    @property
    def k(self):
        return self._get("k")

    @property
    def p_vc(self):
        return self._get("p")

    @property
    def vp(self):
        return self._get("vp")

    @property
    def t(self):
        return self._get("t")

    @property
    def point_indices(self):
        pts = np.zeros(self.n_mu, dtype=np.int32)
        _check(self.ctx._lib.lrgw_eps_get(self.ctx.handle, self.handle, None, None, None, None, _ip(pts)),
               self.ctx.handle, "eps_get")
        return pts

    def info(self) -> dict:
        """Build diagnostics (lrgw_eps_info): the smallest relative top-2
        pivot margin of the greedy selection and its step, the fit path
        (0 fused L L_P^-1, 1 explicit Gram LU), the lower bound
        (max|L_ii| / min|L_ii|)^2 on cond(G(P, P)), the candidate-block count,
        and the device pointers (theta, k, t, pvp)."""
        inf = L.EpsInfo()
        _check(self.ctx._lib.lrgw_eps_info_get(self.handle, ctypes.byref(inf)), self.ctx.handle, "eps_info")
        return {f: getattr(inf, f) for f, _ in L.EpsInfo._fields_}

    def device_ptrs(self):
        th, k, t = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
        self.ctx._lib.lrgw_eps_device_ptrs(self.handle, ctypes.byref(th), ctypes.byref(k), ctypes.byref(t))
        return th.value, k.value, t.value

    def close(self):
        if getattr(self, "handle", None):
            self.ctx._lib.lrgw_eps_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def build_epsilon_inverse(t, p, dims, cell, threads: int = 1, zero_kernel: bool = False,
                          ctx=None) -> EpsilonInverseLowRank:
    """smw.hpp:84-94."""
    c = _ctx(ctx)
    d, cl = _grid(dims, cell)
    tt, pp = _f(t), _f(p)
    h = L.eps_t()
    _check(c._lib.lrgw_build_epsilon_inverse(c.handle, _dp(tt), _dp(pp), pp.shape[0], pp.shape[1],
                                             d.ctypes.data_as(L.c_int_p), _dp(cl), int(zero_kernel),
                                             ctypes.byref(h)), c.handle, "build_epsilon_inverse")
    return EpsilonInverseLowRank(c, h)


@dataclass
class ScreenedProjections:
    """gw.hpp:65-69."""
    w_vn: np.ndarray  # (P_vn^T V P_vc) K (P_vn^T V P_vc)^T
    w_nn: np.ndarray
    v_vn: np.ndarray  # P_vn^T V P_vn


def project_screened_interactions(e: EpsilonInverseLowRank, dec_vn, dec_nn, threads: int = 1) -> ScreenedProjections:
    """gw.hpp:73-88 on the GPU (G-space contractions against e's device
    factors). dec_vn / dec_nn: IsdfDecomposition or N_r x n matrices."""
    p_vn = _f(getattr(dec_vn, "p", dec_vn))
    p_nn = _f(getattr(dec_nn, "p", dec_nn))
    if p_vn.shape[0] != e.n_r or p_nn.shape[0] != e.n_r:
        raise InvalidInput("project_screened_interactions: grid mismatch")
    n_vn, n_nn = p_vn.shape[1], p_nn.shape[1]
    w_vn = np.zeros((n_vn, n_vn), order="F")
    w_nn = np.zeros((n_nn, n_nn), order="F")
    v_vn = np.zeros((n_vn, n_vn), order="F")
    c = e.ctx
    _check(c._lib.lrgw_project_screened_interactions(c.handle, e.handle, _dp(p_vn), n_vn, _dp(p_nn), n_nn,
                                                     _dp(w_vn), _dp(w_nn), _dp(v_vn)),
           c.handle, "project_screened_interactions")
    return ScreenedProjections(w_vn, w_nn, v_vn)


@dataclass
class SelfEnergies:
    """gw.hpp:28-42 — per-band static-COHSEX components (hartree)."""
    sigma_sex_x: np.ndarray
    sigma_x: np.ndarray
    sigma_coh: np.ndarray
    sigma_total: np.ndarray
    pipeline_tag: str = "lowrank"


def self_energies_lowrank(psi, n_v: int, w_vn, w_nn, v_vn, dec_vn, dec_nn, ctx=None) -> SelfEnergies:
    """gw.hpp:143-153 (detail::sigma_hadamard, gw.hpp:93-137) on the GPU.
    psi: N_r x (n_v + n_c) orbitals; w_vn / w_nn / v_vn from
    project_screened_interactions; dec_vn / dec_nn: IsdfDecomposition or
    point-index arrays. Raises NumericError on a non-finite band
    (SelfEnergies::finalize)."""
    c = _ctx(ctx)
    ps = _f(psi)
    n_r, nb = ps.shape
    if not 0 <= n_v <= nb:
        raise InvalidInput("self_energies_lowrank: n_v out of range")
    pv = np.ascontiguousarray(getattr(dec_vn, "point_indices", dec_vn), dtype=np.int32)
    pn = np.ascontiguousarray(getattr(dec_nn, "point_indices", dec_nn), dtype=np.int32)
    wv, wn, vv = _f(w_vn), _f(w_nn), _f(v_vn)
    if wv.shape != (pv.size, pv.size) or vv.shape != wv.shape or wn.shape != (pn.size, pn.size):
        raise InvalidInput("self_energies_lowrank: interaction block / point count mismatch")
    out = [np.zeros(nb) for _ in range(4)]
    _check(c._lib.lrgw_self_energies_lowrank(c.handle, _dp(ps), n_r, n_v, nb - n_v, _ip(pv), pv.size, _ip(pn),
                                             pn.size, _dp(wv), _dp(wn), _dp(vv), *[_dp(o) for o in out]),
           c.handle, "self_energies_lowrank")
    return SelfEnergies(*out)


@dataclass
class QuasiparticleEnergies:
    """gw.hpp:44-46."""
    eps_gw: np.ndarray


def quasiparticle_energies(energies, vxc, sig: SelfEnergies) -> QuasiparticleEnergies:
    """gw.hpp:48-58: eps_gw = eps + sigma_total - vxc (host, O(N_b))."""
    e = np.asarray(energies, dtype=np.float64)
    v = np.asarray(vxc, dtype=np.float64)
    if sig.sigma_total.shape != e.shape or v.shape != e.shape:
        raise InvalidInput("quasiparticle_energies: length mismatch")
    return QuasiparticleEnergies(e + sig.sigma_total - v)


# ---- WFN1 orbital files (model.hpp:236-339) --------------------------------

@dataclass
class ElectronicStructure:
    """model.hpp:27-50 (host arrays; psi N_r x (n_v + n_c), column major)."""
    dims: tuple
    cell: tuple
    psi: np.ndarray
    energies: np.ndarray
    vxc: np.ndarray
    n_v: int
    n_c: int

    @property
    def n_r(self) -> int:
        return int(np.prod(self.dims))

    @property
    def n_bands(self) -> int:
        return self.n_v + self.n_c


def _io_check(rc, what):
    if rc != 0:
        msg = (L.load().lrgw_last_error() or b"").decode() or what
        _raise(rc, None, msg)


def save_system(path: str, es: ElectronicStructure) -> None:
    """model.hpp:262-285 — byte-identical to the reference writer."""
    lib = L.load()
    d = np.ascontiguousarray(es.dims, dtype=np.int32)
    cl = np.ascontiguousarray(es.cell, dtype=np.float64)
    psi = _f(es.psi)
    e = np.ascontiguousarray(es.energies, dtype=np.float64)
    v = np.ascontiguousarray(es.vxc, dtype=np.float64)
    nb = es.n_v + es.n_c
    if psi.shape != (int(np.prod(d)), nb) or e.size != nb or v.size != nb:
        raise InvalidInput("save_system: array shapes do not match the header")
    _io_check(lib.lrgw_wfn1_save(str(path).encode(), d.ctypes.data_as(L.c_int_p), _dp(cl), es.n_v, es.n_c,
                                 _dp(psi), _dp(e), _dp(v)), "save_system")


def _wfn1_info(path):
    lib = L.load()
    d = np.zeros(3, dtype=np.int32)
    cl = np.zeros(3)
    nv, nc = ctypes.c_int(0), ctypes.c_int(0)
    _io_check(lib.lrgw_wfn1_info(str(path).encode(), d.ctypes.data_as(L.c_int_p), _dp(cl), ctypes.byref(nv),
                                 ctypes.byref(nc)), "load_system")
    return tuple(int(x) for x in d), tuple(float(x) for x in cl), nv.value, nc.value


def load_system(path: str) -> ElectronicStructure:
    """model.hpp:287-339 — same validation and io_error messages."""
    lib = L.load()
    dims, cell, nv, nc = _wfn1_info(path)
    n_r = int(np.prod(dims))
    psi = np.zeros((n_r, nv + nc), order="F")
    e, v = np.zeros(nv + nc), np.zeros(nv + nc)
    _io_check(lib.lrgw_wfn1_load(str(path).encode(), _dp(psi), _dp(e), _dp(v)), "load_system")
    return ElectronicStructure(dims, cell, psi, e, v, nv, nc)


def load_system_device(path: str, ctx=None):
    """WFN1 straight into HBM: psi streamed in column blocks through pinned
    buffers (a column-major torch.cuda tensor), energies / vxc on the host.
    Returns (dims, cell, psi_dev, energies, vxc, n_v, n_c)."""
    import torch

    c = _ctx(ctx)
    dims, cell, nv, nc = _wfn1_info(path)
    n_r = int(np.prod(dims))
    psi = torch.empty((nv + nc, n_r), dtype=torch.float64, device=f"cuda:{c.device}").t()
    e, v = np.zeros(nv + nc), np.zeros(nv + nc)
    _check(c._lib.lrgw_wfn1_load_device(c.handle, str(path).encode(), psi.data_ptr(), n_r, _dp(e), _dp(v)),
           c.handle, "")
    return dims, cell, psi, e, v, nv, nc


def epsilon_inverse_from_parts(p, k, dims, cell, ctx=None) -> EpsilonInverseLowRank:
    c = _ctx(ctx)
    d, cl = _grid(dims, cell)
    pp, kk = _f(p), _f(k)
    h = L.eps_t()
    _check(c._lib.lrgw_eps_from_parts(c.handle, _dp(pp), _dp(kk), pp.shape[0], pp.shape[1],
                                      d.ctypes.data_as(L.c_int_p), _dp(cl), 0, ctypes.byref(h)), c.handle,
           "eps_from_parts")
    return EpsilonInverseLowRank(c, h)


def epsilon_inverse_apply(e: EpsilonInverseLowRank, x) -> np.ndarray:
    """smw.hpp:97-103: X + V P (K (P^T X))."""
    xx = _f(x)
    if xx.ndim == 1:
        xx = xx.reshape(-1, 1, order="F")
    if xx.shape[0] != e.n_r:
        raise InvalidInput("epsilon_inverse_apply: row mismatch")
    y = np.zeros_like(xx, order="F")
    _check(e.ctx._lib.lrgw_epsilon_inverse_apply(e.ctx.handle, e.handle, _dp(xx), xx.shape[1], _dp(y)),
           e.ctx.handle, "epsilon_inverse_apply")
    return y


# ---------------------------------------------------------------------------
# device-resident build (stages 1-5) over torch CUDA tensors
# ---------------------------------------------------------------------------


def _dev_ptr_cm(t):
    """Device pointer and leading dim of a column-major view of a 2-D CUDA tensor."""
    import torch

    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64):
        raise InvalidInput("expected a float64 CUDA tensor")
    if t.dim() != 2 or (t.stride(0) != 1 and t.shape[0] > 1):
        raise InvalidInput("expected a column-major (stride(0) == 1) 2-D tensor")
    ld = t.stride(1) if t.shape[1] > 1 else t.shape[0]
    if ld < t.shape[0]:
        raise InvalidInput("column stride below the row count")
    return t.data_ptr(), max(ld, 1)


def _build_params(c, phi_v, phi_c, energies, dims, cell, k_mu, n_lambda, delta_rel, max_nodes, zero_kernel,
                  rows=None):
    """Validated lrgw_build_params + device pointers (rows: the panel's row count)."""
    for name, t in (("phi_v", phi_v), ("phi_c", phi_c)):
        if not getattr(t, "is_cuda", False) or t.dim() != 2:
            raise InvalidInput(f"build: {name} must be a 2-D CUDA tensor")
        if t.device.index != c.device:
            raise InvalidInput(f"build: {name} is on cuda:{t.device.index}, the context on cuda:{c.device}")
    if phi_c.shape[0] != phi_v.shape[0]:
        raise InvalidInput("build: phi_v and phi_c must have the same number of grid rows")
    n_r = int(np.prod([int(x) for x in dims]))
    if phi_v.shape[0] != (n_r if rows is None else rows):
        raise InvalidInput(f"build: orbital rows {phi_v.shape[0]} != {n_r if rows is None else rows}")
    pv, ldv = _dev_ptr_cm(phi_v)
    pc, ldc = _dev_ptr_cm(phi_c)
    e = np.ascontiguousarray(energies, dtype=np.float64)
    if e.ndim != 1 or e.size != phi_v.shape[1] + phi_c.shape[1]:
        raise InvalidInput("build: energies must hold exactly N_v + N_c values")
    prm = L.BuildParams()
    prm.n_r, prm.n_v, prm.n_c = n_r, phi_v.shape[1], phi_c.shape[1]
    prm.n_e = e.size
    prm.dims[:] = [int(x) for x in dims]
    prm.cell[:] = [float(x) for x in cell]
    prm.k_mu = float(k_mu)
    prm.n_lambda = int(n_lambda)
    prm.delta_rel = float(delta_rel)
    prm.max_nodes = int(max_nodes)
    prm.zero_kernel = int(zero_kernel)
    return prm, pv, ldv, pc, ldc, e


def build(phi_v, phi_c, energies, dims, cell, k_mu: float = 8.0, n_lambda: int = 16, delta_rel: float = 1e-7,
          max_nodes: int = 1025, zero_kernel: bool = False, ctx=None) -> EpsilonInverseLowRank:
    """Stages 1-5 from device-resident orbitals (column-major float64 CUDA
    tensors, N_r x N_v and N_r x N_c) and host energies: point selection,
    Theta fit, Cauchy quadrature core, G-space Theta^T V Theta, SMW core K."""
    c = _ctx(ctx)
    prm, pv, ldv, pc, ldc, e = _build_params(c, phi_v, phi_c, energies, dims, cell, k_mu, n_lambda, delta_rel,
                                             max_nodes, zero_kernel)
    _sync_torch(phi_v)
    h = L.eps_t()
    _check(c._lib.lrgw_build(c.handle, ctypes.byref(prm), ctypes.c_void_p(pv), ldv, ctypes.c_void_p(pc), ldc,
                             _dp(e), ctypes.byref(h)), c.handle, "build")
    return EpsilonInverseLowRank(c, h)


def _sync_torch(t):
    import torch

    torch.cuda.current_stream(t.device).synchronize()


def eps_apply_dev(e: EpsilonInverseLowRank, x, y):
    """y = eps^-1 x for column-major float64 CUDA tensors (N_r x m)."""
    px, ldx = _dev_ptr_cm(x)
    py, ldy = _dev_ptr_cm(y)
    _sync_torch(x)
    _check(e.ctx._lib.lrgw_eps_apply_dev(e.ctx.handle, e.handle, ctypes.c_void_p(px), ldx, x.shape[1],
                                         ctypes.c_void_p(py), ldy), e.ctx.handle, "eps_apply_dev")
    return y


def dgemm_dev(trans_a: str, trans_b: str, alpha: float, a, b, beta: float, c, ctx=None):
    """C = alpha op(A) op(B) + beta C on column-major float64 CUDA tensors
    through the path's DMMA GEMM engine (BLAS argument semantics)."""
    cx = _ctx(ctx)
    pa, lda = _dev_ptr_cm(a)
    pb, ldb = _dev_ptr_cm(b)
    pc, ldc = _dev_ptr_cm(c)
    m, n = c.shape
    k = a.shape[1] if trans_a.upper() == "N" else a.shape[0]
    _sync_torch(a)
    _check(cx._lib.lrgw_dev_dgemm(cx.handle, trans_a.upper().encode(), trans_b.upper().encode(), m, n, k,
                                  float(alpha), ctypes.c_void_p(pa), lda, ctypes.c_void_p(pb), ldb, float(beta),
                                  ctypes.c_void_p(pc), ldc), cx.handle, "dgemm")
    return c


def hadamard_dev(a1, b1, a2, b2, c, ctx=None):
    """C = (A1 B1^T) o (A2 B2^T) on column-major float64 CUDA tensors through the
    path's Hadamard-pair engine (the ISDF Gram pair, isdf.hpp:132)."""
    cx = _ctx(ctx)
    p = [_dev_ptr_cm(x) for x in (a1, b1, a2, b2, c)]
    m, n = c.shape
    _sync_torch(a1)
    _check(cx._lib.lrgw_dev_hadamard(cx.handle, m, n, ctypes.c_void_p(p[0][0]), p[0][1], ctypes.c_void_p(p[1][0]),
                                     p[1][1], a1.shape[1], ctypes.c_void_p(p[2][0]), p[2][1],
                                     ctypes.c_void_p(p[3][0]), p[3][1], a2.shape[1], ctypes.c_void_p(p[4][0]),
                                     p[4][1]), cx.handle, "hadamard")
    return c


def trtri_lower_dev(a, ctx=None):
    """In-place inverse of the lower triangle of a square column-major float64
    CUDA matrix (the strict upper triangle is left untouched)."""
    cx = _ctx(ctx)
    pa, lda = _dev_ptr_cm(a)
    _sync_torch(a)
    _check(cx._lib.lrgw_dev_trtri_lower(cx.handle, ctypes.c_void_p(pa), a.shape[0], lda), cx.handle, "trtri")
    return a


def select_topk_dev(d, pos, k: int, s1: int, ctx=None):
    """Top s1 rows by (d desc, position asc) among rows with pos >= k (one
    selection block's candidate set). d: float64, pos: int32 CUDA vectors.
    Returns (rows, values, positions) numpy arrays; missing entries have row -1."""
    import numpy as np

    cx = _ctx(ctx)
    n_r = d.shape[0]
    rows = np.empty(s1, np.int32)
    vals = np.empty(s1, np.float64)
    poss = np.empty(s1, np.int32)
    _sync_torch(d)
    _check(cx._lib.lrgw_dev_select_topk(cx.handle, ctypes.c_void_p(d.data_ptr()), ctypes.c_void_p(pos.data_ptr()),
                                        n_r, int(k), int(s1), rows.ctypes.data, vals.ctypes.data, poss.ctypes.data),
           cx.handle, "select_topk")
    return rows, vals, poss


def theta_from_factor_dev(l, x, colmap, theta, ctx=None):
    """theta(:, colmap[q]) = (L X)(:, q) for X = L_P^-1 lower triangular
    (column-major float64 CUDA tensors; colmap a permutation, host)."""
    import numpy as np

    cx = _ctx(ctx)
    rows, n_mu = theta.shape
    if x.shape != (n_mu, n_mu) or l.shape[0] != rows or l.shape[1] < n_mu:
        raise InvalidInput("theta_from_factor: shape mismatch")
    pl, ldl = _dev_ptr_cm(l)
    px, ldx = _dev_ptr_cm(x)
    pt, ldt = _dev_ptr_cm(theta)
    cm = np.ascontiguousarray(colmap, dtype=np.int32)
    _sync_torch(l)
    _check(cx._lib.lrgw_dev_theta_from_factor(cx.handle, ctypes.c_void_p(pl), ldl, rows, n_mu, ctypes.c_void_p(px),
                                              ldx, cm.ctypes.data_as(L.c_int32_p), ctypes.c_void_p(pt), ldt),
           cx.handle, "theta_from_factor")
    return theta


def select_panel_update_dev(a, b, L, k: int, piv_rows, x, pos, d, ctx=None):
    """One selection block's update of a row panel (column-major float64
    CUDA tensors a, b, L; pos int32, d float64; piv_rows nb x (n1 + n2 + k) =
    [A_sel | B_sel | L_sel]; x = L_sel^-1, nb x nb)."""
    cx = _ctx(ctx)
    pa, lda = _dev_ptr_cm(a)
    pb, ldb = _dev_ptr_cm(b)
    pl, ldl = _dev_ptr_cm(L)
    px, ldx = _dev_ptr_cm(x)
    pp, ldp = _dev_ptr_cm(piv_rows)
    nb = piv_rows.shape[0]
    n1, n2 = a.shape[1], b.shape[1]
    if piv_rows.shape[1] != n1 + n2 + k or x.shape[0] < nb or L.shape[1] < k + nb:
        raise InvalidInput("select_panel_update: shape mismatch")
    _sync_torch(d)
    _check(cx._lib.lrgw_dev_select_panel_update(cx.handle, ctypes.c_void_p(pa), lda, n1, ctypes.c_void_p(pb), ldb,
                                                n2, a.shape[0], ctypes.c_void_p(pl), ldl, int(k), nb,
                                                ctypes.c_void_p(pp), ldp, ctypes.c_void_p(px), ldx,
                                                ctypes.c_void_p(pos.data_ptr()), ctypes.c_void_p(d.data_ptr())),
           cx.handle, "select_panel_update")


def gram_weighted_dev(x, w, out, ctx=None):
    """out = X^T diag(w) X for a column-major float64 CUDA X (kdim x m), w
    (kdim,) and out (m x m)."""
    cx = _ctx(ctx)
    px, ldx = _dev_ptr_cm(x)
    po, ldo = _dev_ptr_cm(out)
    kdim, m = x.shape
    if w.numel() != kdim or not w.is_contiguous() or out.shape != (m, m):
        raise InvalidInput("gram_weighted: shape mismatch")
    _sync_torch(x)
    _check(cx._lib.lrgw_dev_gram_weighted(cx.handle, ctypes.c_void_p(px), ldx, kdim, m, ctypes.c_void_p(w.data_ptr()),
                                          ctypes.c_void_p(po), ldo), cx.handle, "gram_weighted")
    return out


def cand_greedy_dev(n_r: int, steps: int, k: int, top_vals, top_pos, top_rows, wcc, pos, perm, x, ctx=None):
    """One selection block's certified greedy on the device (the kernel of
    the single-GPU selection): top_* = the s+1 candidate entries (host), wcc
    = their Schur block (s x s column-major CUDA), pos / perm = int32 CUDA
    position bookkeeping (updated in place), x (s x s CUDA) <- L_sel^-1.
    Returns (b, pivot rows, margins) with host arrays of length b."""
    import numpy as np

    cx = _ctx(ctx)
    s = int(wcc.shape[0])
    tv = np.ascontiguousarray(top_vals, dtype=np.float64)
    tp = np.ascontiguousarray(top_pos, dtype=np.int32)
    tr = np.ascontiguousarray(top_rows, dtype=np.int32)
    if tv.size != s + 1 or tp.size != s + 1 or tr.size != s + 1:
        raise InvalidInput("cand_greedy: top needs s + 1 entries")
    pw, ldw = _dev_ptr_cm(wcc)
    px, ldx = _dev_ptr_cm(x)
    if ldw != s or ldx != s or x.shape[0] != s:
        raise InvalidInput("cand_greedy: wcc and x must be s x s with ld s")
    piv = np.empty(s, np.int32)
    mg = np.empty(s, np.float64)
    b = np.zeros(1, np.int32)
    _sync_torch(wcc)
    _check(cx._lib.lrgw_dev_cand_greedy(cx.handle, int(n_r), s, int(steps), int(k), _dp(tv),
                                        tp.ctypes.data_as(L.c_int32_p), tr.ctypes.data_as(L.c_int32_p),
                                        ctypes.c_void_p(pw), ctypes.c_void_p(pos.data_ptr()),
                                        ctypes.c_void_p(perm.data_ptr()), ctypes.c_void_p(px),
                                        piv.ctypes.data_as(L.c_int32_p), _dp(mg), b.ctypes.data_as(L.c_int32_p)),
           cx.handle, "cand_greedy")
    nb = int(b[0])
    return nb, piv[:nb].copy(), mg[:nb].copy()


def coulomb_apply_dev(dims, cell, x, y, zero_kernel: bool = False, ctx=None):
    """y = V x for column-major float64 CUDA tensors (N_r x m)."""
    cx = _ctx(ctx)
    d, cl = _grid(dims, cell)
    px, ldx = _dev_ptr_cm(x)
    py, ldy = _dev_ptr_cm(y)
    _sync_torch(x)
    _check(cx._lib.lrgw_dev_coulomb_apply(cx.handle, d.ctypes.data_as(L.c_int_p), _dp(cl), int(zero_kernel),
                                          ctypes.c_void_p(px), ldx, x.shape[1], ctypes.c_void_p(py), ldy),
           cx.handle, "coulomb_apply")
    return y


def contour_partial_dev(pv, pc, energies, n_lambda: int, node0: int, count: int, acc, ctx=None):
    """acc (N_mu x N_mu, CUDA, column-major) = sum over nodes [node0, node0 +
    count) of an n_lambda-interval trapezoid of w_k term_k, unscaled (the
    multi-rank node split; contour.hpp:185-222)."""
    cx = _ctx(ctx)
    ppv, ldv = _dev_ptr_cm(pv)
    ppc, ldc = _dev_ptr_cm(pc)
    pa, _ = _dev_ptr_cm(acc)
    e = _f(energies).ravel()
    _sync_torch(pv)
    _check(cx._lib.lrgw_dev_contour_partial(cx.handle, ctypes.c_void_p(ppv), ldv, ctypes.c_void_p(ppc), ldc,
                                            pv.shape[0], pv.shape[1], pc.shape[1], _dp(e), e.size, int(n_lambda),
                                            int(node0), int(count), ctypes.c_void_p(pa)),
           cx.handle, "contour_partial")
    return acc


def smw_core_dev(t, pvp, k, ctx=None):
    """K = (T^-1/2 - Theta^T V Theta)^-1 on CUDA N_mu x N_mu matrices (smw.hpp:42-73)."""
    cx = _ctx(ctx)
    pt, _ = _dev_ptr_cm(t)
    pp, _ = _dev_ptr_cm(pvp)
    pk, _ = _dev_ptr_cm(k)
    _sync_torch(t)
    _check(cx._lib.lrgw_dev_smw_core(cx.handle, ctypes.c_void_p(pt), ctypes.c_void_p(pp), t.shape[0],
                                     ctypes.c_void_p(pk)), cx.handle, "smw_core")
    return k


# ---------------------------------------------------------------------------
# multi-rank build through the C-ABI (lrgw_comm, lrgw_build_sharded)
# ---------------------------------------------------------------------------

def z_panel(dims, world: int, rank: int):
    """This rank's grid-row panel (row0, rows): whole z-planes, floor(n3 p / world)."""
    d = (ctypes.c_int * 3)(*[int(x) for x in dims])
    r0, rows = ctypes.c_int(0), ctypes.c_int(0)
    _check(L.load().lrgw_z_panel(d, int(world), int(rank), ctypes.byref(r0), ctypes.byref(rows)), None, "z_panel")
    return r0.value, rows.value


class Comm:
    """An lrgw_comm: NCCL (device buffers over NVLink) or a host transport
    (three Python callables on numpy views; e.g. torch.distributed gloo)."""

    def __init__(self, handle, rank, world, keep=()):
        self._lib = L.load()
        self.handle, self.rank, self.world = handle, rank, world
        self._keep = keep  # the ctypes callbacks must outlive the communicator

    @classmethod
    def nccl(cls, ctx, rank: int, world: int, uid: bytes):
        lib = L.load()
        h = L.comm_t()
        buf = (ctypes.c_ubyte * 128).from_buffer_copy(uid)
        _check(lib.lrgw_comm_create_nccl(ctx.handle, rank, world, buf, ctypes.byref(h)), ctx.handle, "comm_nccl")
        return cls(h, rank, world)

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = (ctypes.c_ubyte * 128)()
        _check(L.load().lrgw_nccl_unique_id(buf), None, "nccl_unique_id")
        return bytes(buf)

    @classmethod
    def host(cls, rank: int, world: int, allreduce, allgather, alltoallv):
        """allreduce(arr float64, in place); allgather(send uint8, recv uint8
        (world * n)); alltoallv(send uint8, send_sizes, recv uint8, recv_sizes)."""

        def _guard(fn):
            def inner(*a):
                try:
                    fn(*a)
                    return 0
                except Exception as exc:  # surfaces as the C call's failure
                    print(f"lrgw host transport: {exc!r}", flush=True)
                    return 1
            return inner

        def _u8(ptr, n):
            if n == 0:
                return np.zeros(0, np.uint8)
            return np.ctypeslib.as_array((ctypes.c_uint8 * n).from_address(ptr))

        def ar(_u, buf, n):
            allreduce(np.ctypeslib.as_array((ctypes.c_double * n).from_address(buf)) if n else np.zeros(0))

        def ag(_u, send, recv, n):
            allgather(_u8(send, n), _u8(recv, n * world))

        def a2a(_u, send, sb, recv, rb):
            ss = np.ctypeslib.as_array((ctypes.c_longlong * world).from_address(sb)).copy()
            rs = np.ctypeslib.as_array((ctypes.c_longlong * world).from_address(rb)).copy()
            alltoallv(_u8(send, int(ss.sum())), ss, _u8(recv, int(rs.sum())), rs)

        cbs = (L.ALLREDUCE_FN(_guard(ar)), L.ALLGATHER_FN(_guard(ag)), L.ALLTOALLV_FN(_guard(a2a)))
        t = L.HostTransport(None, *cbs)
        h = L.comm_t()
        _check(L.load().lrgw_comm_create_host(rank, world, ctypes.byref(t), ctypes.byref(h)), None, "comm_host")
        return cls(h, rank, world, keep=(cbs, t))

    @classmethod
    def from_torch(cls, ctx, group=None, transport: str = "auto"):
        """A communicator over the ranks of a torch.distributed group: NCCL
        (the id broadcast from rank 0) when the group's backend is nccl and
        transport is auto / nccl; otherwise the host transport on the group."""
        import torch.distributed as dist

        rank, world = dist.get_rank(group), dist.get_world_size(group)
        use_nccl = transport == "nccl" or (transport == "auto" and dist.get_backend(group) == "nccl")
        if use_nccl:
            obj = [cls.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group else 0, group=group)
            return cls.nccl(ctx, rank, world, obj[0])
        return cls.host(rank, world, *torch_host_transport(group))

    def close(self):
        if getattr(self, "handle", None):
            self._lib.lrgw_comm_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def torch_host_transport(group=None):
    """The three host-transport callables over a torch.distributed group
    (CPU tensors viewing the library's pinned staging buffers)."""
    import torch
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)

    def _glob(q):
        return dist.get_global_rank(group, q) if group is not None else q

    def allreduce(arr):
        if arr.size:
            dist.all_reduce(torch.from_numpy(arr), group=group)

    def allgather(send, recv):
        n = send.size
        if n == 0:
            return
        outs = [torch.from_numpy(recv[q * n:(q + 1) * n]) for q in range(world)]
        dist.all_gather(outs, torch.from_numpy(send), group=group)

    def alltoallv(send, ss, recv, rs):
        so = np.concatenate([[0], np.cumsum(ss)]).astype(np.int64)
        ro = np.concatenate([[0], np.cumsum(rs)]).astype(np.int64)
        recv[ro[rank]:ro[rank + 1]] = send[so[rank]:so[rank + 1]]
        reqs = []
        for q in range(world):
            if q == rank:
                continue
            if ss[q]:
                reqs.append(dist.isend(torch.from_numpy(send[so[q]:so[q + 1]]), _glob(q), group=group))
            if rs[q]:
                reqs.append(dist.irecv(torch.from_numpy(recv[ro[q]:ro[q + 1]]), _glob(q), group=group))
        for r in reqs:
            r.wait()

    return allreduce, allgather, alltoallv


def build_sharded(comm: Comm, phi_v_p, phi_c_p, energies, dims, cell, k_mu: float = 8.0, n_lambda: int = 16,
                  delta_rel: float = 1e-7, max_nodes: int = 1025, zero_kernel: bool = False,
                  ctx=None) -> EpsilonInverseLowRank:
    """lrgw_build_sharded: each rank passes its own z-panel (z_panel) of the
    orbitals (column-major float64 CUDA tensors, rows x N_v / rows x N_c)."""
    c = _ctx(ctx)
    _, rows = z_panel(dims, comm.world, comm.rank)
    prm, pv, ldv, pc, ldc, e = _build_params(c, phi_v_p, phi_c_p, energies, dims, cell, k_mu, n_lambda, delta_rel,
                                             max_nodes, zero_kernel, rows=rows)
    _sync_torch(phi_v_p)
    h = L.eps_t()
    _check(c._lib.lrgw_build_sharded(c.handle, comm.handle, ctypes.byref(prm), ctypes.c_void_p(pv), ldv,
                                     ctypes.c_void_p(pc), ldc, _dp(e), ctypes.byref(h)), c.handle, "build_sharded")
    return EpsilonInverseLowRank(c, h)


def eps_apply_sharded(comm: Comm, e: EpsilonInverseLowRank, x_p, y_p):
    """y_p = (eps^-1 x)_p on this rank's panel rows (column-major float64 CUDA tensors)."""
    px, ldx = _dev_ptr_cm(x_p)
    py, ldy = _dev_ptr_cm(y_p)
    _sync_torch(x_p)
    _check(e.ctx._lib.lrgw_eps_apply_sharded(e.ctx.handle, comm.handle, e.handle, ctypes.c_void_p(px), ldx,
                                             x_p.shape[1], ctypes.c_void_p(py), ldy), e.ctx.handle,
           "eps_apply_sharded")
    return y_p
