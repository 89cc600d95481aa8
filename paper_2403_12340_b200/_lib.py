"""ctypes loader for liblrgw_cuda.so (include/lrgw_cuda.h).

The product path has no fallback: if the shared library is missing or fails to
load, importing the API raises. Build it with `python -c "import
__graft_entry__ as g; g.build()"` or `make -C paper_2403_12340_b200/csrc`.
"""
from __future__ import annotations

import ctypes
import os
import re

_HERE = os.path.dirname(os.path.abspath(__file__))
# LRGW_LIB: an alternative build of the same library (A/B experiments of tools/)
LIB_PATH = os.environ.get("LRGW_LIB") or os.path.join(_HERE, "lib", "liblrgw_cuda.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "lrgw_cuda.h")

_lib = None

c_double_p = ctypes.POINTER(ctypes.c_double)
c_int_p = ctypes.POINTER(ctypes.c_int)
c_int32_p = ctypes.POINTER(ctypes.c_int32)
c_ll = ctypes.c_longlong
ctx_t = ctypes.c_void_p
eps_t = ctypes.c_void_p


class BuildParams(ctypes.Structure):
    """lrgw_build_params (include/lrgw_cuda.h)."""
    _fields_ = [
        ("n_r", ctypes.c_int), ("n_v", ctypes.c_int), ("n_c", ctypes.c_int),
        ("dims", ctypes.c_int * 3), ("cell", ctypes.c_double * 3),
        ("k_mu", ctypes.c_double), ("n_lambda", ctypes.c_int),
        ("delta_rel", ctypes.c_double), ("max_nodes", ctypes.c_int),
        ("zero_kernel", ctypes.c_int), ("n_e", ctypes.c_int),
    ]


class EpsInfo(ctypes.Structure):
    """lrgw_eps_info (include/lrgw_cuda.h)."""
    _fields_ = [
        ("n_r", ctypes.c_int), ("n_mu", ctypes.c_int),
        ("theta", ctypes.c_void_p), ("k", ctypes.c_void_p), ("t", ctypes.c_void_p), ("pvp", ctypes.c_void_p),
        ("min_margin", ctypes.c_double), ("min_margin_step", ctypes.c_int), ("fit_path", ctypes.c_int),
        ("lp_diag_ratio", ctypes.c_double), ("select_blocks", ctypes.c_int),
    ]


comm_t = ctypes.c_void_p
ALLREDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_longlong)
ALLGATHER_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_longlong)
ALLTOALLV_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                ctypes.c_void_p)


class HostTransport(ctypes.Structure):
    """lrgw_host_transport (include/lrgw_cuda.h)."""
    _fields_ = [("user", ctypes.c_void_p), ("allreduce_sum_f64", ALLREDUCE_FN), ("allgather", ALLGATHER_FN),
                ("alltoallv", ALLTOALLV_FN)]


# name -> (restype, argtypes)
_SIGS = {
    "lrgw_abi_version": (ctypes.c_int, []),
    "lrgw_ctx_create": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ctx_t)]),
    "lrgw_ctx_destroy": (ctypes.c_int, [ctx_t]),
    "lrgw_ctx_set_stream": (ctypes.c_int, [ctx_t, ctypes.c_void_p]),
    "lrgw_ctx_stream": (ctypes.c_void_p, [ctx_t]),
    "lrgw_ctx_synchronize": (ctypes.c_int, [ctx_t]),
    "lrgw_ctx_last_error": (ctypes.c_char_p, [ctx_t]),
    "lrgw_ctx_last_pivot": (ctypes.c_int, [ctx_t]),
    "lrgw_ctx_stage_ms": (ctypes.c_int, [ctx_t, c_double_p, ctypes.c_int]),
    "lrgw_ctx_kernel_launches": (ctypes.c_longlong, [ctx_t]),
    "lrgw_ctx_set_select_batch": (ctypes.c_int, [ctx_t, ctypes.c_int]),
    "lrgw_ctx_set_theta_implicit": (ctypes.c_int, [ctx_t, ctypes.c_int]),
    "lrgw_num_aux": (ctypes.c_int, [ctypes.c_double, ctypes.c_int, ctypes.c_int, c_int_p]),
    "lrgw_elliptic_k": (ctypes.c_int, [ctypes.c_double, c_double_p]),
    "lrgw_jacobi_sn_cn_dn": (ctypes.c_int, [ctypes.c_double, ctypes.c_double, c_double_p]),
    "lrgw_jacobi_complex": (ctypes.c_int, [ctypes.c_double, ctypes.c_double, ctypes.c_double, c_double_p]),
    "lrgw_elliptic_params": (ctypes.c_int, [c_double_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                            ctypes.c_double, ctypes.c_int, c_double_p]),
    "lrgw_cauchy_error_bound": (ctypes.c_int, [c_double_p, ctypes.c_int, c_double_p]),
    "lrgw_select_interpolation_points": (ctypes.c_int, [ctx_t, c_double_p, c_double_p, ctypes.c_int,
                                                        ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                                        ctypes.c_int, c_int32_p]),
    "lrgw_fit_auxiliary_basis": (ctypes.c_int, [ctx_t, c_double_p, c_double_p, ctypes.c_int, ctypes.c_int,
                                                ctypes.c_int, c_int32_p, ctypes.c_int, c_double_p]),
    "lrgw_coupled_coefficients_direct": (ctypes.c_int, [ctx_t, c_double_p, c_double_p, ctypes.c_int,
                                                        ctypes.c_int, ctypes.c_int, c_double_p, ctypes.c_int,
                                                        c_double_p]),
    "lrgw_sum_node_terms": (ctypes.c_int, [ctx_t, c_double_p, c_double_p, ctypes.c_int, ctypes.c_int,
                                           ctypes.c_int, c_double_p, ctypes.c_int, c_double_p, c_double_p,
                                           c_double_p, ctypes.c_int, c_double_p]),
    "lrgw_coupled_coefficients_fixed": (ctypes.c_int, [ctx_t, c_double_p, c_double_p, ctypes.c_int,
                                                       ctypes.c_int, ctypes.c_int, c_double_p, ctypes.c_int,
                                                       ctypes.c_int, c_double_p]),
    "lrgw_coupled_coefficients_contour": (ctypes.c_int, [ctx_t, c_double_p, c_double_p, ctypes.c_int,
                                                         ctypes.c_int, ctypes.c_int, c_double_p, ctypes.c_int,
                                                         ctypes.c_double, ctypes.c_int, c_double_p, c_int_p,
                                                         c_double_p]),
    "lrgw_contour_refinement_levels": (ctypes.c_int, [ctx_t, c_double_p, c_double_p, ctypes.c_int,
                                                      ctypes.c_int, ctypes.c_int, c_double_p, ctypes.c_int,
                                                      ctypes.c_int, ctypes.c_int, c_double_p, c_int_p,
                                                      c_int_p]),
    "lrgw_coulomb_kernel": (ctypes.c_int, [c_int_p, c_double_p, c_double_p]),
    "lrgw_apply_coulomb": (ctypes.c_int, [ctx_t, c_int_p, c_double_p, ctypes.c_int, c_double_p,
                                          ctypes.c_int, c_double_p]),
    "lrgw_assemble_K": (ctypes.c_int, [ctx_t, c_double_p, c_double_p, ctypes.c_int, ctypes.c_int, c_int_p,
                                       c_double_p, ctypes.c_int, c_double_p]),
    "lrgw_build_epsilon_inverse": (ctypes.c_int, [ctx_t, c_double_p, c_double_p, ctypes.c_int, ctypes.c_int,
                                                  c_int_p, c_double_p, ctypes.c_int, ctypes.POINTER(eps_t)]),
    "lrgw_eps_from_parts": (ctypes.c_int, [ctx_t, c_double_p, c_double_p, ctypes.c_int, ctypes.c_int,
                                           c_int_p, c_double_p, ctypes.c_int, ctypes.POINTER(eps_t)]),
    "lrgw_epsilon_inverse_apply": (ctypes.c_int, [ctx_t, eps_t, c_double_p, ctypes.c_int, c_double_p]),
    "lrgw_eps_get": (ctypes.c_int, [ctx_t, eps_t, c_double_p, c_double_p, c_double_p, c_double_p,
                                    c_int32_p]),
    "lrgw_eps_shape": (ctypes.c_int, [eps_t, c_int_p, c_int_p]),
    "lrgw_eps_destroy": (ctypes.c_int, [eps_t]),
    "lrgw_build": (ctypes.c_int, [ctx_t, ctypes.POINTER(BuildParams), ctypes.c_void_p, c_ll, ctypes.c_void_p,
                                  c_ll, c_double_p, ctypes.POINTER(eps_t)]),
    "lrgw_eps_info_get": (ctypes.c_int, [eps_t, ctypes.POINTER(EpsInfo)]),
    "lrgw_eps_device_ptrs": (ctypes.c_int, [eps_t, ctypes.POINTER(ctypes.c_void_p),
                                            ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_void_p)]),
    "lrgw_eps_apply_dev": (ctypes.c_int, [ctx_t, eps_t, ctypes.c_void_p, c_ll, ctypes.c_int, ctypes.c_void_p,
                                          c_ll]),
    "lrgw_dev_select": (ctypes.c_int, [ctx_t, ctypes.c_void_p, c_ll, ctypes.c_int, ctypes.c_void_p, c_ll,
                                       ctypes.c_int, ctypes.c_int, ctypes.c_int, c_int32_p, c_double_p]),
    "lrgw_dev_fit": (ctypes.c_int, [ctx_t, ctypes.c_void_p, c_ll, ctypes.c_int, ctypes.c_void_p, c_ll,
                                    ctypes.c_int, ctypes.c_int, c_int32_p, ctypes.c_int, ctypes.c_void_p, c_ll]),
    "lrgw_dev_fit_panel": (ctypes.c_int, [ctx_t, ctypes.c_void_p, c_ll, ctypes.c_int, ctypes.c_void_p, c_ll,
                                          ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                          ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, c_ll]),
    "lrgw_dev_contour_partial": (ctypes.c_int, [ctx_t, ctypes.c_void_p, c_ll, ctypes.c_void_p, c_ll,
                                                ctypes.c_int, ctypes.c_int, ctypes.c_int, c_double_p,
                                                ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                                ctypes.c_void_p]),
    "lrgw_dev_contour_fixed": (ctypes.c_int, [ctx_t, ctypes.c_void_p, c_ll, ctypes.c_void_p, c_ll,
                                              ctypes.c_int, ctypes.c_int, ctypes.c_int, c_double_p, ctypes.c_int,
                                              ctypes.c_int, ctypes.c_void_p, c_ll]),
    "lrgw_dev_pvp": (ctypes.c_int, [ctx_t, c_int_p, c_double_p, ctypes.c_int, ctypes.c_void_p, c_ll,
                                    ctypes.c_int, ctypes.c_void_p]),
    "lrgw_dev_smw_core": (ctypes.c_int, [ctx_t, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                                         ctypes.c_void_p]),
    "lrgw_dev_coulomb_apply": (ctypes.c_int, [ctx_t, c_int_p, c_double_p, ctypes.c_int, ctypes.c_void_p,
                                              c_ll, ctypes.c_int, ctypes.c_void_p, c_ll]),
    "lrgw_dev_trtri_lower": (ctypes.c_int, [ctx_t, ctypes.c_void_p, ctypes.c_int, ctypes.c_longlong]),
    "lrgw_dev_select_topk": (ctypes.c_int, [ctx_t, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                            ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "lrgw_dev_cand_greedy": (ctypes.c_int, [ctx_t, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                            c_double_p, c_int32_p, c_int32_p, ctypes.c_void_p, ctypes.c_void_p,
                                            ctypes.c_void_p, ctypes.c_void_p, c_int32_p, c_double_p, c_int32_p]),
    "lrgw_dev_theta_from_factor": (ctypes.c_int, [ctx_t, ctypes.c_void_p, c_ll, ctypes.c_int, ctypes.c_int,
                                                  ctypes.c_void_p, c_ll, c_int32_p, ctypes.c_void_p, c_ll]),
    "lrgw_dev_select_panel_update": (ctypes.c_int, [ctx_t, ctypes.c_void_p, c_ll, ctypes.c_int, ctypes.c_void_p,
                                                    c_ll, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, c_ll,
                                                    ctypes.c_int, ctypes.c_int, ctypes.c_void_p, c_ll,
                                                    ctypes.c_void_p, c_ll, ctypes.c_void_p, ctypes.c_void_p]),
    "lrgw_dev_gram_weighted": (ctypes.c_int, [ctx_t, ctypes.c_void_p, c_ll, ctypes.c_int, ctypes.c_int,
                                              ctypes.c_void_p, ctypes.c_void_p, c_ll]),
    "lrgw_project_screened_interactions": (ctypes.c_int, [ctx_t, eps_t, c_double_p, ctypes.c_int, c_double_p,
                                                          ctypes.c_int, c_double_p, c_double_p, c_double_p]),
    "lrgw_dev_project_screened": (ctypes.c_int, [ctx_t, eps_t, ctypes.c_void_p, c_ll, ctypes.c_int, ctypes.c_void_p,
                                                 c_ll, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                                 ctypes.c_void_p]),
    "lrgw_self_energies_lowrank": (ctypes.c_int, [ctx_t, c_double_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                                  c_int32_p, ctypes.c_int, c_int32_p, ctypes.c_int, c_double_p,
                                                  c_double_p, c_double_p, c_double_p, c_double_p, c_double_p,
                                                  c_double_p]),
    "lrgw_dev_self_energies": (ctypes.c_int, [ctx_t, ctypes.c_void_p, c_ll, ctypes.c_int, ctypes.c_int,
                                              ctypes.c_int, c_int32_p, ctypes.c_int, c_int32_p, ctypes.c_int,
                                              ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                              ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "lrgw_last_error": (ctypes.c_char_p, []),
    "lrgw_wfn1_info": (ctypes.c_int, [ctypes.c_char_p, c_int_p, c_double_p, c_int_p, c_int_p]),
    "lrgw_wfn1_load": (ctypes.c_int, [ctypes.c_char_p, c_double_p, c_double_p, c_double_p]),
    "lrgw_wfn1_load_device": (ctypes.c_int, [ctx_t, ctypes.c_char_p, ctypes.c_void_p, c_ll, c_double_p,
                                             c_double_p]),
    "lrgw_wfn1_save": (ctypes.c_int, [ctypes.c_char_p, c_int_p, c_double_p, ctypes.c_int, ctypes.c_int,
                                      c_double_p, c_double_p, c_double_p]),
    "lrgw_nccl_available": (ctypes.c_int, []),
    "lrgw_nccl_unique_id": (ctypes.c_int, [ctypes.c_void_p]),
    "lrgw_comm_create_nccl": (ctypes.c_int, [ctx_t, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                             ctypes.POINTER(comm_t)]),
    "lrgw_comm_create_host": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.POINTER(HostTransport),
                                             ctypes.POINTER(comm_t)]),
    "lrgw_comm_destroy": (ctypes.c_int, [comm_t]),
    "lrgw_comm_info": (ctypes.c_int, [comm_t, c_int_p, c_int_p]),
    "lrgw_z_panel": (ctypes.c_int, [c_int_p, ctypes.c_int, ctypes.c_int, c_int_p, c_int_p]),
    "lrgw_build_sharded": (ctypes.c_int, [ctx_t, comm_t, ctypes.POINTER(BuildParams), ctypes.c_void_p, c_ll,
                                          ctypes.c_void_p, c_ll, c_double_p, ctypes.POINTER(eps_t)]),
    "lrgw_eps_apply_sharded": (ctypes.c_int, [ctx_t, comm_t, eps_t, ctypes.c_void_p, c_ll, ctypes.c_int,
                                              ctypes.c_void_p, c_ll]),
    "lrgw_dev_dgemm": (ctypes.c_int, [ctx_t, ctypes.c_char, ctypes.c_char, ctypes.c_int, ctypes.c_int,
                                      ctypes.c_int, ctypes.c_double, ctypes.c_void_p, c_ll, ctypes.c_void_p,
                                      c_ll, ctypes.c_double, ctypes.c_void_p, c_ll]),
    "lrgw_dev_hadamard": (ctypes.c_int, [ctx_t, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, c_ll, ctypes.c_void_p,
                                         c_ll, ctypes.c_int, ctypes.c_void_p, c_ll, ctypes.c_void_p, c_ll,
                                         ctypes.c_int, ctypes.c_void_p, c_ll]),
}


def header_symbols(path: str = HEADER_PATH):
    """Every function the C-ABI header declares."""
    text = open(path).read()
    return sorted(set(re.findall(r"\b(lrgw_[a-z0-9_]+)\s*\(", text)))


def load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"liblrgw_cuda.so not found at {LIB_PATH}: the B200 extension is not built "
            "(there is no CPU fallback). Run __graft_entry__.build().")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib
