"""ctypes declarations for libftk.so (include/ftk.h).  Argument marshalling only."""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libftk.so")


class PlanOpts(C.Structure):
    _fields_ = [("n_k", C.c_int), ("n_psi", C.c_int), ("radial_rule", C.c_int), ("device", C.c_int),
                ("rank", C.c_int), ("world", C.c_int), ("engine", C.c_int), ("svd_nodes", C.c_int),
                ("workspace_bytes", C.c_size_t), ("n_gamma", C.c_int), ("nccl_comm", C.c_void_p)]


class PlanInfo(C.Structure):
    _fields_ = [("n", C.c_int), ("n_k", C.c_int), ("n_psi", C.c_int), ("N_t", C.c_int), ("H", C.c_int),
                ("H_plus", C.c_int), ("H0", C.c_int), ("K3", C.c_int), ("ell_max", C.c_int),
                ("K_cycles", C.c_double), ("k_max", C.c_double), ("delta_max", C.c_double), ("W", C.c_double),
                ("eps", C.c_double), ("certificate", C.c_double), ("n_images", C.c_int64),
                ("n_templates_total", C.c_int64), ("n_templates_local", C.c_int64), ("template_offset", C.c_int64),
                ("engine", C.c_int), ("device", C.c_int), ("rank", C.c_int), ("world", C.c_int),
                ("K3p", C.c_int), ("n_rep", C.c_int), ("s3_cols", C.c_int),
                ("s3_nch", C.c_int), ("s3_groups", C.c_int), ("s3_rtiles", C.c_int),
                ("n_gamma", C.c_int), ("n_tau", C.c_int), ("N_t_base", C.c_int)]


class Best(C.Structure):
    _fields_ = [("value", C.c_float), ("template_idx", C.c_int32), ("shift_idx", C.c_int32), ("rot_idx", C.c_int32)]


SYMBOLS = {
    "ftk_plan_create": (C.c_int, [C.c_int, C.c_double, C.c_double, C.c_void_p, C.c_int, C.c_double,
                                  C.POINTER(PlanOpts), C.POINTER(C.c_void_p)]),
    "ftk_plan_create_ctf": (C.c_int, [C.c_int, C.c_double, C.c_double, C.c_void_p, C.c_int, C.c_int, C.c_void_p,
                                      C.c_double, C.POINTER(PlanOpts), C.POINTER(C.c_void_p)]),
    "ftk_radial_rule": (C.c_int, [C.c_int, C.c_double, C.c_int, C.c_int, C.c_void_p, C.c_void_p]),
    "ftk_plan_destroy": (None, [C.c_void_p]),
    "ftk_plan_query": (C.c_int, [C.c_void_p, C.POINTER(PlanInfo)]),
    "ftk_plan_radial": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "ftk_plan_terms": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "ftk_plan_factors": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "ftk_load_images": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_void_p]),
    "ftk_load_templates": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_void_p]),
    "ftk_fb_coeffs": (C.c_int, [C.c_void_p, C.c_int, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p]),
    "ftk_align": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]),
    "ftk_landscape_pairs": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_int64,
                                      C.c_void_p]),
    "ftk_nccl_unique_id": (C.c_int, [C.c_void_p]),
    "ftk_nccl_comm_create": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p)]),
    "ftk_nccl_comm_destroy": (C.c_int, [C.c_void_p]),
    "ftk_align_marginal": (C.c_int, [C.c_void_p, C.c_double, C.c_void_p, C.c_void_p]),
    "ftk_polar_from_pixels": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_void_p, C.c_void_p]),
    "ftk_load_images_pixels": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_void_p]),
    "ftk_load_templates_pixels": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_void_p]),
    "ftk_merge_bests": (C.c_int, [C.c_void_p, C.c_int, C.c_int64, C.c_void_p, C.c_void_p]),
    "ftk_merge_bests_host": (C.c_int, [C.c_void_p, C.c_int, C.c_int64, C.c_void_p]),
    "ftk_set_profiling": (C.c_int, [C.c_void_p, C.c_int]),
    "ftk_kernel_times": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "ftk_tc_selftest": (C.c_int, [C.c_int, C.c_void_p, C.c_void_p]),
    "ftk_last_error": (C.c_char_p, [C.c_void_p]),
    "ftk_status_string": (C.c_char_p, [C.c_int]),
    "ftk_version": (C.c_int, []),
}

_lib = None


def lib():
    """Load libftk.so (fails loudly if it was not built: no fallback exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SYMBOLS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib
