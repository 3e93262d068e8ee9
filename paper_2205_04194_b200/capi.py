"""ctypes binding of libimqfast.so (include/imqfast.h).

This is the reference-facing surface: the same 22 ``imq_*`` entry points as
/root/reference/proj/include/imqfast.h plus the additive ``imq_ext_*`` device
extensions.  Loading fails loudly when the CUDA library has not been built;
there is no Python or CPU fallback behind any of these calls.
"""
from __future__ import annotations

import ctypes as C
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("IMQ_LIB_PATH") or os.path.join(HERE, "libimqfast.so")  # override: experiments
HEADER = os.path.join(os.path.dirname(HERE), "include", "imqfast.h")

IMQ_OK = 0
IMQ_ERR_INVALID_ARG = 1
IMQ_ERR_SINGULAR = 2
IMQ_ERR_IO = 3
IMQ_ERR_INTERNAL = 4

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_vp = C.c_void_p


class imq_solve_stats(C.Structure):
    _fields_ = [("iterations", C.c_int), ("final_relative_residual", C.c_double),
                ("converged", C.c_int)]


class imq_verify_config(C.Structure):
    _fields_ = [("xy", _dp), ("n", C.c_size_t), ("t", C.c_double), ("m", C.c_int),
                ("levels", C.c_int), ("seed", C.c_ulonglong)]


class imq_ext_stats(C.Structure):
    _fields_ = [("n", C.c_int), ("m", C.c_int), ("levels", C.c_int), ("device", C.c_int),
                ("origin_x", C.c_double), ("origin_y", C.c_double), ("side", C.c_double),
                ("far_pairs", C.c_double), ("near_pairs", C.c_double),
                ("far_items", C.c_longlong), ("near_items", C.c_longlong),
                ("near_mode", C.c_int), ("far_pairs_direct", C.c_double),
                ("cheb_node_pairs", C.c_double), ("cheb_levels", C.c_int), ("cheb_ring", C.c_int),
                ("kernel_launches", C.c_int), ("cheb_xring", C.c_int),
                ("cert_estimate", C.c_double), ("cert_budget", C.c_double),
                ("cert_scale", C.c_double), ("cert_by_kind", C.c_double * 5),
                ("cert_fallbacks", C.c_int), ("cert_rounds", C.c_int),
                ("gemm_node_pairs", C.c_double)]


class imq_ext_options(C.Structure):
    _fields_ = [("flags", C.c_uint), ("ring_tau", C.c_double), ("ring2_tau", C.c_double),
                ("inner_tau", C.c_double), ("xring_tau", C.c_double), ("far_rmax", C.c_int),
                ("far_streams", C.c_int), ("cert_budget", C.c_double)]


OPT = dict(no_cheb=0x1, no_ring=0x2, no_inner=0x4, no_xring=0x8, no_lsplit=0x10, no_split=0x20,
           near_no_sym=0x40, near_no_pair=0x80, cert_report=0x100, trace=0x200)

VERIFY_CB = C.CFUNCTYPE(None, C.c_char_p, C.c_int, C.c_double, C.c_void_p)

_SIGS = {
    "imq_last_error": (C.c_char_p, []),
    "imq_operator_create": (C.c_int, [_dp, C.c_size_t, C.c_double, C.c_int, C.c_int,
                                      C.POINTER(_vp)]),
    "imq_operator_destroy": (None, [_vp]),
    "imq_operator_size": (C.c_int, [_vp, C.POINTER(C.c_size_t)]),
    "imq_operator_levels": (C.c_int, [_vp, _ip]),
    "imq_operator_apply": (C.c_int, [_vp, _dp, _dp]),
    "imq_dense_matvec": (C.c_int, [_dp, C.c_size_t, C.c_double, _dp, _dp]),
    "imq_dense_solve": (C.c_int, [_dp, C.c_size_t, C.c_double, _dp, _dp, _dp]),
    "imq_iterative_solve": (C.c_int, [_vp, _dp, C.c_double, C.c_int, C.c_int, _dp,
                                      C.POINTER(imq_solve_stats)]),
    "imq_evaluate_interpolant": (C.c_int, [_dp, _dp, C.c_size_t, C.c_double, _dp, C.c_size_t,
                                           _dp]),
    "imq_green_exact": (C.c_int, [_dp, _dp, _dp]),
    "imq_green_truncated": (C.c_int, [_dp, _dp, C.c_int, _dp]),
    "imq_truncation_error_bound": (C.c_int, [C.c_double, C.c_double, C.c_int, _dp]),
    "imq_auto_level": (C.c_int, [C.c_size_t, C.c_int, _ip]),
    "imq_cost_upper_bound": (C.c_int, [C.c_size_t, C.c_int, C.c_int, _dp]),
    "imq_halton2d": (C.c_int, [C.c_size_t, _dp]),
    "imq_random_vector": (C.c_int, [C.c_size_t, C.c_ulonglong, _dp]),
    "imq_read_points": (C.c_int, [C.c_char_p, C.POINTER(_dp), C.POINTER(C.c_size_t)]),
    "imq_write_points": (C.c_int, [C.c_char_p, _dp, C.c_size_t]),
    "imq_free": (None, [_vp]),
    "imq_set_threads": (C.c_int, [C.c_int]),
    "imq_verify": (C.c_int, [C.POINTER(imq_verify_config), VERIFY_CB, _vp]),
    "imq_ext_operator_create_opts": (C.c_int, [_dp, C.c_size_t, C.c_double, C.c_int, C.c_int,
                                               C.POINTER(imq_ext_options), C.POINTER(_vp)]),
    "imq_ext_operator_apply_batch": (C.c_int, [_vp, C.c_int, _dp, _dp]),
    "imq_ext_operator_apply_block": (C.c_int, [_vp, C.c_int, _dp, _dp]),
    "imq_ext_operator_apply_block_device": (C.c_int, [_vp, C.c_int, _vp, _vp, _vp]),
    "imq_ext_operator_apply_device": (C.c_int, [_vp, _vp, _vp, _vp]),
    "imq_ext_operator_apply_sorted_device": (C.c_int, [_vp, _vp, _vp, _vp]),
    "imq_ext_operator_synchronize": (C.c_int, [_vp]),
    "imq_ext_operator_permutation": (C.c_int, [_vp, _ip]),
    "imq_ext_operator_leaf_start": (C.c_int, [_vp, _ip, C.c_size_t]),
    "imq_ext_operator_stats": (C.c_int, [_vp, C.POINTER(imq_ext_stats)]),
    "imq_ext_iterative_solve": (C.c_int, [_vp, _dp, C.c_double, C.c_int, C.c_int, _dp,
                                          C.POINTER(imq_solve_stats), _dp, C.c_int, _ip]),
    "imq_ext_operator_moments": (C.c_int, [_vp, _vp, _vp]),
    "imq_ext_operator_coefficients": (C.c_int, [_vp, C.POINTER(_vp), C.POINTER(C.c_size_t),
                                                C.POINTER(C.c_longlong), C.c_int]),
    "imq_ext_operator_items": (C.c_int, [_vp, C.c_int, _ip, C.c_size_t,
                                         C.POINTER(C.c_size_t)]),
    "imq_ext_operator_far_near": (C.c_int, [_vp, _vp, _vp, C.c_int, C.c_int, C.c_int, C.c_int,
                                            C.c_int, _vp]),
    "imq_ext_operator_gather": (C.c_int, [_vp, _vp, _vp, _vp]),
    "imq_ext_operator_near_begin": (C.c_int, [_vp, _vp, _vp]),
    "imq_ext_operator_moments_local": (C.c_int, [_vp, _vp, _vp]),
    "imq_ext_operator_coarse_moments": (C.c_int, [_vp, C.POINTER(_vp), C.POINTER(C.c_size_t)]),
    "imq_ext_operator_moments_finish": (C.c_int, [_vp, _vp]),
    "imq_ext_shard_bounds": (C.c_int, [_ip, C.c_int, C.c_int, _ip]),
    "imq_ext_shard_bounds_work": (C.c_int, [_ip, C.c_int, C.c_int, C.c_int, _ip]),
    "imq_ext_operator_restrict": (C.c_int, [_vp, C.c_int, C.c_int]),
    "imq_ext_operator_check_lists": (C.c_int, [_vp, C.c_int, C.POINTER(C.c_longlong)]),
    "imq_ext_operator_local_leaves": (C.c_int, [_vp, _ip, C.c_size_t, C.POINTER(C.c_size_t)]),
    "imq_ext_fp64_peak": (C.c_int, [C.c_int, _dp, _dp]),
    "imq_ext_device_count": (C.c_int, [_ip]),
    "imq_ext_set_device": (C.c_int, [C.c_int]),
}

_lib = None


class IMQError(RuntimeError):
    """Error returned through the C ABI; ``code`` is the IMQ_ERR_* value."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code
        self.msg = msg


def header_symbols() -> list[str]:
    """Function names declared in include/imqfast.h."""
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(imq_\w+)\s*\(", txt)) - {"imq_verify_callback"})


def lib() -> C.CDLL:
    """The loaded CUDA library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with "
                              "`python -m paper_2205_04194_b200.build` (nvcc, sm_100a)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc != IMQ_OK:
        raise IMQError(rc, lib().imq_last_error().decode())
