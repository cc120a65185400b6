"""ctypes binding of libcscb200.so (the C ABI in include/csc_b200.h).

There is no CPU fallback: every compute entry point requires the CUDA
library and a visible CUDA device, and fails loudly otherwise.
"""
from __future__ import annotations

import ctypes
import os
import re

from ._build import LIB, INCLUDE

CSC_OK, CSC_ERR_ARG, CSC_ERR_CUDA, CSC_ERR_CAPACITY = 0, 1, 2, 3
CSC_F64, CSC_F32 = 0, 1
CSC_LAP_NORMALIZED, CSC_LAP_COMBINATORIAL = 0, 1

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int32
_INT = ctypes.c_int
_D = ctypes.c_double
_PI64 = ctypes.POINTER(ctypes.c_int64)
_PD = ctypes.POINTER(ctypes.c_double)

# argtypes per exported symbol (mirrors include/csc_b200.h)
SIGNATURES = {
    "csc_version": ([], _INT),
    "csc_last_error": ([], ctypes.c_char_p),
    "csc_device_info": ([ctypes.POINTER(_INT)] * 3, _INT),
    "csc_laplacian_build": ([_I64, _I64, _P, _P, _P, _INT, _P, _P, _P, _I64, _P, _PI64, _PD, _P], _INT),
    "csc_edge_delta": ([_I64, _P, _I64, _P, _I64, _P, _I64, _P, _I64, _PI64, _P], _INT),
    "csc_graph_canonicalize": ([_I64, _I64, _P, _P, _P, _P, _P, _P, _P], _INT),
    "csc_codes_split": ([_I64, _P, _I64, _P, _P, _P], _INT),
    "csc_chebop_create": ([_P, _P, _P, _I64, _I64, _D, _INT, _P, ctypes.POINTER(_P)], _INT),
    "csc_chebop_destroy": ([_P], _INT),
    "csc_chebop_export": ([_P, _P, _P, _P, _P, _P, _P], _INT),
    "csc_chebop_info": ([_P, _PI64, _PI64, _PI64, _PI64], _INT),
    "csc_chebop_schedule": ([_P, ctypes.POINTER(_I32), _PD], _INT),
    "csc_cheb_filter": ([_P, _P, _I64, _I64, _PD, _I32, _P, _P, _P, _P], _INT),
    "csc_cheb_filter_download": ([_P, _P, _I64, _I64, _PD, _I32, _P, _P, _P, _I64, _I32, _P, _P], _INT),
    "csc_cheb_moments": ([_P, _P, _I64, _I64, _I32, _P, _P, _P], _INT),
    "csc_cheb_moments_keep": ([_P, _P, _I64, _I64, _I32, _P, _P, _P], _INT),
    "csc_cheb_combine": ([_P, _P, _I64, _I64, _I64, _PD, _I32, _P, _P, _P], _INT),
    "csc_sumsq": ([_P, _I64, _INT, _P, _P, _P], _INT),
    "csc_copy2d_async": ([_P, _I64, _P, _I64, _I64, _I64, _P], _INT),
    "csc_set_tuning": ([ctypes.c_char_p, _I64], _INT),
    "csc_sweep_timing": ([_INT], _INT),
    "csc_sweep_last_launch": ([ctypes.c_char_p, _INT, ctypes.POINTER(_INT)], _INT),
    "csc_sweep_times": ([ctypes.POINTER(ctypes.c_float), _INT, ctypes.POINTER(_INT)], _INT),
    "csc_kmeans_rownorms": ([_P, _I64, _I64, _I64, _P, _P], _INT),
    "csc_kmeans_assign": ([_P, _P, _I64, _I64, _I64, _P, _I64, _P, _I64, _P, _P, _P, _P], _INT),
    "csc_kmeans_plan_create": ([_I64, _I64, _I64, _I64, _P, ctypes.POINTER(_P)], _INT),
    "csc_kmeans_plan_destroy": ([_P], _INT),
    "csc_kmeans_plan_stats": ([_P, _PI64, ctypes.POINTER(_I32)], _INT),
    "csc_kmeans_plan_screen_stats": ([_P, _PI64], _INT),
    "csc_gen_planted_partition": ([_I64, _I32, _P, ctypes.c_uint64, _P, _I64, _PI64, _P], _INT),
    "csc_gen_chung_lu": ([_I64, _I32, _P, _P, _I64, ctypes.c_uint64, _P, _I64, _PI64, _P], _INT),
    "csc_gen_edge_churn": ([_I64, _P, _I64, _P, _I32, _D, _D, _I64, ctypes.c_uint64, _P, _PI64, _P, _PI64, _P],
                           _INT),
    "csc_gen_node_switch": ([_I64, _P, _I64, _P, _I32, _D, _D, _I64, ctypes.c_uint64, _P, _PI64, _P, _I64, _PI64,
                             _P], _INT),
    "csc_kmeans_iterate": ([_P, _P, _P, _P, _I64, _P, _P, _P, _INT, _P, _P], _INT),
    "csc_kmeans_run": ([_P, _P, _P, _P, _I64, _P, _P, _P, _INT, _D, _P, _P, _P], _INT),
    "csc_kmeans_tuning": ([ctypes.c_char_p, _I64], _INT),
    "csc_pool_stats": ([_P], _INT),
    "csc_kmeans_screen_supported": ([_I64, _I64], _INT),
    "csc_kmeans_tc_supported": ([_I64, _I64], _INT),
    "csc_kmeans_tc_distances": ([_P, _I64, _I64, _I64, _P, _P, _I64, _I64, _P, _P, _P], _INT),
    "csc_kmeans_screen_prepare": ([_P, _I64, _I64, _I64, _P, _I64, _P, _P], _INT),
    "csc_kmeans_plan_set_screen": ([_P, _P, _I64, _P], _INT),
    "csc_kmeans_repair": ([_P, _P, _P, _I64, _I64, _P], _INT),
    "csc_kmeans_update": ([_P, _P, _I64, _I64, _I64, _I64, _P, _I64, _P, _P, _P], _INT),
    "csc_kmeans_cost": ([_P, _P, _P, _I64, _I64, _I64, _I64, _P, _P], _INT),
    "csc_kmeans_fused_supported": ([_I64, _I64, _I64, _I64, _INT], _INT),
    "csc_kmeans_fused_trace": ([_P, _I64], _INT),
    "csc_kmeans_fused_kpp_run": ([_P, _I64, _I64, _I64, _I64, _I64, _P, _P, _I64, _INT, _D, _P, _P, _P, _P, _P, _P],
                                 _INT),
    "csc_kmeans_fused_run": ([_P, _P, _I64, _I64, _I64, _I64, _I64, _P, _I64, _INT, _D, _P, _P, _P, _P], _INT),
    "csc_kmeanspp_nchunks": ([_I64], _INT),
    "csc_kmeanspp_dist": ([_P, _I64, _I64, _I64, _P, _P, _INT, _P, _I64, _P, _P], _INT),
    "csc_kmeanspp_pick": ([_P, _I64, _I64, _I64, _P, _P, _I64, _D, _I64, _P, _P, _P], _INT),
    "csc_kmeanspp_batch": ([_P, _I64, _I64, _I64, _I64, _I64, _P, _P, _P, _I64, _P, _P], _INT),
    "csc_seed_states": ([_P, _I64, _P, _I64, _I64, _I64, _I32, _P], _INT),
    "csc_normal_columns": ([_P, _I64, _I64, _D, _P, _I64, _I64, _P, _P], _INT),
    "csc_normal_columns_async": ([_P, _I64, _I64, _D, _P, _I64, _I64, _P, _P], _INT),
    "csc_gather_columns": ([_P, _I64, _I64, _P, _I64, _P, _I64, _I64, _P], _INT),
}

_lib = None


class NativeError(RuntimeError):
    """A CUDA-side failure inside libcscb200."""


def header_symbols() -> list[str]:
    """Function names declared in include/csc_b200.h."""
    with open(os.path.join(INCLUDE, "csc_b200.h")) as fh:
        text = fh.read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(csc_\w+)\s*\(", text, re.M)))


def load(path: str | None = None):
    """Load the shared library (no device needed) and bind every signature.

    CSC_LIB overrides the in-tree path (A/B of alternative builds in tools/)."""
    global _lib
    if path is None:
        path = os.environ.get("CSC_LIB") or LIB
    if _lib is None:
        if not os.path.exists(path):
            raise ImportError(f"libcscb200.so not built ({path}); run __graft_entry__.build()")
        lib = ctypes.CDLL(path)
        for name, (args, res) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        _lib = lib
    return _lib


def lib():
    return load()


def last_error() -> str:
    msg = lib().csc_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str) -> None:
    """Map a C status to the reference's exception types."""
    if rc == CSC_OK:
        return
    msg = last_error() or what
    if rc in (CSC_ERR_ARG, CSC_ERR_CAPACITY):
        raise ValueError(msg)
    raise NativeError(msg)


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args), name)
