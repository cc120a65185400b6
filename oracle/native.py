"""ctypes loader for oracle/build/liboracle.so — TEST INFRASTRUCTURE ONLY."""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "build", "liboracle.so")
_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        p = ctypes.c_void_p
        L.oracle_cheb_filter_f64.argtypes = [ctypes.c_int64, p, p, p, ctypes.c_int64, p, p,
                                             ctypes.c_int32, ctypes.c_double, p, p, ctypes.c_int32]
        L.oracle_cheb_filter_f64.restype = ctypes.c_int
        L.oracle_sumsq_f64.argtypes = [ctypes.c_int64, p]
        L.oracle_sumsq_f64.restype = ctypes.c_double
        L.oracle_num_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def num_threads() -> int:
    return int(lib().oracle_num_threads())


def cheb_filter(indptr, indices, data, lambda_max, coeffs, x, nthreads: int = 0) -> np.ndarray:
    """C restatement of apply_filter (filters.py:155-187); returns a new array."""
    indptr = np.ascontiguousarray(indptr, dtype=np.int32)
    indices = np.ascontiguousarray(indices, dtype=np.int32)
    data = np.ascontiguousarray(data, dtype=np.float64)
    x = np.ascontiguousarray(x, dtype=np.float64)
    coeffs = np.ascontiguousarray(coeffs, dtype=np.float64)
    n, d = x.shape
    out = np.empty_like(x)
    work = np.empty(2 * n * d, dtype=np.float64)
    rc = lib().oracle_cheb_filter_f64(n, indptr.ctypes.data, indices.ctypes.data, data.ctypes.data,
                                      d, x.ctypes.data, coeffs.ctypes.data, len(coeffs),
                                      float(lambda_max), out.ctypes.data, work.ctypes.data,
                                      int(nthreads))
    if rc != 0:
        raise ValueError("oracle_cheb_filter_f64 rejected its arguments")
    return out
