"""Build/load the oracle's plain-C helpers (TEST INFRASTRUCTURE ONLY).

`build()` compiles oracle/csrc/*.c with gcc into oracle/liboracle.so; the
library is loaded lazily with ctypes.  Nothing here is linked by the product.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRCS = [os.path.join(_HERE, "csrc", f) for f in ("oracle_thomas.c", "oracle_band.c")]
_SO = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(_SO) or any(os.path.getmtime(_SO) < os.path.getmtime(s) for s in _SRCS):
        cmd = ["gcc", "-O3", "-fopenmp", "-fPIC", "-shared", "-o", _SO + ".tmp"] + _SRCS + ["-lm"]
        subprocess.check_call(cmd)
        os.replace(_SO + ".tmp", _SO)
    return _SO


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        dp = ctypes.POINTER(ctypes.c_double)
        L.oracle_thomas_batch.argtypes = [ctypes.c_int, dp, dp, dp, dp, dp, ctypes.c_long, dp]
        L.oracle_thomas_batch.restype = None
        L.oracle_band_factor.argtypes = [ctypes.c_int, ctypes.c_double, dp]
        L.oracle_band_factor.restype = ctypes.c_long
        L.oracle_band_solve.argtypes = [ctypes.c_int, dp, ctypes.c_long, dp]
        L.oracle_band_solve.restype = None
        _lib = L
    return _lib


def _ptr(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def thomas_batch(sub, diag, sup, X, shift=None, rowsum=None):
    """Solve tridiag(sub, diag + shift[s], sup) x_s = X[s] in place; X is (nsys, n).

    rowsum (optional, exact sub+diag+sup) selects the row-sum pivot recurrence."""
    assert X.dtype == np.float64 and X.flags.c_contiguous and X.ndim == 2
    n = X.shape[1]
    sub = np.ascontiguousarray(sub, dtype=np.float64)
    diag = np.ascontiguousarray(diag, dtype=np.float64)
    sup = np.ascontiguousarray(sup, dtype=np.float64)
    sh = None
    if shift is not None:
        sh = np.ascontiguousarray(shift, dtype=np.float64)
        assert sh.shape == (X.shape[0],)
    rs = None
    if rowsum is not None:
        rs = np.ascontiguousarray(rowsum, dtype=np.float64)
        assert rs.shape == (n,)
    lib().oracle_thomas_batch(n, _ptr(sub), _ptr(diag), _ptr(sup),
                              _ptr(rs) if rs is not None else None,
                              _ptr(sh) if sh is not None else None, X.shape[0], _ptr(X))
    return X


def band_factor(n: int, dt: float) -> np.ndarray:
    """Banded Cholesky factor of I + dt A for the n x n 5-point Dirichlet
    Laplacian (oracle_band.c): ((n*n), n+1) band rows."""
    L = np.zeros((n * n, n + 1))
    bad = lib().oracle_band_factor(int(n), float(dt), _ptr(L))
    if bad:
        raise np.linalg.LinAlgError(f"non-positive pivot at row {bad - 1}")
    return L


def band_solve(n: int, L: np.ndarray, X: np.ndarray) -> np.ndarray:
    """X (nvec, n*n), C-contiguous fp64, solved in place with the factor L."""
    assert X.dtype == np.float64 and X.flags.c_contiguous and X.shape[-1] == n * n
    lib().oracle_band_solve(int(n), _ptr(L), X.shape[0], _ptr(X))
    return X
