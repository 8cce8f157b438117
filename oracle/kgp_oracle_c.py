"""ctypes binding for the C oracle (oracle/kgp_oracle.c). Test/baseline infrastructure only."""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "build", "libkgp_oracle.so")
KERNEL_IDS = {"gaussian": 0, "matern32": 1, "matern52": 2}
_lib = None


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        _lib = ctypes.CDLL(LIB_PATH)
        _lib.kgpo_matmul.restype = ctypes.c_int
        _lib.kgpo_matmul.argtypes = [
            ctypes.c_int, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, ctypes.c_double,
            ctypes.c_double, ctypes.c_double, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
        _lib.kgpo_max_threads.restype = ctypes.c_int
        _lib.kgpo_panel.restype = ctypes.c_int
        _lib.kgpo_panel.argtypes = [
            ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p,
            ctypes.c_void_p, ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_int, ctypes.c_void_p,
            ctypes.c_int]
    return _lib


def max_threads() -> int:
    return int(lib().kgpo_max_threads())


def matmul(kt, x, l, f, s, b, row0=0, nrows=None, want_k=True, want_dl=False, nthreads=0):
    """Rows [row0, row0+nrows) of Khat.B and/or dKhat/dl.B (fp64)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    if b.ndim == 1:
        b = b[:, None]
    n, d = x.shape
    k = b.shape[1]
    nrows = n - row0 if nrows is None else nrows
    ok = np.empty((nrows, k)) if want_k else None
    od = np.empty((nrows, k)) if want_dl else None
    rc = lib().kgpo_matmul(KERNEL_IDS[kt], n, d, x.ctypes.data, l, f, s, row0, nrows, k,
                           b.ctypes.data, None if ok is None else ok.ctypes.data,
                           None if od is None else od.ctypes.data, nthreads)
    if rc != 0:
        raise ValueError("kgpo_matmul: bad arguments")
    return ok, od


def panel(kt, x, y, l, which="k", scale=1.0, diag=0.0, nthreads=0):
    """scale * kappa(x, y) (which "k") or scale * dkappa/dl (which "l"), plus ``diag`` on the
    diagonal when diag != 0 (Khat = f^2 kappa + s I): the materialised panels of kernels.py:79-94
    / kmat.py:107-141, OpenMP over rows like the numba prange panels."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    out = np.empty((x.shape[0], y.shape[0]))
    rc = lib().kgpo_panel(KERNEL_IDS[kt], 0 if which == "k" else 1, x.shape[0], y.shape[0], x.shape[1],
                          x.ctypes.data, y.ctypes.data, l, scale, diag, int(diag != 0.0), out.ctypes.data,
                          nthreads)
    if rc != 0:
        raise ValueError("kgpo_panel: bad arguments")
    return out
