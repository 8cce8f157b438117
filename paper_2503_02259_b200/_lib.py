"""ctypes binding of libkgp.so (the C ABI declared in include/kgp.h).

The library is built in-tree (``paper_2503_02259_b200/libkgp.so``) by
``__graft_entry__.build()`` / ``make -C paper_2503_02259_b200/csrc``. There is
no fallback: if the library or a CUDA device is missing, every operator raises
``KernelGpError`` at first use.
"""

from __future__ import annotations

import ctypes
import os
import threading

from paper_2503_02259_b200.errors import (
    BreakdownError,
    KernelGpError,
    NumericalError,
    ResourceLimitError,
)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("KGP_LIB") or os.path.join(HERE, "libkgp.so")  # KGP_LIB: tuning builds only

OK, ERR_INVALID, ERR_RESOURCE, ERR_BREAKDOWN, ERR_NUMERICAL, ERR_CUDA, ERR_STATE = range(7)
KERNEL_IDS = {"gaussian": 0, "matern32": 1, "matern52": 2}
PRECISIONS = {"fp64": 0, "fast": 1, "tf32": 2, "bf16x3": 3}

_EXC = {
    ERR_INVALID: ValueError,
    ERR_RESOURCE: ResourceLimitError,
    ERR_BREAKDOWN: BreakdownError,
    ERR_NUMERICAL: NumericalError,
    ERR_CUDA: KernelGpError,
    ERR_STATE: KernelGpError,
}

_lib = None
_lock = threading.Lock()

c_i32, c_i64, c_dbl, c_vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p
_P = ctypes.POINTER

# (name, argtypes); every function returns int
_SIGNATURES = {
    "kgp_version": [],
    "kgp_device_count": [_P(ctypes.c_int)],
    "kgp_engine_create": [_P(c_vp), ctypes.c_int, ctypes.c_int, ctypes.c_int, c_i64, ctypes.c_int, c_vp,
                          ctypes.c_int, c_dbl, c_dbl, c_dbl, c_vp],
    "kgp_engine_set_params": [c_vp, c_dbl, c_dbl, c_dbl, c_vp],
    "kgp_engine_set_precision": [c_vp, ctypes.c_int],
    "kgp_engine_set_rows": [c_vp, c_i64, c_i64],
    "kgp_engine_destroy": [c_vp],
    "kgp_engine_matmul": [c_vp, c_i64, c_vp, c_i64, c_i64, c_vp, c_vp, c_vp, c_i64, c_i64, c_vp],
    "kgp_engine_cross_matmul": [c_vp, c_i64, c_vp, c_i64, c_vp, c_i64, c_i64, c_vp, c_i64, c_i64, c_vp],
    "kgp_eval_panel": [ctypes.c_int, ctypes.c_int, c_i64, c_i64, ctypes.c_int, c_vp, c_vp, c_dbl, c_vp, c_i64,
                       c_vp],
    "kgp_fps": [c_i64, ctypes.c_int, c_vp, c_i64, c_i64, c_vp, c_vp],
    "kgp_precond_create": [_P(c_vp), c_i64, c_i64, c_vp, c_dbl, c_vp],
    "kgp_precond_destroy": [c_vp],
    "kgp_precond_apply_inverse": [c_vp, c_i64, c_vp, c_i64, c_i64, c_vp, c_i64, c_i64, c_vp],
    "kgp_lowrank_apply": [c_vp, c_dbl, c_dbl, c_i64, c_vp, c_i64, c_i64, c_vp, c_i64, c_i64, c_vp],
    "kgp_lowrank_project": [c_vp, c_i64, c_vp, c_i64, c_i64, c_vp, c_vp],
    "kgp_lowrank_expand": [c_vp, c_dbl, c_dbl, c_i64, c_vp, c_i64, c_i64, c_vp, c_vp, c_i64, c_i64, c_vp],
    "kgp_pcg": [c_vp, c_vp, c_i64, c_vp, c_dbl, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp],
    "kgp_slq_logdet": [c_i64, c_i32, c_vp, c_vp, c_vp, c_vp, _P(c_dbl), c_vp],
    "kgp_nlml_grad": [c_vp, c_vp, c_vp, c_i64, c_vp, c_dbl, c_i32, c_dbl, c_i32, _P(c_dbl), _P(c_i32), c_vp],
    "kgp_engine_set_timing": [c_vp, ctypes.c_int],
    "kgp_engine_set_dense": [c_vp, ctypes.c_int],
    "kgp_knn_cross": [c_i64, c_vp, c_i64, c_vp, ctypes.c_int, ctypes.c_int, c_vp, c_vp],
    "kgp_local_variance": [ctypes.c_int, c_i64, ctypes.c_int, c_vp, c_vp, c_dbl, c_dbl, c_dbl, ctypes.c_int, c_vp,
                           c_vp, c_vp],
    "kgp_gpc_nlml_grad_pp": [c_vp, ctypes.c_int, c_vp, c_vp, c_vp, c_i64, c_vp, c_dbl, c_dbl, c_i32, c_dbl, c_i32,
                             _P(c_dbl), _P(c_i32), c_vp],
    "kgp_nlml_grad_pp": [c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_dbl, c_dbl, c_i32, c_dbl, c_i32, _P(c_dbl), _P(c_i32),
                         c_vp],
    "kgp_engine_matmul_host": [c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp],
    "kgp_knn_prev": [c_i64, ctypes.c_int, c_vp, ctypes.c_int, c_vp, c_vp],
    "kgp_afn_fsai": [ctypes.c_int, c_i64, ctypes.c_int, c_vp, c_dbl, c_dbl, c_dbl, c_vp, c_i64, c_vp, ctypes.c_int,
                     c_vp, c_vp, c_vp, c_vp],
    "kgp_engine_set_diag": [c_vp, ctypes.c_int, c_vp, c_i64, c_vp, c_vp],
    "kgp_pcg_grouped": [c_vp, c_vp, ctypes.c_int, c_i64, c_i64, c_vp, c_dbl, c_i32, c_dbl, c_i32, c_vp, c_vp, c_vp,
                        c_vp, c_vp, c_vp, c_vp],
    "kgp_gpc_nlml_grad": [c_vp, ctypes.c_int, c_vp, ctypes.c_int, c_vp, c_vp, c_i64, c_vp, c_dbl, c_i32, c_dbl, c_i32,
                          _P(c_dbl), _P(c_i32), c_vp],
    "kgp_afn_create": [_P(c_vp), c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, ctypes.c_int, c_vp, c_vp, c_i64, c_vp, c_vp,
                       c_vp, c_dbl, c_vp],
    "kgp_afn_sample": [c_vp, c_i64, c_vp, c_i64, c_i64, c_vp, c_vp],
    "kgp_precond_kind": [c_vp, _P(ctypes.c_int)],
    "kgp_engine_kernel_time": [c_vp, _P(c_dbl), _P(c_i64)],
    "kgp_peer_alloc": [c_i64, _P(c_vp), c_vp],
    "kgp_peer_open": [c_vp, _P(c_vp)],
    "kgp_peer_close": [c_vp],
    "kgp_peer_free": [c_vp],
    "kgp_engine_peer_buffer_bytes": [c_vp, c_i64, c_i64, _P(c_i64)],
    "kgp_engine_set_peers": [c_vp, ctypes.c_int, ctypes.c_int, c_vp, c_vp, c_i64],
    "kgp_engine_peer_publish": [c_vp, c_i64, c_vp, c_i64, c_i64, ctypes.c_uint64, c_vp],
    "kgp_engine_peer_matmul": [c_vp, c_i64, ctypes.c_uint64, c_vp, c_vp, c_vp, c_i64, c_i64, c_vp],
}

EXPORTED = tuple(_SIGNATURES) + ("kgp_last_error", "kgp_launch_count")


def load():
    """Load libkgp.so (no GPU needed to load; compute calls need one)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise KernelGpError(
                    f"libkgp.so not found at {LIB_PATH}; build it with "
                    "`python -c 'import __graft_entry__ as g; g.build()'` (there is no CPU fallback)")
            lib = ctypes.CDLL(LIB_PATH)
            for name, args in _SIGNATURES.items():
                fn = getattr(lib, name)
                fn.argtypes = args
                fn.restype = ctypes.c_int
            lib.kgp_last_error.argtypes = []
            lib.kgp_last_error.restype = ctypes.c_char_p
            lib.kgp_launch_count.argtypes = []
            lib.kgp_launch_count.restype = ctypes.c_int64
            _lib = lib
    return _lib


def launch_count() -> int:
    """Kernels libkgp has launched in this process (graph replays counted per kernel node)."""
    return int(load().kgp_launch_count())


def kernel_time(handle) -> tuple:
    """(total ms, launches) of the tensor-core operator kernel since the last read
    (requires kgp_engine_set_timing(handle, 1))."""
    ms, n = ctypes.c_double(), ctypes.c_int64()
    call("kgp_engine_kernel_time", handle, ctypes.byref(ms), ctypes.byref(n))
    return ms.value, n.value


def last_error() -> str:
    return load().kgp_last_error().decode(errors="replace")


def check(rc: int, what: str = "") -> None:
    """Raise the reference's exception type for a libkgp return code."""
    if rc == OK:
        return
    exc = _EXC.get(rc, KernelGpError)
    msg = last_error() or f"{what} failed with code {rc}"
    raise exc(msg)


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)
