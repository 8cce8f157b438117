"""KernelEngine on the B200: Khat = f^2 kappa(X, X; l) + s I behind a matmul interface.

Drop-in for kernelgp.kmat (kmat.py:30-189). The engine keeps X resident in HBM
(a private fp64 copy, as kmat.py:90 keeps a private host copy) and every
product -- matmul, grad_matmul, the fused three-output pass -- runs as one
launch of the fused sm_100a kernel in libkgp: the kernel matrix is generated
tile by tile on chip and never stored, whatever ``mode`` says. ``mode`` keeps
its reference meaning only for the dense helpers ``materialize`` /
``materialize_grad`` (the exact-path oracle), which are budgeted exactly as in
kmat.py:107-141.

Precision (``precision=`` or env ``KGP_PRECISION``):
  "fp64" -- fp64 tile and contraction; matches the reference to ~1e-15 (default).
  "fast" -- fp32 centred tile + 3xTF32 tcgen05 contraction (fp32-class operator).
  "tf32" -- fp32 centred tile + 1xTF32 tcgen05 contraction (throughput mode).

Inputs may be host array-likes (results come back as numpy, like the
reference) or CUDA tensors of shape (n, k) with any strides (results stay on
the device; a transposed (k, n) buffer passed as ``t.T`` is used in place).
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from enum import Enum
from math import isfinite

import numpy as np

from paper_2503_02259_b200 import _device
from paper_2503_02259_b200._lib import PRECISIONS, call, load
from paper_2503_02259_b200.errors import ResourceLimitError
from paper_2503_02259_b200.kernels import as_points, device_panel, kernel_id

DEFAULT_BLOCK_SIZE = 256
DEFAULT_DENSE_BUDGET = 20000


@dataclass(frozen=True)
class Hyperparams:
    """(l, f, s): length scale, signal scale, noise; each strictly positive and finite."""

    l: float
    f: float
    s: float

    def __post_init__(self):
        for key in ("l", "f", "s"):
            value = float(getattr(self, key))
            if not (value > 0.0 and isfinite(value)):
                raise ValueError(f"hyperparameter {key} must be positive and finite, got {value}")
            object.__setattr__(self, key, value)

    def as_array(self) -> np.ndarray:
        return np.array([self.l, self.f, self.s])


class Theta(Enum):
    """Derivative selector (kmat.py:49-54)."""

    L = "l"
    F = "f"
    S = "s"


class EngineMode(Enum):
    DENSE = "dense"
    ON_THE_FLY = "on_the_fly"


def theta_key(theta) -> str:
    """'l' | 'f' | 's' for this package's Theta, the reference's, or a string."""
    return str(getattr(theta, "value", theta))


def default_precision() -> str:
    return os.environ.get("KGP_PRECISION", "fp64").strip().lower() or "fp64"


def _as_matrix(b, n: int):
    """kmat.py:62-73: fp64, 1-D -> (n, 1), row count and finiteness checks."""
    b = np.asarray(b, dtype=np.float64)
    squeeze = b.ndim == 1
    if squeeze:
        b = b[:, None]
    if b.ndim != 2 or b.shape[0] != n:
        raise ValueError(f"B must have {n} rows, got shape {b.shape}")
    if b.shape[1] < 1:
        raise ValueError("B must have at least one column")
    if not np.isfinite(b).all():
        raise ValueError("B contains non-finite entries")
    return b, squeeze


class KernelEngine:
    """Device matmul handle for Khat and its hyperparameter derivatives."""

    def __init__(self, kt, x, params, mode=None, block_size: int = DEFAULT_BLOCK_SIZE,
                 dense_budget: int = DEFAULT_DENSE_BUDGET, backend=None, precision: str | None = None):
        self.kt = kt
        self.x = as_points(x, "X").copy()
        if not isinstance(params, Hyperparams):
            params = Hyperparams(float(params.l), float(params.f), float(params.s))
        self.params = params
        self.n = self.x.shape[0]
        if mode is None:
            mode = EngineMode.DENSE if self.n <= dense_budget else EngineMode.ON_THE_FLY
        self.mode = mode
        if block_size < 1:
            raise ValueError("block_size must be >= 1")
        self.block_size = int(block_size)
        self.dense_budget = int(dense_budget)
        self.backend = backend  # accepted for signature parity; the device kernel is the only backend
        self.precision = (precision or default_precision()).lower()
        if self.precision not in PRECISIONS:
            raise ValueError(f"precision must be one of {sorted(PRECISIONS)}, got {self.precision!r}")
        self._kid = kernel_id(kt)
        self._khat = None
        self._xd = None
        self._handle = ctypes.c_void_p()
        load()
        _device.device()
        call("kgp_engine_create", ctypes.byref(self._handle), _device.torch().cuda.current_device(), self._kid,
             PRECISIONS[self.precision], self.n, self.x.shape[1], self.x.ctypes.data, 0, self.params.l,
             self.params.f, self.params.s, _device.stream_ptr())
        self.x.setflags(write=False)
        if self.mode == EngineMode.DENSE and self.precision == "fp64":
            # the reference's DENSE mode (kmat.py:93-94): Khat materialised once on the device,
            # K.B by cuBLAS DGEMM; derivative products stay on the fused kernel
            call("kgp_engine_set_dense", self._handle, 1)

    def set_params(self, params) -> None:
        """Reset (l, f, s) in place, keeping X resident (a training loop's per-step update;
        the reference builds a new engine per step, train.py:198-204)."""
        if not isinstance(params, Hyperparams):
            params = Hyperparams(float(params.l), float(params.f), float(params.s))
        call("kgp_engine_set_params", self._handle, params.l, params.f, params.s, _device.stream_ptr())
        self.params = params
        self._khat = None

    # ----------------------------------------------------------------- lifetime
    @property
    def handle(self):
        return self._handle

    @property
    def d(self) -> int:
        return self.x.shape[1]

    def close(self):
        if self._handle:
            call("kgp_engine_destroy", self._handle)
            self._handle = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def x_device(self):
        if self._xd is None:
            self._xd = _device.to_device(self.x)
        return self._xd

    # ----------------------------------------------------------------- dense helpers (oracle path)
    def _check_budget(self, what="materializing"):
        if self.n > self.dense_budget:
            raise ResourceLimitError(
                f"{what} {self.n} points exceeds the dense budget of {self.dense_budget}; "
                "raise dense_budget or use ON_THE_FLY mode")

    def materialize_device(self):
        self._check_budget()
        p = self.params
        k = device_panel(self._kid, 0, self.x_device(), self.x_device(), p.l)
        k.mul_(p.f * p.f)
        k.diagonal().add_(p.s)
        return k

    def materialize(self) -> np.ndarray:
        """Dense Khat, cached and read-only (kmat.py:107-123)."""
        if self._khat is None:
            k = _device.to_host(self.materialize_device())
            k.setflags(write=False)
            self._khat = k
        return self._khat

    def materialize_grad_device(self, theta):
        self._check_budget()
        key = theta_key(theta)
        p = self.params
        torch = _device.torch()
        if key == "s":
            return torch.eye(self.n, dtype=torch.float64, device=_device.device())
        k = device_panel(self._kid, 1 if key == "l" else 0, self.x_device(), self.x_device(), p.l)
        k.mul_(p.f * p.f if key == "l" else 2.0 * p.f)
        return k

    def materialize_grad(self, theta) -> np.ndarray:
        """Dense dKhat/dtheta (kmat.py:125-141)."""
        return _device.to_host(self.materialize_grad_device(theta))

    # ----------------------------------------------------------------- fused products (device)
    def apply(self, b, want_k=True, want_dl=False, want_df=False, outs=None):
        """Device entry: b is an (n, k) CUDA tensor (any strides). Returns the requested
        outputs (K, dL, dF) as (n, k) CUDA tensors laid out like b."""
        torch = _device.torch()
        if b.dim() != 2 or b.shape[0] != self.n:
            raise ValueError(f"B must have {self.n} rows, got shape {tuple(b.shape)}")
        k = b.shape[1]
        col_major = b.stride(0) == 1 and k > 1

        def alloc():
            if col_major:
                return torch.empty((k, self.n), dtype=torch.float64, device=b.device).T
            return torch.empty((self.n, k), dtype=torch.float64, device=b.device)

        res = list(outs) if outs is not None else [alloc() if w else None for w in (want_k, want_dl, want_df)]
        o = next(t for t in res if t is not None)
        call("kgp_engine_matmul", self._handle, k, b.data_ptr(), b.stride(0), b.stride(1),
             *(0 if t is None else t.data_ptr() for t in res), o.stride(0), o.stride(1), _device.stream_ptr())
        return res

    def _host_apply(self, b, which):
        """numpy in, numpy out (the reference's calling convention) through the host-buffer
        entry kgp_engine_matmul_host: results land in pinned host memory, the device->host
        transfer pipelined behind the computation."""
        torch = _device.torch()
        b, squeeze = _as_matrix(b, self.n)
        b = np.ascontiguousarray(b, dtype=np.float64)
        k = b.shape[1]
        outs = [torch.empty((self.n, k), dtype=torch.float64, pin_memory=True) if w else None for w in which]
        call("kgp_engine_matmul_host", self._handle, k, b.ctypes.data,
             *(None if t is None else t.data_ptr() for t in outs), _device.stream_ptr())
        res = [None if t is None else t.numpy() for t in outs]
        return [None if o is None else (o[:, 0] if squeeze else o) for o in res]

    def matmul(self, b):
        """Khat @ B (kmat.py:145-152)."""
        if _device.is_tensor(b):
            return self.apply(b)[0]
        return self._host_apply(b, (True, False, False))[0]

    def grad_matmul(self, theta, b):
        """(dKhat/dtheta) @ B (kmat.py:154-163). dKhat/ds @ B is B itself, returned as a copy."""
        key = theta_key(theta)
        if _device.is_tensor(b):
            if key == "s":
                return b.clone()
            return self.apply(b, want_k=False, want_dl=key == "l", want_df=key == "f")[1 if key == "l" else 2]
        if key == "s":
            b, squeeze = _as_matrix(b, self.n)
            out = b.copy()
            return out[:, 0] if squeeze else out
        outs = self._host_apply(b, (False, key == "l", key == "f"))
        return outs[1] if key == "l" else outs[2]

    def matmul_with_grads(self, b):
        """(Khat B, dKhat/dl B, dKhat/df B) from ONE fused pass over the kernel matrix."""
        if _device.is_tensor(b):
            return tuple(self.apply(b, True, True, True))
        return tuple(self._host_apply(b, (True, True, True)))

    def cross_matmul(self, xs_dev, b):
        """f^2 kappa(Xs, X) @ B on the device, never materialising the cross kernel."""
        torch = _device.torch()
        m = xs_dev.shape[0]
        out = torch.empty((m, b.shape[1]), dtype=torch.float64, device=b.device)
        call("kgp_engine_cross_matmul", self._handle, m, xs_dev.data_ptr(), b.shape[1], b.data_ptr(),
             b.stride(0), b.stride(1), out.data_ptr(), out.stride(0), out.stride(1), _device.stream_ptr())
        return out


# SURVEY.md §8(b) names the drop-in ``CudaKernelEngine``: this package's engine IS that class
CudaKernelEngine = KernelEngine
