"""Kernel families, point validation and materialised panels (kernelgp kernels.py:29-94).

Entries are evaluated on the device by ``kgp_eval_panel`` (fp64, direct
differences in the numba panel order, _panels_numba.py:23-131). The functions
return host numpy arrays like the reference; ``device_panel`` keeps the result
on the GPU for callers that stay there (preconditioner build, exact path).
"""

from __future__ import annotations

from enum import Enum

import numpy as np

from paper_2503_02259_b200 import _device
from paper_2503_02259_b200._lib import KERNEL_IDS, call


class KernelType(Enum):
    """Same values as the reference enum, so ``KernelType(ref_kt.value)`` round-trips."""

    GAUSSIAN = "gaussian"
    MATERN32 = "matern32"
    MATERN52 = "matern52"

    @classmethod
    def from_name(cls, name: str) -> "KernelType":
        key = name.strip().lower()
        for member in cls:
            if member.value == key:
                return member
        raise ValueError(f"unknown kernel {name!r}; expected one of: "
                         + ", ".join(m.value for m in cls))


def kernel_id(kt) -> int:
    """Accepts this package's KernelType, the reference's, or a plain name."""
    value = getattr(kt, "value", kt)
    try:
        return KERNEL_IDS[str(value)]
    except KeyError:
        raise ValueError(f"unknown kernel {value!r}") from None


def as_points(x, name: str = "points") -> np.ndarray:
    """(n, d) float64 C-contiguous copy-or-view with the reference's checks (kernels.py:43-52)."""
    arr = np.ascontiguousarray(x, dtype=np.float64)
    if arr.ndim == 1:
        arr = arr[:, None]
    if arr.ndim != 2 or arr.shape[0] < 1 or arr.shape[1] < 1:
        raise ValueError(f"{name} must be a nonempty 2-d array, got shape {np.shape(x)}")
    if not np.isfinite(arr).all():
        raise ValueError(f"{name} contains non-finite entries")
    return arr


def _pair(x, y):
    x = as_points(x, "X")
    y = as_points(y, "Y")
    if x.shape[1] != y.shape[1]:
        raise ValueError("point sets disagree on dimension: "
                         f"X has d={x.shape[1]}, Y has d={y.shape[1]}")
    return x, y


def _lengthscale(l) -> float:
    l = float(l)
    if not (l > 0.0) or not np.isfinite(l):
        raise ValueError(f"length scale must be positive and finite, got {l}")
    return l


def device_panel(kid: int, mode: int, xd, yd, l: float):
    """(nx, ny) panel on the device from device point tensors (mode 0 kappa, 1 dkappa/dl, 2 r^2)."""
    torch = _device.torch()
    out = torch.empty((xd.shape[0], yd.shape[0]), dtype=torch.float64, device=xd.device)
    call("kgp_eval_panel", kid, mode, xd.shape[0], yd.shape[0], xd.shape[1], xd.data_ptr(), yd.data_ptr(),
         float(l), out.data_ptr(), out.shape[1], _device.stream_ptr())
    return out


def _host_panel(kid, mode, x, y, l):
    xd, yd = _device.to_device(x), _device.to_device(y)
    return _device.to_host(device_panel(kid, mode, xd, yd, l))


def pairwise_sq_dist(x, y) -> np.ndarray:
    """Squared Euclidean distances (kernels.py:72-76)."""
    x, y = _pair(x, y)
    return _host_panel(0, 2, x, y, 1.0)


def eval_kernel(kt, x, y, l: float) -> np.ndarray:
    """Entry (i, j) = kappa(X_i, Y_j; l) (kernels.py:79-85)."""
    x, y = _pair(x, y)
    return _host_panel(kernel_id(kt), 0, x, y, _lengthscale(l))


def eval_kernel_grad_l(kt, x, y, l: float) -> np.ndarray:
    """Entrywise d kappa / d l (kernels.py:88-94)."""
    x, y = _pair(x, y)
    return _host_panel(kernel_id(kt), 1, x, y, _lengthscale(l))
