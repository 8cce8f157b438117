"""Landmark (Nystrom) preconditioner on the device (kernelgp precond.py:31-126).

Build (precond.py:95-126): farthest-point landmarks (``kgp_fps``), the ridged
landmark block K_mm and the cross block K_mn from the device panel kernel, then
the two Cholesky factorisations and triangular solves through cuSOLVER/cuBLAS
(torch.linalg on CUDA tensors):

    K_mm + ridge I = L L^T,   V^T = L^-1 K_mn,   C = I/f^2 + V^T V / s = L_C L_C^T,
    W^T = L_C^-1 V^T.

Apply (precond.py:74-92), every PCG iteration, in libkgp:
    M^-1 B = B/s - W (W^T B)/s^2          M B = s B + f^2 V (V^T B)
which equals the reference's cho_solve form in exact arithmetic.
"""

from __future__ import annotations

import ctypes
import math

import numpy as np

from paper_2503_02259_b200 import _device
from paper_2503_02259_b200._lib import call
from paper_2503_02259_b200.errors import BreakdownError
from paper_2503_02259_b200.kernels import as_points, device_panel

RIDGE_SCALE = 1e-10


def default_rank(n: int) -> int:
    """precond.py:34-36."""
    return min(int(math.ceil(math.sqrt(n))) * 4, 500, n)


def fps_device(xd, m: int, seed_index: int = 0):
    """Farthest-point sampling on a device point tensor; returns an int64 CUDA tensor."""
    torch = _device.torch()
    n, d = xd.shape
    idx = torch.empty(m, dtype=torch.int64, device=xd.device)
    call("kgp_fps", n, d, xd.data_ptr(), m, int(seed_index), idx.data_ptr(), _device.stream_ptr())
    return idx


def fps_select(x, m: int, seed_index: int = 0) -> np.ndarray:
    """Greedy farthest-point landmarks, lowest index on ties (precond.py:39-59)."""
    x = as_points(x, "X")
    n = x.shape[0]
    if not 1 <= m <= n:
        raise ValueError(f"need 1 <= m <= n, got m={m}, n={n}")
    if not 0 <= seed_index < n:
        raise ValueError(f"seed_index {seed_index} out of range for n={n}")
    return _device.to_host(fps_device(_device.to_device(x), m, seed_index)).astype(np.intp)


class _LowRank:
    """Owns one libkgp low-rank handle (U^T on the device)."""

    def __init__(self, ut, s):
        ut = ut.contiguous()  # torch.linalg returns column-major factors; libkgp wants (m, n) row-major
        self.h = ctypes.c_void_p()
        call("kgp_precond_create", ctypes.byref(self.h), ut.shape[1], ut.shape[0], ut.data_ptr(), float(s),
             _device.stream_ptr())

    def close(self):
        if self.h:
            call("kgp_precond_destroy", self.h)
            self.h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class NystromPreconditioner:
    """M = s I + f^2 V V^T with Woodbury inverse, factors resident in HBM."""

    def __init__(self, landmark_indices, shift, inv, fwd, f2, n):
        self.landmark_indices = landmark_indices
        self.shift = float(shift)
        self._inv = inv
        self._fwd = fwd
        self._f2 = float(f2)
        self.n = int(n)

    @property
    def rank(self) -> int:
        return len(self.landmark_indices)

    @property
    def handle(self):
        return self._inv.h

    def _run(self, which, b, beta, alpha):
        torch = _device.torch()
        host = not _device.is_tensor(b)
        if host:
            b = np.asarray(b, dtype=np.float64)
        squeeze = b.ndim == 1
        bd = _device.to_device(b) if host else b
        if squeeze:
            bd = bd[:, None]
        out = torch.empty((bd.shape[0], bd.shape[1]), dtype=torch.float64, device=bd.device)
        call("kgp_lowrank_apply", which.h, beta, alpha, bd.shape[1], bd.data_ptr(), bd.stride(0), bd.stride(1),
             out.data_ptr(), out.stride(0), out.stride(1), _device.stream_ptr())
        if squeeze:
            out = out[:, 0]
        return _device.to_host(out) if host else out

    def apply_inverse(self, b):
        """inv(M) @ B via Woodbury (precond.py:74-83)."""
        s = self.shift
        return self._run(self._inv, b, 1.0 / s, -1.0 / (s * s))

    def apply(self, b):
        """M @ B (precond.py:85-92)."""
        return self._run(self._fwd, b, self.shift, self._f2)


def build(engine, m: int | None = None) -> NystromPreconditioner:
    """Landmark preconditioner for an engine's Khat (precond.py:95-126)."""
    torch = _device.torch()
    n = engine.n
    if m is None:
        m = default_rank(n)
    if not 1 <= m <= n:
        raise ValueError(f"need 1 <= m <= n, got m={m}, n={n}")
    p = engine.params
    xd = engine.x_device()
    idx = fps_device(xd, m, 0)
    xm = xd.index_select(0, idx)
    kid = engine._kid
    kmm = device_panel(kid, 0, xm, xm, p.l)
    ridge = RIDGE_SCALE * float(torch.trace(kmm)) / m
    kmm.diagonal().add_(ridge)
    f2 = p.f * p.f

    def fail():
        return BreakdownError(f"landmark factorization failed even after ridge {ridge:.3e}; "
                              "increase the noise term s or reduce the rank m")

    low, info = torch.linalg.cholesky_ex(kmm)
    if int(info) != 0:
        raise fail()
    vt = torch.linalg.solve_triangular(low, device_panel(kid, 0, xm, xd, p.l), upper=False)
    cap = (vt @ vt.T) / p.s
    cap.diagonal().add_(1.0 / f2)
    lc, info = torch.linalg.cholesky_ex(cap)
    if int(info) != 0 or not bool(torch.isfinite(vt).all()):
        raise fail()
    wt = torch.linalg.solve_triangular(lc, vt, upper=False)
    inv = _LowRank(wt, p.s)
    del wt
    fwd = _LowRank(vt, p.s)
    return NystromPreconditioner(_device.to_host(idx).astype(np.intp), p.s, inv, fwd, f2, n)
