"""CG / batched PCG with Lanczos coefficient capture, and SLQ (kernelgp solver.py:35-265).

``pcg_solve(engine.matmul, pre.apply_inverse | None, Y, tol, max_iter)`` with a
KernelEngine of this package runs entirely on the device through ``kgp_pcg``:
one fused operator launch per iteration for all k columns, per-column
alpha/beta recurrences and freezing in device kernels, one status word read
back per iteration. Any other operator (a user callable) runs through the same
recurrences with the vector state on the device; the callable itself is
invoked on host arrays, exactly as the reference would invoke it.

``slq_logdet`` diagonalises the Lanczos tridiagonals on the device
(``kgp_slq_logdet``: implicit-shift QL tracking the first eigenvector row).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np

from paper_2503_02259_b200 import _device
from paper_2503_02259_b200._lib import call
from paper_2503_02259_b200.errors import BreakdownError, NumericalError

DEFAULT_TOL = 1e-6
DEFAULT_PROBE_TOL = 1e-2
DEFAULT_MAX_ITER = 500


@dataclass
class CgTrace:
    """Coefficients of one solve: equal-length alphas and betas (solver.py:40-47)."""

    alphas: np.ndarray
    betas: np.ndarray
    iterations: int
    final_rel_residual: float


@dataclass
class SolveReport:
    solution: np.ndarray
    traces: list = field(default_factory=list)
    converged: list = field(default_factory=list)

    @property
    def all_converged(self) -> bool:
        return all(self.converged)

    def iteration_counts(self) -> list:
        return [t.iterations for t in self.traces]


def _check_args(tol, max_iter):
    if tol < 0 or max_iter < 1:
        raise ValueError("need tol >= 0 and max_iter >= 1")


def _engine_of(apply_a):
    from paper_2503_02259_b200.kmat import KernelEngine

    owner = getattr(apply_a, "__self__", None)
    if isinstance(owner, KernelEngine) and getattr(apply_a, "__func__", None) is KernelEngine.matmul:
        return owner
    return None


def _precond_of(apply_minv):
    from paper_2503_02259_b200.precond import AFNPreconditioner, NystromPreconditioner

    owner = getattr(apply_minv, "__self__", None)
    for cls in (NystromPreconditioner, AFNPreconditioner):
        if isinstance(owner, cls) and getattr(apply_minv, "__func__", None) is cls.apply_inverse:
            return owner
    return None


# --------------------------------------------------------------------- device driver
def pcg_device(engine, precond, yt, tol: float, max_iter: int):
    """Batched PCG on the device. yt: (k, n) CUDA fp64 (column c contiguous).

    Returns (x (k, n), alphas (k, max_iter), betas, iters (k,), rel (k,), converged (k,))
    as CUDA tensors."""
    torch = _device.torch()
    k, n = yt.shape
    dev = yt.device
    x = torch.empty((k, n), dtype=torch.float64, device=dev)
    alphas = torch.empty((k, max_iter), dtype=torch.float64, device=dev)
    betas = torch.empty((k, max_iter), dtype=torch.float64, device=dev)
    iters = torch.empty(k, dtype=torch.int32, device=dev)
    rel = torch.empty(k, dtype=torch.float64, device=dev)
    conv = torch.empty(k, dtype=torch.int32, device=dev)
    call("kgp_pcg", engine.handle, None if precond is None else precond.handle, k, yt.data_ptr(), float(tol),
         int(max_iter), x.data_ptr(), alphas.data_ptr(), betas.data_ptr(), iters.data_ptr(), rel.data_ptr(),
         conv.data_ptr(), _device.stream_ptr())
    return x, alphas, betas, iters, rel, conv


def _report(x, alphas, betas, iters, rel, conv, squeeze, tol):
    a = _device.to_host(alphas)
    b = _device.to_host(betas)
    it = _device.to_host(iters)
    rl = _device.to_host(rel)
    traces = [CgTrace(a[c, :it[c]].copy(), b[c, :it[c]].copy(), int(it[c]), float(rl[c]))
              for c in range(len(it))]
    sol = _device.to_host(x)
    sol = sol[0] if squeeze else np.ascontiguousarray(sol.T)
    return SolveReport(sol, traces, [bool(r <= tol) for r in rl])


# --------------------------------------------------------------------- generic operators
def _generic_pcg(apply_a, apply_minv, y, tol, max_iter, x0=None):
    """Same recurrences as solver.py:143-192 for user callables; state on the device."""
    torch = _device.torch()
    y = np.asarray(y, dtype=np.float64)
    squeeze = y.ndim == 1
    y2 = y[:, None] if squeeze else y
    n, k = y2.shape
    dev = _device.device()
    yt = torch.from_numpy(np.ascontiguousarray(y2.T)).to(dev)
    xt = torch.zeros((k, n), dtype=torch.float64, device=dev)

    def op(fn, t):
        res = fn(_device.to_host(t).T[:, 0] if (squeeze and k == 1) else _device.to_host(t).T)
        res = np.asarray(res, dtype=np.float64)
        res = res[:, None] if res.ndim == 1 else res
        return torch.from_numpy(np.ascontiguousarray(res.T)).to(dev)

    if x0 is None:
        rt = yt.clone()
    else:
        xt = torch.from_numpy(np.ascontiguousarray(np.asarray(x0, np.float64).reshape(n, k).T)).to(dev)
        rt = yt - op(apply_a, xt)
    ynorm = torch.sqrt((yt * yt).sum(dim=1)).cpu().numpy()
    alphas = [[] for _ in range(k)]
    betas = [[] for _ in range(k)]
    if x0 is None:
        rel = np.where(ynorm > 0, 1.0, 0.0)
    else:
        rn = torch.sqrt((rt * rt).sum(dim=1)).cpu().numpy()
        rel = np.where(ynorm > 0, rn / np.where(ynorm > 0, ynorm, 1.0), 0.0)
    active = rel > tol
    if active.any():
        zt = rt if apply_minv is None else op(apply_minv, rt)
        pt = zt.clone()
        rz = (rt * zt).sum(dim=1).cpu().numpy()
        for _ in range(max_iter):
            apt = op(apply_a, pt)
            pap = (pt * apt).sum(dim=1).cpu().numpy()
            for j in np.flatnonzero(active):
                if not np.isfinite(pap[j]) or pap[j] <= 0.0:
                    raise BreakdownError(f"p^T A p = {pap[j]} in column {j}; operator is not SPD")
                a = rz[j] / pap[j]
                xt[j] += a * pt[j]
                rt[j] -= a * apt[j]
                alphas[j].append(float(a))
            zt = rt if apply_minv is None else op(apply_minv, rt)
            rr = (rt * rt).sum(dim=1).cpu().numpy()
            rzn_all = rr if apply_minv is None else (rt * zt).sum(dim=1).cpu().numpy()
            for j in np.flatnonzero(active):
                if not np.isfinite(rr[j]):
                    raise NumericalError("residual became non-finite during PCG")
                beta = rzn_all[j] / rz[j]
                betas[j].append(float(beta))
                rz[j] = rzn_all[j]
                rel[j] = math.sqrt(rr[j]) / ynorm[j]
                if rel[j] <= tol:
                    active[j] = False
                else:
                    pt[j] = zt[j] + beta * pt[j]
            if not active.any():
                break
    traces = [CgTrace(np.array(alphas[j]), np.array(betas[j]), len(alphas[j]), float(rel[j])) for j in range(k)]
    sol = _device.to_host(xt)
    sol = sol[0] if squeeze else np.ascontiguousarray(sol.T)
    return SolveReport(sol, traces, [bool(rel[j] <= tol) for j in range(k)])


# --------------------------------------------------------------------- public API
def pcg_solve(apply_a, apply_minv, y, tol: float = DEFAULT_TOL, max_iter: int = DEFAULT_MAX_ITER) -> SolveReport:
    """Preconditioned CG over a block of right-hand sides (solver.py:122-192)."""
    _check_args(tol, max_iter)
    engine = _engine_of(apply_a)
    pre = _precond_of(apply_minv) if apply_minv is not None else None
    if engine is not None and (apply_minv is None or pre is not None):
        torch = _device.torch()
        if _device.is_tensor(y):  # device in, device out: solution is a CUDA (n, k) view
            yt = (y[None, :] if y.dim() == 1 else y.T).to(torch.float64).contiguous()
            x, al, be, it, rel, conv = pcg_device(engine, pre, yt, tol, max_iter)
            rep = _report(x[:1], al, be, it, rel, conv, True, tol)
            rep.solution = x[0] if y.dim() == 1 else x.T
            return rep
        y = np.asarray(y, dtype=np.float64)
        squeeze = y.ndim == 1
        y2 = y[:, None] if squeeze else y
        if y2.ndim != 2 or y2.shape[0] != engine.n:
            raise ValueError(f"B must have {engine.n} rows, got shape {y.shape}")
        yt = torch.from_numpy(np.ascontiguousarray(y2.T)).to(_device.device())
        return _report(*pcg_device(engine, pre, yt, tol, max_iter), squeeze, tol)
    return _generic_pcg(apply_a, apply_minv, y, tol, max_iter)


def cg_solve(apply_a, y, x0=None, tol: float = DEFAULT_TOL, max_iter: int = DEFAULT_MAX_ITER):
    """Single-vector CG returning (x, CgTrace) (solver.py:68-119)."""
    _check_args(tol, max_iter)
    y = np.asarray(y, dtype=np.float64)
    if float(np.sqrt(y @ y)) == 0.0:
        return np.zeros_like(y), CgTrace(np.empty(0), np.empty(0), 0, 0.0)
    if x0 is None and _engine_of(apply_a) is not None:
        rep = pcg_solve(apply_a, None, y, tol, max_iter)
    else:
        rep = _generic_pcg(apply_a, None, y, tol, max_iter, x0=x0)
    return rep.solution, rep.traces[0]


def _tridiag_bands(trace: CgTrace):
    """solver.py:220-235, including its validation messages."""
    a = np.asarray(trace.alphas, dtype=np.float64)
    b = np.asarray(trace.betas, dtype=np.float64)
    m = len(a)
    if m < 1:
        raise ValueError("trace holds no iterations; T is undefined")
    if len(b) < m - 1:
        raise ValueError(f"need at least {m - 1} betas for {m} alphas, got {len(b)}")
    if np.any(a <= 0):
        raise ValueError("trace has non-positive alphas; solve was not SPD")
    if np.any(b[: m - 1] < 0):
        raise ValueError("trace has negative betas")
    diag = 1.0 / a
    diag[1:] += b[: m - 1] / a[: m - 1]
    off = np.sqrt(b[: m - 1]) / a[: m - 1]
    return diag, off


def build_tridiag(trace: CgTrace) -> np.ndarray:
    """Dense Lanczos tridiagonal T_m from CG coefficients (solver.py:202-217)."""
    diag, off = _tridiag_bands(trace)
    return np.diag(diag) + np.diag(off, 1) + np.diag(off, -1)


def slq_logdet_device(alphas, betas, iters, norms_sq) -> float:
    """SLQ from device-resident coefficient arrays (k, max_iter) -- no host round trip."""
    out = ctypes.c_double()
    k, max_iter = alphas.shape
    call("kgp_slq_logdet", k, max_iter, alphas.data_ptr(), betas.data_ptr(), iters.data_ptr(),
         norms_sq.data_ptr(), ctypes.byref(out), _device.stream_ptr())
    return float(out.value)


def slq_logdet(traces, probe_norms_sq) -> float:
    """Stochastic Lanczos quadrature estimate of log|A| (solver.py:238-265)."""
    norms_sq = np.asarray(probe_norms_sq, dtype=np.float64)
    if len(traces) != len(norms_sq):
        raise ValueError(f"got {len(traces)} traces but {len(norms_sq)} probe norms")
    if len(traces) == 0:
        raise ValueError("need at least one probe trace")
    for t in traces:
        if t.iterations:
            _tridiag_bands(t)  # same validation as the reference, before the device solve
    torch = _device.torch()
    k = len(traces)
    width = max(1, max(t.iterations for t in traces))
    a = np.zeros((k, width))
    b = np.zeros((k, width))
    it = np.zeros(k, dtype=np.int32)
    for j, t in enumerate(traces):
        m = t.iterations
        it[j] = m
        a[j, :m] = np.asarray(t.alphas, dtype=np.float64)[:m]
        nb = min(m, len(t.betas))
        b[j, :nb] = np.asarray(t.betas, dtype=np.float64)[:nb]
    dev = _device.device()
    return slq_logdet_device(torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev),
                             torch.from_numpy(it).to(dev), torch.from_numpy(norms_sq).to(dev))
