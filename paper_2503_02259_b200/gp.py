"""GP negative log marginal likelihood, gradient and prediction on the device (kernelgp gp.py).

    L = 1/2 (y^T Khat^-1 y + log|Khat| + n log 2 pi)
    dL/dtheta = 1/2 (-w^T dKhat/dtheta w + tr(Khat^-1 dKhat/dtheta)),  w = Khat^-1 y

``nlml_grad_iterative`` with this package's KernelEngine is ONE call into
libkgp (``kgp_nlml_grad``): preconditioned w-solve, unpreconditioned probe
solves whose CG coefficients feed SLQ, and a single fused derivative pass over
[w, Z] for dKhat/dl and dKhat/df together (the reference makes one streamed
pass per theta, gp.py:173-174). Probes are drawn on the host with numpy's
PCG64 exactly as the reference (gp.py:81-85), so both see the same vectors.

The exact route (dense Cholesky, gp.py:107-130) runs on the device through
cuSOLVER (torch.linalg) and is the oracle the iterative route is checked against.
"""

from __future__ import annotations

import ctypes
import math
import warnings
from dataclasses import dataclass

import numpy as np

from paper_2503_02259_b200 import _device
from paper_2503_02259_b200 import precond as precond_mod
from paper_2503_02259_b200 import solver
from paper_2503_02259_b200._lib import call
from paper_2503_02259_b200.errors import NumericalError
from paper_2503_02259_b200.kernels import as_points, device_panel, kernel_id
from paper_2503_02259_b200.kmat import (
    DEFAULT_BLOCK_SIZE,
    DEFAULT_DENSE_BUDGET,
    EngineMode,
    KernelEngine,
    Theta,
)

LOG_2PI = math.log(2.0 * math.pi)
DEFAULT_NUM_PROBES = 16


@dataclass
class LossGrad:
    loss: float
    grad_l: float
    grad_f: float
    grad_s: float
    converged: bool = True  # an inner solve stopped at max_iter when False

    def grads(self) -> np.ndarray:
        return np.array([self.grad_l, self.grad_f, self.grad_s])


@dataclass
class Prediction:
    mean: np.ndarray
    stddev: np.ndarray

    # Listing 1's field names (pred.prediction_mean, pred.prediction_stddev)
    @property
    def prediction_mean(self) -> np.ndarray:
        return self.mean

    @property
    def prediction_stddev(self) -> np.ndarray:
        return self.stddev


class ProbeSet:
    """Standard-normal probe block Z (n, k_z), reproducible from its seed (gp.py:65-85)."""

    def __init__(self, vectors, rng_seed=None):
        z = np.asarray(vectors, dtype=np.float64)
        if z.ndim != 2 or z.shape[1] < 1:
            raise ValueError("probe vectors must form an n x k_z matrix")
        self.vectors = z
        self.rng_seed = rng_seed
        self.norms_sq = np.einsum("ij,ij->j", z, z)

    @property
    def k_z(self) -> int:
        return self.vectors.shape[1]

    @classmethod
    def generate(cls, n: int, k_z: int, rng_seed) -> "ProbeSet":
        if k_z < 1:
            raise ValueError("need at least one probe")
        return cls(np.random.default_rng(rng_seed).standard_normal((n, k_z)), rng_seed)


def _check_y(y, n: int) -> np.ndarray:
    y = np.asarray(y, dtype=np.float64).reshape(-1)
    if y.shape[0] != n:
        raise ValueError(f"y must have length {n}, got {y.shape[0]}")
    if not np.isfinite(y).all():
        raise ValueError("y contains non-finite entries")
    return y


def _chol(a):
    torch = _device.torch()
    low, info = torch.linalg.cholesky_ex(a)
    if int(info) != 0:
        raise NumericalError("Cholesky factorization failed; Khat is not SPD, which should be "
                             "impossible for s > 0 and indicates a kernel bug")
    return low


def _dense(engine, theta=None):
    if isinstance(engine, KernelEngine):
        return engine.materialize_device() if theta is None else engine.materialize_grad_device(theta)
    m = engine.materialize() if theta is None else engine.materialize_grad(theta)
    return _device.to_device(np.asarray(m, dtype=np.float64))


def _exact_parts(engine, y):
    torch = _device.torch()
    low = _chol(_dense(engine))
    yd = _device.to_device(y)
    w = torch.cholesky_solve(yd[:, None], low)[:, 0]
    logdet = 2.0 * float(torch.log(torch.diagonal(low)).sum())
    loss = 0.5 * (float(yd @ w) + logdet + len(y) * LOG_2PI)
    return low, w, loss


def nlml_exact(engine, y) -> float:
    """Dense-path loss from one Cholesky factorisation (gp.py:107-113)."""
    y = _check_y(y, engine.n)
    return _exact_parts(engine, y)[2]


def grad_exact(engine, y) -> LossGrad:
    """Dense-path loss and gradient (gp.py:116-130)."""
    torch = _device.torch()
    y = _check_y(y, engine.n)
    low, w, loss = _exact_parts(engine, y)
    g = {}
    for theta in (Theta.L, Theta.F, Theta.S):
        dk = _dense(engine, theta)
        quad = -float(w @ (dk @ w))
        tr = float(torch.diagonal(torch.cholesky_solve(dk, low)).sum())
        g[theta] = 0.5 * (quad + tr)
    return LossGrad(loss, g[Theta.L], g[Theta.F], g[Theta.S])


def _generic_iterative(engine, y, preconditioner, probes, tol, max_iter, probe_tol):
    """Duck-typed operators (e.g. the reference's IdentityOperator test double)."""
    minv = preconditioner.apply_inverse if preconditioner is not None else None
    wr = solver.pcg_solve(engine.matmul, minv, y, tol=tol, max_iter=max_iter)
    w = wr.solution
    ur = solver.pcg_solve(engine.matmul, None, probes.vectors, tol=probe_tol, max_iter=max_iter)
    logdet = solver.slq_logdet(ur.traces, probes.norms_sq)
    loss = 0.5 * (float(y @ w) + logdet + engine.n * LOG_2PI)
    u = ur.solution
    v = np.column_stack([w, probes.vectors])
    g = []
    for theta in (Theta.L, Theta.F, Theta.S):
        dv = np.asarray(engine.grad_matmul(theta, v), dtype=np.float64)
        g.append(0.5 * (-float(w @ dv[:, 0]) + float(np.einsum("ij,ij->", u, dv[:, 1:])) / probes.k_z))
    return LossGrad(loss, g[0], g[1], g[2], converged=wr.all_converged and ur.all_converged)


PP_TAIL_SEED = precond_mod.PP_TAIL_SEED


def nlml_grad_iterative(engine, y, preconditioner, probes: ProbeSet, tol: float = solver.DEFAULT_TOL,
                        max_iter: int = solver.DEFAULT_MAX_ITER, probe_tol: float | None = None, *,
                        probe_max_iter: int | None = None, preconditioned_probes=False) -> LossGrad:
    """Matrix-free loss and gradient from one probe set (gp.py:133-179).

    Keyword-only extensions: ``probe_max_iter`` caps the probe CG / Lanczos length
    separately from the w-solve (None keeps the reference's single ``max_iter``).
    ``preconditioned_probes`` = True (M = ``preconditioner``) or a preconditioner M (then
    ``preconditioner`` serves the w-solve only) switches to the preconditioned estimator:
    probes z ~ N(0, M) -- Nystrom: z = sqrt(s) w1 + f V w2 with w1 the probe set's vectors
    and w2 drawn from default_rng([seed..., PP_TAIL_SEED]); AFN: z = L diag(L11, G^-1) w with
    w the probe set's vectors (kgp_afn_sample) -- the probe solves are preconditioned (a
    fraction of the reference's unpreconditioned CG iterations),
    log|Khat| = log|M| + SLQ of M^-1/2 Khat M^-1/2, and the trace terms use
    E[(M^-1 z)^T dK Khat^-1 z]. Unbiased for the same loss and gradient; not the reference's
    same-probe numbers."""
    n = engine.n
    y = _check_y(y, n)
    if probes.vectors.shape[0] != n:
        raise ValueError(f"probes have {probes.vectors.shape[0]} rows, need {n}")
    if probe_tol is None:
        probe_tol = tol
    if getattr(engine, "precision", None) == "tf32":
        warnings.warn("nlml_grad_iterative on a single-pass tf32 operator: loss/gradient errors reach "
                      "1e-1 and more (DESIGN.md §4); use precision='fast' (3xTF32) or 'fp64'", stacklevel=2)
    if preconditioned_probes is not False and preconditioned_probes is not None:
        pm = preconditioner if preconditioned_probes is True else preconditioned_probes
        return _nlml_grad_pp(engine, y, preconditioner, pm, probes, tol, max_iter, probe_tol, probe_max_iter)
    ours = isinstance(engine, KernelEngine)
    pre_ok = preconditioner is None or isinstance(
        preconditioner, (precond_mod.NystromPreconditioner, precond_mod.AFNPreconditioner))
    if not (ours and pre_ok):
        if probe_max_iter is not None:
            raise ValueError("probe_max_iter needs this package's KernelEngine")
        return _generic_iterative(engine, y, preconditioner, probes, tol, max_iter, probe_tol)
    torch = _device.torch()
    dev = _device.device()
    yd = torch.from_numpy(y).to(dev)
    zt = torch.from_numpy(np.ascontiguousarray(probes.vectors.T)).to(dev)
    out = (ctypes.c_double * 4)()
    conv = ctypes.c_int32()
    call("kgp_nlml_grad", engine.handle, None if preconditioner is None else preconditioner.handle,
         yd.data_ptr(), probes.k_z, zt.data_ptr(), float(tol), int(max_iter), float(probe_tol),
         int(probe_max_iter or 0), out,
         ctypes.byref(conv), _device.stream_ptr())
    return LossGrad(out[0], out[1], out[2], out[3], converged=bool(conv.value))


def _nlml_grad_pp(engine, y, pre_w, pre, probes, tol, max_iter, probe_tol, probe_max_iter) -> LossGrad:
    if not isinstance(engine, KernelEngine) or getattr(pre, "logdet", None) is None:
        raise ValueError("preconditioned_probes needs this package's KernelEngine and a Nystrom/AFN preconditioner")
    torch = _device.torch()
    zt = pre.draw_probes(probes)                             # (k_z, n) on the device, z ~ N(0, M)
    yd = torch.from_numpy(y).to(zt.device)
    out = (ctypes.c_double * 4)()
    conv = ctypes.c_int32()
    call("kgp_nlml_grad_pp", engine.handle, None if pre_w is None or pre_w is pre else pre_w.handle, pre.handle,
         yd.data_ptr(), probes.k_z, zt.data_ptr(), float(pre.logdet),
         float(tol), int(max_iter), float(probe_tol), int(probe_max_iter or 0), out, ctypes.byref(conv),
         _device.stream_ptr())
    return LossGrad(out[0], out[1], out[2], out[3], converged=bool(conv.value))


def predict(kt, x, y, xstar, params, mode: str = "exact", tol: float = solver.DEFAULT_TOL,
            max_iter: int = solver.DEFAULT_MAX_ITER, precond_rank: int | None = None,
            block_size: int = DEFAULT_BLOCK_SIZE, dense_budget: int = DEFAULT_DENSE_BUDGET,
            precision: str | None = None) -> Prediction:
    """Posterior mean and latent-function stddev at the test points (gp.py:182-244)."""
    if mode not in ("exact", "iterative"):
        raise ValueError(f"mode must be 'exact' or 'iterative', got {mode!r}")
    torch = _device.torch()
    x = as_points(x, "X")
    n = x.shape[0]
    y = _check_y(y, n)
    xstar = np.asarray(xstar, dtype=np.float64)
    if xstar.ndim == 1:
        xstar = xstar[:, None]
    if xstar.size == 0:
        return Prediction(mean=np.empty(0), stddev=np.empty(0))
    xstar = as_points(xstar, "Xstar")
    if xstar.shape[1] != x.shape[1]:
        raise ValueError(f"train/test dimension mismatch: d={x.shape[1]} vs d={xstar.shape[1]}")
    f2 = params.f * params.f
    xd, xsd = _device.to_device(x), _device.to_device(xstar)
    cross = device_panel(kernel_id(kt), 0, xd, xsd, params.l).mul_(f2)  # n x m_test (gp.py:224)
    yd = _device.to_device(y)
    if mode == "exact":
        engine = KernelEngine(kt, x, params, mode=EngineMode.DENSE, dense_budget=dense_budget,
                              precision="fp64")
        low = _chol(engine.materialize_device())
        w = torch.cholesky_solve(yd[:, None], low)[:, 0]
        sol = torch.cholesky_solve(cross, low)
    else:
        engine = KernelEngine(kt, x, params, block_size=block_size, dense_budget=dense_budget,
                              precision=precision)
        pre = precond_mod.build(engine, precond_rank)
        rhs_t = torch.cat([yd[None, :], cross.T], dim=0).contiguous()  # (1 + m, n)
        parts = []
        for c0 in range(0, rhs_t.shape[0], 1024):  # columns are independent in batched PCG
            parts.append(solver.pcg_device(engine, pre, rhs_t[c0:c0 + 1024].contiguous(), tol, max_iter)[0])
        solt = torch.cat(parts, dim=0)
        w = solt[0]
        sol = solt[1:].T
    mean = cross.T @ w
    var = f2 - (cross * sol).sum(dim=0)
    stddev = torch.sqrt(torch.clamp(var, min=0.0))
    return Prediction(mean=_device.to_host(mean), stddev=_device.to_host(stddev))


def _build_pre(engine, kind: str, rank):
    if kind == "afn":
        return precond_mod.build_afn(engine, rank)
    if kind == "adaptive":
        return precond_mod.build_adaptive(engine, rank)
    if kind != "nystrom":
        raise ValueError(f"preconditioner must be 'nystrom', 'afn' or 'adaptive', got {kind!r}")
    return precond_mod.build(engine, rank)


def predict_hutchinson(kt, x, y, xstar, params, tol: float = solver.DEFAULT_TOL,
                       max_iter: int = solver.DEFAULT_MAX_ITER, precond_rank: int | None = None,
                       num_probes: int = 64, seed=0, precision: str | None = None,
                       preconditioner: str = "nystrom") -> Prediction:
    """Large-scale prediction (BASELINE configs[4]): no n x m_test cross kernel is formed.

    mean = f^2 kappa(X*, X) w with w = Khat^-1 y, one fused cross product (gp.py:241);
    variance by Hutchinson's diagonal estimator instead of one solve per test point
    (gp.py:242 needs all m_test columns):
        diag(C^T Khat^-1 C) ~= (1/S) sum_s z_s o (C^T Khat^-1 C z_s),  C = f^2 kappa(X, X*),
    with Rademacher z_s (m_test,), so each probe costs two fused cross products and one
    column of a batched PCG solve. The estimate is unbiased; its spread shrinks as
    1/sqrt(S). The reference has no estimator: this path is checked against
    the exact variance statistically (tests/test_gpu_parity.py)."""
    torch = _device.torch()
    x = as_points(x, "X")
    n = x.shape[0]
    y = _check_y(y, n)
    xstar = as_points(np.asarray(xstar, dtype=np.float64).reshape(-1, x.shape[1]), "Xstar")
    m = xstar.shape[0]
    f2 = params.f * params.f
    engine = KernelEngine(kt, x, params, precision=precision)          # columns: training points
    star = KernelEngine(kt, xstar, params, precision=precision)        # columns: test points
    pre = _build_pre(engine, preconditioner, precond_rank)
    xd, xsd = engine.x_device(), star.x_device()
    rng = np.random.default_rng(seed)
    zs = torch.from_numpy(rng.choice([-1.0, 1.0], size=(m, num_probes))).to(xd.device)
    u = star.cross_matmul(xd, zs)                                       # C z      (n, S)
    rhs = torch.cat([_device.to_device(y)[None, :], u.T], dim=0).contiguous()  # (1 + S, n)
    parts = [solver.pcg_device(engine, pre, rhs[c0:c0 + 1024].contiguous(), tol, max_iter)[0]
             for c0 in range(0, rhs.shape[0], 1024)]
    sol = torch.cat(parts, dim=0)                                       # [w; Khat^-1 C z]
    az = engine.cross_matmul(xsd, sol.T.contiguous())                   # C^T [w, Khat^-1 C z]
    mean = az[:, 0]
    diag = (zs * az[:, 1:]).mean(dim=1)
    stddev = torch.sqrt(torch.clamp(f2 - diag, min=0.0))
    return Prediction(mean=_device.to_host(mean), stddev=_device.to_host(stddev))


def predict_local(kt, x, y, xstar, params, tol: float = solver.DEFAULT_TOL, max_iter: int = solver.DEFAULT_MAX_ITER,
                  precond_rank: int | None = None, k_nn: int = 64, precision: str | None = None,
                  preconditioner: str = "afn") -> Prediction:
    """Large-scale prediction with a LOCAL variance (extension; SURVEY §8(f)2 leaves large-m
    variance open): mean = f^2 kappa(X*, X) w (w = Khat^-1 y by device PCG, one fused cross
    product), variance = f^2 - c^T Khat_NN^-1 c over the k_nn nearest training points of each
    test point (kgp_knn_cross + kgp_local_variance). Equal to the exact variance when k_nn
    covers the training set; otherwise an approximation that is good when the kernel's
    correlation length is short against the data's extent (measured in DESIGN.md)."""
    torch = _device.torch()
    x = as_points(x, "X")
    n = x.shape[0]
    y = _check_y(y, n)
    xstar = as_points(np.asarray(xstar, dtype=np.float64).reshape(-1, x.shape[1]), "Xstar")
    m = xstar.shape[0]
    k_nn = int(min(k_nn, n))
    engine = KernelEngine(kt, x, params, precision=precision)
    pre = _build_pre(engine, preconditioner, precond_rank)
    xd = engine.x_device()
    xsd = _device.to_device(xstar)
    w = solver.pcg_device(engine, pre, _device.to_device(y)[None, :].contiguous(), tol, max_iter)[0]
    mean = engine.cross_matmul(xsd, w.T.contiguous())[:, 0]
    nbr = torch.empty((m, k_nn), dtype=torch.int64, device=xd.device)
    call("kgp_knn_cross", m, xsd.data_ptr(), n, xd.data_ptr(), x.shape[1], k_nn, nbr.data_ptr(), _device.stream_ptr())
    var = torch.empty(m, dtype=torch.float64, device=xd.device)
    call("kgp_local_variance", kernel_id(kt), m, x.shape[1], xsd.data_ptr(), xd.data_ptr(), float(params.l),
         float(params.f), float(params.s), k_nn, nbr.data_ptr(), var.data_ptr(), _device.stream_ptr())
    return Prediction(mean=_device.to_host(mean), stddev=_device.to_host(torch.sqrt(var)))
