"""GP classification on the device: the GPC problem setup, loss+gradient, training and
prediction the north star asks for ("GPR/GPC problem setup").

The reference has no GPC (SPEC.md:382 lists it as a non-goal; HiGP's paper names a
``gpcproblemmodule`` without formulas), so this module restates a published method
that runs entirely on the GPR hot path: Dirichlet-based GP classification (Milios,
Camoriano, Michiardi, Rosasco, NeurIPS 2018). Labels become C regression problems with
label-dependent heteroscedastic noise:

    alpha_ic = alpha_eps + [label_i == c]
    noise_ic = log(1 / alpha_ic + 1)                  (lognormal moment match)
    target_ic = log(alpha_ic) - noise_ic / 2 - mean_c (class mean removed: zero-mean GPR)

and class c is a GP regression with Khat_c = f^2 kappa + s I + diag(noise_c); the
classes share (l, f, s). The loss is the sum of the C regression NLMLs. On the device
all C target solves and all C * k_z probe solves run as ONE grouped PCG
(kgp_gpc_nlml_grad): every iteration is one fused Khat [p_1..p_C, P_Z] application, the
per-class diagonal being added in the epilogue pass (kgp_engine_set_diag). Each class's
target column is preconditioned by its own AFN (or Nystrom-free: None).

Prediction: latent mean m_c + K(X*, X) w_c from one fused cross product over all C
columns; class probabilities by Monte-Carlo over the latent Gaussians when variances are
available (exact mode), else softmax of the latent means.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np

from paper_2503_02259_b200 import _device
from paper_2503_02259_b200 import precond as precond_mod
from paper_2503_02259_b200 import solver
from paper_2503_02259_b200._lib import call
from paper_2503_02259_b200.errors import NumericalError
from paper_2503_02259_b200.gp import LOG_2PI, LossGrad
from paper_2503_02259_b200.kernels import as_points
from paper_2503_02259_b200.kmat import Hyperparams, KernelEngine, Theta

DEFAULT_ALPHA_EPS = 0.01


@dataclass
class GPCProblem:
    """Transformed regression problems of a labelled data set (n points, C classes)."""

    x: np.ndarray
    labels: np.ndarray
    num_classes: int
    alpha_eps: float
    targets: np.ndarray   # (C, n) zero-mean regression targets
    noise: np.ndarray     # (C, n) heteroscedastic noise variances
    means: np.ndarray     # (C,) removed target means

    @property
    def n(self) -> int:
        return self.x.shape[0]


def setup(x, labels, num_classes: int | None = None, alpha_eps: float = DEFAULT_ALPHA_EPS) -> GPCProblem:
    """GPC problem setup (the analogue of HiGP's gpcproblem.setup(data, label))."""
    x = as_points(x, "X")
    lab = np.asarray(labels).reshape(-1)
    if lab.shape[0] != x.shape[0]:
        raise ValueError(f"labels must have length {x.shape[0]}, got {lab.shape[0]}")
    if not np.issubdtype(lab.dtype, np.integer):
        if not np.all(np.equal(np.mod(lab, 1), 0)):
            raise ValueError("labels must be integers")
        lab = lab.astype(np.int64)
    if lab.size and lab.min() < 0:
        raise ValueError("labels must be non-negative")
    c = int(num_classes) if num_classes is not None else int(lab.max()) + 1
    if c < 2 or (lab.size and lab.max() >= c):
        raise ValueError(f"need labels in [0, {c}) with at least 2 classes")
    if not alpha_eps > 0:
        raise ValueError("alpha_eps must be positive")
    onehot = (lab[None, :] == np.arange(c)[:, None]).astype(np.float64)
    alpha = alpha_eps + onehot
    noise = np.log(1.0 / alpha + 1.0)
    t = np.log(alpha) - 0.5 * noise
    means = t.mean(axis=1)
    return GPCProblem(x, lab.astype(np.int64), c, float(alpha_eps), t - means[:, None], noise, means)


def generate_probes(n: int, num_classes: int, k_z: int, rng_seed) -> np.ndarray:
    """(C * k_z, n): class c's probes at rows [c k_z, (c+1) k_z), seeded numpy PCG64."""
    if k_z < 1:
        raise ValueError("need at least one probe")
    return np.random.default_rng(rng_seed).standard_normal((num_classes * k_z, n))


def build_preconditioners(engine, problem: GPCProblem, rank: int | None = None, kind: str = "afn",
                          fsai_npt: int = precond_mod.AFN_DEFAULT_NPT):
    """One preconditioner per class for Khat + diag(noise_c): 'afn' (the class's noise on the
    diagonal exactly), 'nystrom' (M = (s + mean noise_c) I + f^2 V V^T: cheap, and its
    N(0, M) draws make a good preconditioned-probe estimator when the kernel is smooth), or
    'none'."""
    if kind == "none":
        return []
    if kind == "nystrom":
        s = engine.params.s
        return [precond_mod.build(engine, rank, shift=s + float(np.mean(problem.noise[c])))
                for c in range(problem.num_classes)]
    if kind != "afn":
        raise ValueError(f"kind must be 'afn', 'nystrom' or 'none', got {kind!r}")
    return [precond_mod.build_afn(engine, rank, fsai_npt, diag=problem.noise[c])
            for c in range(problem.num_classes)]


def nlml_grad_iterative(engine: KernelEngine, problem: GPCProblem, preconditioners, probes,
                        tol: float = solver.DEFAULT_TOL, max_iter: int = solver.DEFAULT_MAX_ITER,
                        probe_tol: float | None = None, *, probe_max_iter: int | None = None,
                        preconditioned_probes: bool = False) -> LossGrad:
    """Summed Dirichlet-GPC loss and (l, f, s) gradient, one libkgp call (kgp_gpc_nlml_grad).

    ``preconditioned_probes=True`` (one AFN/Nystrom preconditioner per class): the probe rows
    of class c are standard normals turned into draws from N(0, M_c) and every solve is
    preconditioned (kgp_gpc_nlml_grad_pp; gp.nlml_grad_iterative documents the estimator)."""
    torch = _device.torch()
    n, c = problem.n, problem.num_classes
    if engine.n != n:
        raise ValueError(f"engine has {engine.n} points, problem has {n}")
    probes = np.asarray(probes, dtype=np.float64)
    if probes.ndim != 2 or probes.shape[1] != n or probes.shape[0] % c:
        raise ValueError(f"probes must be (C * k_z, n) = (multiple of {c}, {n}), got {probes.shape}")
    k_z = probes.shape[0] // c
    pcs = list(preconditioners or [])
    if len(pcs) not in (0, 1, c):
        raise ValueError(f"need 0, 1 or {c} preconditioners, got {len(pcs)}")
    if probe_tol is None:
        probe_tol = tol
    dev = _device.device()
    dn = torch.from_numpy(np.ascontiguousarray(problem.noise)).to(dev)
    yd = torch.from_numpy(np.ascontiguousarray(problem.targets)).to(dev)
    zd = torch.from_numpy(np.ascontiguousarray(probes)).to(dev)
    arr = (ctypes.c_void_p * max(1, len(pcs)))(*[p.handle for p in pcs]) if pcs else None
    out = (ctypes.c_double * 4)()
    conv = ctypes.c_int32()
    if preconditioned_probes:
        if len(pcs) != c or any(getattr(p, "logdet", None) is None for p in pcs):
            raise ValueError("preconditioned probes need one AFN/Nystrom preconditioner per class")
        draws = []
        for k in range(c):
            w = zd[k * k_z:(k + 1) * k_z].T                     # (n, k_z) standard normals
            pk = pcs[k]
            draws.append(pk.sample(w) if isinstance(pk, precond_mod.AFNPreconditioner)
                         else pk.sample(w, torch.from_numpy(np.random.default_rng(
                             [k, precond_mod.PP_TAIL_SEED]).standard_normal((pk.rank, k_z))).to(dev)))
        zd = torch.cat(draws, dim=0).contiguous()
        call("kgp_gpc_nlml_grad_pp", engine.handle, c, arr, dn.data_ptr(), yd.data_ptr(), k_z, zd.data_ptr(),
             float(sum(p.logdet for p in pcs)), float(tol), int(max_iter), float(probe_tol),
             int(probe_max_iter or 0), out, ctypes.byref(conv), _device.stream_ptr())
        return LossGrad(out[0], out[1], out[2], out[3], converged=bool(conv.value))
    call("kgp_gpc_nlml_grad", engine.handle, c, arr, len(pcs), dn.data_ptr(), yd.data_ptr(), k_z, zd.data_ptr(),
         float(tol), int(max_iter), float(probe_tol), int(probe_max_iter or 0), out, ctypes.byref(conv),
         _device.stream_ptr())
    return LossGrad(out[0], out[1], out[2], out[3], converged=bool(conv.value))


def solve_targets(engine: KernelEngine, problem: GPCProblem, preconditioners, tol: float, max_iter: int):
    """(C, n) device tensor of w_c = (Khat + diag(noise_c))^-1 target_c: one grouped PCG, one
    column per class, class c preconditioned by preconditioners[c] (kgp_pcg_grouped)."""
    torch = _device.torch()
    c, n = problem.num_classes, problem.n
    dev = engine.x_device().device
    pcs = list(preconditioners or [])
    dn = torch.from_numpy(np.ascontiguousarray(problem.noise)).to(dev)
    yt = torch.from_numpy(np.ascontiguousarray(problem.targets)).to(dev)
    x = torch.empty((c, n), dtype=torch.float64, device=dev)
    al = torch.empty((c, max_iter), dtype=torch.float64, device=dev)
    be = torch.empty_like(al)
    it = torch.empty(c, dtype=torch.int32, device=dev)
    rel = torch.empty(c, dtype=torch.float64, device=dev)
    conv = torch.empty(c, dtype=torch.int32, device=dev)
    arr = (ctypes.c_void_p * len(pcs))(*[p.handle for p in pcs]) if pcs else None
    call("kgp_engine_set_diag", engine.handle, c, dn.data_ptr(), c, (ctypes.c_int32 * c)(*range(c)),
         _device.stream_ptr())
    try:
        call("kgp_pcg_grouped", engine.handle, arr, len(pcs), c, c, yt.data_ptr(), float(tol), int(max_iter),
             float(tol), int(max_iter), x.data_ptr(), al.data_ptr(), be.data_ptr(), it.data_ptr(), rel.data_ptr(),
             conv.data_ptr(), _device.stream_ptr())
    finally:
        call("kgp_engine_set_diag", engine.handle, 0, None, 0, None, _device.stream_ptr())
    return x


def grad_exact(engine: KernelEngine, problem: GPCProblem) -> LossGrad:
    """Dense per-class Cholesky (cuSOLVER) loss and gradient: the small-n reference path."""
    torch = _device.torch()
    kbase = engine.materialize_device()
    dks = [engine.materialize_grad_device(t) for t in (Theta.L, Theta.F, Theta.S)]
    loss, g = 0.0, np.zeros(3)
    for c in range(problem.num_classes):
        k = kbase.clone()
        k.diagonal().add_(torch.from_numpy(problem.noise[c]).to(k.device))
        low, info = torch.linalg.cholesky_ex(k)
        if int(info) != 0:
            raise NumericalError("class covariance is not SPD")
        y = torch.from_numpy(problem.targets[c]).to(k.device)
        w = torch.cholesky_solve(y[:, None], low)[:, 0]
        loss += 0.5 * (float(y @ w) + 2.0 * float(torch.log(torch.diagonal(low)).sum()) + problem.n * LOG_2PI)
        for i, dk in enumerate(dks):
            quad = -float(w @ (dk @ w))
            tr = float(torch.diagonal(torch.cholesky_solve(dk, low)).sum())
            g[i] += 0.5 * (quad + tr)
    return LossGrad(loss, g[0], g[1], g[2])


@dataclass
class GPCPrediction:
    mean: np.ndarray            # (m, C) latent means
    probabilities: np.ndarray   # (m, C)
    labels: np.ndarray          # (m,)
    variance: np.ndarray | None = None


def predict(kt, problem: GPCProblem, xstar, params: Hyperparams, mode: str = "iterative",
            tol: float = 1e-8, max_iter: int = solver.DEFAULT_MAX_ITER, rank: int | None = None,
            num_samples: int = 256, seed=0, precision: str | None = None) -> GPCPrediction:
    """Latent means (and, in exact mode, variances) per class; probabilities by MC over the
    latent Gaussians (exact) or softmax of the means (iterative)."""
    torch = _device.torch()
    if mode not in ("exact", "iterative"):
        raise ValueError(f"mode must be 'exact' or 'iterative', got {mode!r}")
    xstar = as_points(np.asarray(xstar, dtype=np.float64).reshape(-1, problem.x.shape[1]), "Xstar")
    c = problem.num_classes
    engine = KernelEngine(kt, problem.x, params, precision=precision)
    star = KernelEngine(kt, xstar, params, precision=precision)
    dev = engine.x_device().device
    var = None
    if mode == "exact":
        kb = engine.materialize_device()
        cross = star.cross_matmul(engine.x_device(), torch.eye(xstar.shape[0], dtype=torch.float64, device=dev))
        ws, var = [], np.empty((xstar.shape[0], c))
        for k in range(c):
            kc = kb.clone()
            kc.diagonal().add_(torch.from_numpy(problem.noise[k]).to(dev))
            low = torch.linalg.cholesky(kc)
            ws.append(torch.cholesky_solve(torch.from_numpy(problem.targets[k]).to(dev)[:, None], low)[:, 0])
            sol = torch.cholesky_solve(cross, low)
            var[:, k] = _device.to_host(torch.clamp(params.f ** 2 - (cross * sol).sum(dim=0), min=0.0))
        w = torch.stack(ws, dim=1)
    else:
        pcs = build_preconditioners(engine, problem, rank)
        w = solve_targets(engine, problem, pcs, tol, max_iter).T.contiguous()
    mean = _device.to_host(engine.cross_matmul(star.x_device(), w)) + problem.means[None, :]
    if var is not None:
        rng = np.random.default_rng(seed)
        draws = mean[None] + np.sqrt(var)[None] * rng.standard_normal((num_samples,) + mean.shape)
        e = np.exp(draws - draws.max(axis=2, keepdims=True))
        prob = (e / e.sum(axis=2, keepdims=True)).mean(axis=0)
    else:
        e = np.exp(mean - mean.max(axis=1, keepdims=True))
        prob = e / e.sum(axis=1, keepdims=True)
    return GPCPrediction(mean=mean, probabilities=prob, labels=np.argmax(mean, axis=1), variance=var)


@dataclass
class GPCTrainResult:
    params: Hyperparams
    loss_history: list = field(default_factory=list)
    grad_norm_history: list = field(default_factory=list)
    converged: bool = True


def fit(kt, problem: GPCProblem, init: Hyperparams | None = None, steps: int = 10, learning_rate: float = 0.1,
        k_z: int = 16, rank: int | None = None, fsai_npt: int = precond_mod.AFN_DEFAULT_NPT,
        tol: float = solver.DEFAULT_TOL, max_iter: int = solver.DEFAULT_MAX_ITER,
        probe_tol: float | None = None, rng_seed: int = 0, precision: str | None = None,
        preconditioner: str = "afn", preconditioned_probes: bool = False) -> GPCTrainResult:
    """Adam in softplus space over (l, f, s) (train.py's optimiser), probes redrawn per step
    from (rng_seed, step); one engine reused across steps (hyperparameters reset in place)."""
    from paper_2503_02259_b200.train import Adam, RawParams, chain_grads

    hp = init or Hyperparams(l=1.0, f=1.0, s=0.1)
    raw = RawParams.from_hyperparams(hp)
    opt = Adam(learning_rate)
    engine = KernelEngine(kt, problem.x, hp, precision=precision)
    res = GPCTrainResult(params=hp)
    try:
        for step in range(steps):
            hp = raw.to_hyperparams()
            engine.set_params(hp)
            pcs = build_preconditioners(engine, problem, rank, preconditioner, fsai_npt)
            probes = generate_probes(problem.n, problem.num_classes, k_z, (rng_seed, step))
            lg = nlml_grad_iterative(engine, problem, pcs, probes, tol=tol, max_iter=max_iter, probe_tol=probe_tol,
                                     preconditioned_probes=preconditioned_probes)
            for p in pcs:
                p.close()
            g_rho = chain_grads(raw, lg.grads())
            res.loss_history.append(lg.loss)
            res.grad_norm_history.append(float(np.linalg.norm(g_rho)))
            res.converged &= lg.converged
            raw = RawParams.from_array(opt.step(raw.as_array(), g_rho))
    finally:
        engine.close()
    res.params = raw.to_hyperparams()
    return res


def sample_latent_labels(x, num_classes: int, l: float = 1.0, num_features: int = 4096, seed=0) -> np.ndarray:
    """cfg4's labels: argmax over C latent GP draws with a Gaussian kernel of length scale l.
    An exact draw at n = 131072 needs an O(n^3) factorisation, so each latent function is a
    random-Fourier-feature draw (num_features features; converges to the GP as it grows)."""
    x = as_points(x, "X")
    rng = np.random.default_rng(seed)
    d = x.shape[1]
    omega = rng.standard_normal((d, num_features)) / l
    phase = rng.uniform(0.0, 2.0 * math.pi, num_features)
    weights = rng.standard_normal((num_features, num_classes))
    out = np.empty(x.shape[0], dtype=np.int64)
    for r0 in range(0, x.shape[0], 4096):  # bounded host memory at n = 131072
        feats = np.sqrt(2.0 / num_features) * np.cos(x[r0:r0 + 4096] @ omega + phase)
        out[r0:r0 + 4096] = np.argmax(feats @ weights, axis=1)
    return out
