"""GPR problem setup, loss+gradient and prediction: HiGP's Listing-1 user API
("bindings" module) over this package's device path.

    problem = gpr.setup(data=train_x, label=train_y, kernel_type=KernelType.GAUSSIAN)
    model = gpr.GPRModel(problem)
    optimizer = torch.optim.Adam(model.parameters(), lr=0.1)
    for i in range(max_steps):
        loss = model.calc_loss_grad()
        optimizer.step()
    params = model.get_params()
    pred = gpr.gpr_prediction(train_x, train_y, test_x, KernelType.GAUSSIAN, params)
    pred.prediction_mean, pred.prediction_stddev

The binding layer computes nothing itself: ``calc_loss_grad`` is
``gp.grad_exact`` / ``gp.nlml_grad_iterative`` on the device engine followed by the
softplus chain rule of the reference's train.py:79-81, and ``gpr_prediction`` is
``gp.predict``. The problem handle copies the caller's arrays and keeps X
resident on the device between evaluations (``KernelEngine.set_params``), which is what a
training loop over one data set wants.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from paper_2503_02259_b200 import gp, precond, solver
from paper_2503_02259_b200.errors import KernelGpError
from paper_2503_02259_b200.kernels import KernelType, as_points
from paper_2503_02259_b200.kmat import DEFAULT_DENSE_BUDGET, Hyperparams, KernelEngine
from paper_2503_02259_b200.train import RawParams, chain_grads, initial_hyperparams, softplus_inv


@dataclass
class GPROptions:
    """Solver configuration a problem handle carries (the reference's TrainConfig fields
    that shape one loss evaluation, train.py:122-140)."""

    mode: str = "iterative"                  # "exact" (dense Cholesky) | "iterative"
    k_z: int = gp.DEFAULT_NUM_PROBES
    tol: float = solver.DEFAULT_TOL
    probe_tol: float = solver.DEFAULT_PROBE_TOL
    max_iter: int = solver.DEFAULT_MAX_ITER
    precond_rank: int | None = None
    rng_seed: int = 0
    dense_budget: int = DEFAULT_DENSE_BUDGET
    precision: str | None = None             # operator arithmetic: fp64 | fast | tf32
    preconditioner: str = "nystrom"          # "nystrom" (the reference's) | "afn" | "adaptive"

    def __post_init__(self):
        if self.mode not in ("exact", "iterative"):
            raise ValueError(f"mode must be 'exact' or 'iterative', got {self.mode!r}")
        if self.preconditioner not in ("nystrom", "afn", "adaptive"):
            raise ValueError(f"preconditioner must be 'nystrom', 'afn' or 'adaptive', got {self.preconditioner!r}")
        if self.k_z < 1:
            raise ValueError("need at least one probe")


class GPRProblem:
    """Problem handle of ``setup``: kernel type, a copy of the training data, solver options.
    Valid until ``release()``; every evaluation is side-effect free on the caller's data."""

    def __init__(self, data, label, kernel_type, options: GPROptions, operator=None):
        self.x = as_points(data, "X").copy()
        y = np.asarray(label, dtype=np.float64).reshape(-1)
        if y.shape[0] != self.x.shape[0]:
            raise ValueError(f"label length mismatch: {y.shape[0]} labels for {self.x.shape[0]} points")
        if not np.isfinite(y).all():
            raise ValueError("label contains non-finite entries")
        self.y = y.copy()
        self.x.setflags(write=False)
        self.y.setflags(write=False)
        self.kernel_type = KernelType(getattr(kernel_type, "value", kernel_type))
        self.options = options
        self._operator = operator  # duck-typed test operator (the reference's IdentityOperator)
        self._engine = None
        self._released = False

    @property
    def n(self) -> int:
        return self.x.shape[0]

    def _engine_at(self, hp: Hyperparams):
        if self._released:
            raise KernelGpError("GPR problem handle was released")
        if self._operator is not None:
            return self._operator
        if self._engine is None:
            self._engine = KernelEngine(self.kernel_type, self.x, hp, dense_budget=self.options.dense_budget,
                                        precision=self.options.precision)
        else:
            self._engine.set_params(hp)
        return self._engine

    def loss_grad(self, params: Hyperparams, step: int | None = None) -> gp.LossGrad:
        """The core LossGrad at hyperparameters ``params`` (gp.py:116-179). In iterative mode
        the probes are drawn from ``(rng_seed, step)`` as train.py:209 does (``rng_seed`` alone
        when ``step`` is None)."""
        opt = self.options
        engine = self._engine_at(params)
        if opt.mode == "exact":
            return gp.grad_exact(engine, self.y)
        seed = opt.rng_seed if step is None else (opt.rng_seed, step)
        probes = gp.ProbeSet.generate(self.n, opt.k_z, seed)
        pre = None
        if self._operator is None:
            if opt.preconditioner == "afn":
                pre = precond.build_afn(engine, opt.precond_rank)
            elif opt.preconditioner == "adaptive":
                pre = precond.build_adaptive(engine, opt.precond_rank)
            else:
                pre = precond.build(engine, opt.precond_rank)
        return gp.nlml_grad_iterative(engine, self.y, pre, probes, tol=opt.tol, max_iter=opt.max_iter,
                                      probe_tol=opt.probe_tol)

    def calc_loss_grad(self, raw_params, step: int | None = None):
        """(loss, dL/drho) at unconstrained parameters rho (softplus(rho) = (l, f, s)): the
        core loss and gradient with the reference's chain rule (train.py:79-81) applied."""
        raw = raw_params if isinstance(raw_params, RawParams) else RawParams.from_array(
            np.asarray(raw_params, dtype=np.float64).reshape(3))
        lg = self.loss_grad(raw.to_hyperparams(), step)
        return lg.loss, chain_grads(raw, lg.grads())

    def release(self) -> bool:
        """Free the device engine. A second release is a no-op that returns False."""
        if self._released:
            return False
        if self._engine is not None:
            self._engine.close()
            self._engine = None
        self._released = True
        return True

    def __del__(self):
        try:
            self.release()
        except Exception:
            pass


def setup(data, label, kernel_type=KernelType.GAUSSIAN, mode: str = "iterative", options: GPROptions | None = None,
          *, operator=None, **kw) -> GPRProblem:
    """``gprproblem.setup(data=train_x, label=train_y, kernel_type=...)`` (Listing 1, line 1).

    ``options`` or keyword fields of GPROptions configure the solver; ``operator`` injects a
    duck-typed Khat operator instead of the device engine (the reference's test seam,
    tests/test_gp.py:13-30)."""
    if options is None:
        options = GPROptions(mode=mode, **kw)
    elif kw:
        raise ValueError("pass either options or keyword fields, not both")
    return GPRProblem(data, label, kernel_type, options, operator)


class GPRModel:
    """Listing 1's ``GPRModel``: the raw hyperparameters as one torch parameter (rho_l, rho_f,
    rho_s), ``calc_loss_grad()`` sets its ``.grad`` for any torch optimizer and returns the loss;
    ``get_params()`` gives the current Hyperparams. Starts at the reference's data-driven
    initial point (train.py:150-174) unless ``init`` is given."""

    def __init__(self, problem: GPRProblem, init: Hyperparams | None = None):
        import torch

        hp = init if init is not None else initial_hyperparams(problem.x, problem.y, problem.options.rng_seed)
        rho = softplus_inv(hp.as_array())
        self.problem = problem
        self.raw = torch.nn.Parameter(torch.tensor(rho, dtype=torch.float64))
        self.step = 0

    def parameters(self):
        return [self.raw]

    def raw_params(self) -> RawParams:
        return RawParams.from_array(self.raw.detach().cpu().numpy())

    def get_params(self) -> Hyperparams:
        return self.raw_params().to_hyperparams()

    def calc_loss_grad(self) -> float:
        import torch

        loss, g = self.problem.calc_loss_grad(self.raw_params(), step=self.step)
        self.raw.grad = torch.tensor(g, dtype=torch.float64)
        self.step += 1
        return loss


def gpr_prediction(train_x, train_y, test_x, kernel_type, params, mode: str = "exact", **kw) -> gp.Prediction:
    """``gpr_prediction(train_x, train_y, test_x, kernel, params)`` (Listing 1, line 8):
    stateless (re-supplies the training data) and exactly ``gp.predict``.
    ``params`` is Hyperparams, RawParams or an (l, f, s) triple."""
    if isinstance(params, RawParams):
        params = params.to_hyperparams()
    elif not isinstance(params, Hyperparams):
        l, f, s = (float(v) for v in np.asarray(params, dtype=np.float64).reshape(3))
        params = Hyperparams(l=l, f=f, s=s)
    xs = np.asarray(test_x, dtype=np.float64)
    if xs.size == 0:
        return gp.Prediction(mean=np.empty(0), stddev=np.empty(0))
    return gp.predict(kernel_type, train_x, train_y, test_x, params, mode=mode, **kw)
