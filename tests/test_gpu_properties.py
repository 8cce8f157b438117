"""The reference's own property checks, restated against the device path.

kernelgp's test-suite (pkg/tests/test_kmat.py, test_solver.py, test_gp.py, test_precond.py) pins
the hot path with closed forms, edge cases and invariants rather than goldens. A drop-in has to
pass the same checks, so each one is restated here in this repository's words and run through
the CUDA engine, the device PCG driver, the device SLQ and the device preconditioner (the
reference file:line each check follows is cited next to it). Tolerances are the reference's
unless a comment says otherwise."""

import math

import numpy as np
import pytest

from conftest import rel_max

pytestmark = pytest.mark.gpu

KTS = ["gaussian", "matern32", "matern52"]


@pytest.fixture(scope="module")
def pkg():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2503_02259_b200 as p

    return p


def _hp(pkg, l, f, s):
    return pkg.Hyperparams(l=l, f=f, s=s)


def _kappa(kt, r, l):
    """Closed forms on a distance (kernels.py:30-60), written out independently of every engine."""
    if kt == "gaussian":
        return math.exp(-r * r / (2 * l * l))
    t = (math.sqrt(3.0) if kt == "matern32" else math.sqrt(5.0)) * r / l
    return (1 + t) * math.exp(-t) if kt == "matern32" else (1 + t + t * t / 3) * math.exp(-t)


def _khat_loops(kt, x, hp):
    n = x.shape[0]
    k = np.empty((n, n))
    for i in range(n):
        for j in range(n):
            k[i, j] = hp.f**2 * _kappa(kt, float(np.linalg.norm(x[i] - x[j])), hp.l)
    return k + hp.s * np.eye(n)


def _spd(n, rng, shift=1.0):
    g = rng.standard_normal((n, n))
    return g @ g.T + shift * np.eye(n)


# ---------------------------------------------------------------------------- operator (test_kmat.py)
@pytest.mark.parametrize("bad", [dict(l=0), dict(f=-1), dict(s=0), dict(l=float("nan"))])
def test_hyperparams_reject_nonpositive(pkg, bad):
    """test_kmat.py:20-26"""
    args = dict(l=1.0, f=1.0, s=1.0)
    args.update(bad)
    with pytest.raises(ValueError):
        pkg.Hyperparams(**args)


@pytest.mark.parametrize("mode", ["DENSE", "ON_THE_FLY"])
def test_basis_vector_extracts_column(pkg, mode):
    """test_kmat.py:34-40: Khat e_j is column j of the materialised matrix."""
    x = np.random.default_rng(0).standard_normal((15, 2))
    e = pkg.KernelEngine(pkg.KernelType.GAUSSIAN, x, _hp(pkg, 1.0, 1.0, 0.5), mode=getattr(pkg.EngineMode, mode))
    khat = e.materialize()
    for j in (0, 7, 14):
        ej = np.zeros(15)
        ej[j] = 1.0
        np.testing.assert_allclose(e.matmul(ej), khat[:, j], rtol=1e-14, atol=1e-300)


@pytest.mark.parametrize("kt", KTS)
def test_operator_matches_scalar_loops(pkg, kt, rng):
    """test_kmat.py:53-60 (every kernel type here): the device product against a double loop over
    the closed forms."""
    x = rng.standard_normal((12, 2))
    b = rng.standard_normal((12, 3))
    hp = _hp(pkg, 0.8, 1.5, 0.3)
    for mode in (pkg.EngineMode.DENSE, pkg.EngineMode.ON_THE_FLY):
        e = pkg.KernelEngine(pkg.KernelType(kt), x, hp, mode=mode)
        np.testing.assert_allclose(e.matmul(b), _khat_loops(kt, x, hp) @ b, rtol=1e-12)


def test_shapes_and_row_mismatch(pkg, rng):
    """test_kmat.py:62-75: a wrong row count is a ValueError, a 1-D right-hand side keeps its shape."""
    e = pkg.KernelEngine(pkg.KernelType.GAUSSIAN, rng.standard_normal((20, 2)), _hp(pkg, 1.0, 1.0, 0.5))
    with pytest.raises(ValueError):
        e.matmul(np.ones((19, 2)))
    with pytest.raises(ValueError):
        e.grad_matmul(pkg.Theta.L, np.ones(21))
    v = rng.standard_normal(20)
    assert e.matmul(v).shape == (20,)
    assert e.grad_matmul(pkg.Theta.L, v).shape == (20,)
    assert e.matmul(v[:, None]).shape == (20, 1)


@pytest.mark.parametrize("kt", KTS)
def test_derivative_products(pkg, kt, rng):
    """test_kmat.py:78-118: dKhat/ds B = B to the bit; dKhat/df B = (2/f)(Khat - sI) B; dKhat/dl B
    against a central finite difference of the operator itself."""
    x = rng.standard_normal((40, 3))
    b = rng.standard_normal((40, 2))
    hp = _hp(pkg, 1.1, 1.4, 0.2)
    e = pkg.KernelEngine(pkg.KernelType(kt), x, hp, mode=pkg.EngineMode.ON_THE_FLY)
    np.testing.assert_array_equal(e.grad_matmul(pkg.Theta.S, b), b)
    np.testing.assert_allclose(e.grad_matmul(pkg.Theta.F, b), (2 / hp.f) * (e.matmul(b) - hp.s * b), rtol=1e-12,
                               atol=1e-14)
    h = 1e-6 * hp.l
    up = pkg.KernelEngine(pkg.KernelType(kt), x, _hp(pkg, hp.l + h, hp.f, hp.s), mode=pkg.EngineMode.ON_THE_FLY)
    dn = pkg.KernelEngine(pkg.KernelType(kt), x, _hp(pkg, hp.l - h, hp.f, hp.s), mode=pkg.EngineMode.ON_THE_FLY)
    fd = (up.matmul(b) - dn.matmul(b)) / (2 * h)
    assert rel_max(e.grad_matmul(pkg.Theta.L, b), fd) <= 1e-6


def test_two_point_closed_form(pkg):
    """test_kmat.py:120-128: two points at distance r: Khat = [[f^2 + s, f^2 k(r)], [f^2 k(r), f^2 + s]]."""
    l, f, s, r = 0.7, 1.3, 0.05, 0.9
    for kt in KTS:
        e = pkg.KernelEngine(pkg.KernelType(kt), [[0.0], [r]], _hp(pkg, l, f, s), mode=pkg.EngineMode.ON_THE_FLY)
        off = f * f * _kappa(kt, r, l)
        np.testing.assert_allclose(e.matmul(np.eye(2)), [[f * f + s, off], [off, f * f + s]], rtol=1e-14)


@pytest.mark.parametrize("precision,tol", [("fp64", 1e-10), ("fast", 2e-5)])
def test_symmetry_and_noise_floor(pkg, precision, tol, rng):
    """test_kmat.py:143-155: c^T (Khat b) = (b^T Khat c)^T, and v^T Khat v >= s v^T v (the spectrum is
    bounded below by the noise), through the on-the-fly device operator in both precisions."""
    n = 64 if precision == "fp64" else 640
    x = rng.standard_normal((n, 2))
    e = pkg.KernelEngine(pkg.KernelType.MATERN52, x, _hp(pkg, 1.0, 1.0, 0.5), mode=pkg.EngineMode.ON_THE_FLY,
                         precision=precision)
    b = rng.standard_normal((n, 3))
    c = rng.standard_normal((n, 2))
    left = c.T @ e.matmul(b)
    right = (b.T @ e.matmul(c)).T
    assert np.max(np.abs(left - right)) <= tol * np.max(np.abs(left))
    e2 = pkg.KernelEngine(pkg.KernelType.GAUSSIAN, x, _hp(pkg, 2.0, 1.0, 0.05), mode=pkg.EngineMode.ON_THE_FLY,
                          precision=precision)
    slack = 1e-10 if precision == "fp64" else 1e-3
    for _ in range(10):
        v = rng.standard_normal(n)
        assert v @ e2.matmul(v) >= 0.05 * (v @ v) * (1 - slack)


def test_materialize_symmetric_and_budget(pkg, rng):
    """test_kmat.py:130-139: the materialised matrix is symmetric to the bit; the dense budget is
    enforced with the budget in the message."""
    x = rng.standard_normal((30, 2))
    e = pkg.KernelEngine(pkg.KernelType.MATERN32, x, _hp(pkg, 1.0, 1.0, 0.5))
    k = e.materialize()
    np.testing.assert_array_equal(k, k.T)
    small = pkg.KernelEngine(pkg.KernelType.GAUSSIAN, x, _hp(pkg, 1.0, 1.0, 0.5), dense_budget=25,
                             mode=pkg.EngineMode.ON_THE_FLY)
    from paper_2503_02259_b200.errors import ResourceLimitError

    with pytest.raises(ResourceLimitError, match="25"):
        small.materialize()


# ---------------------------------------------------------------------------- batched PCG (test_solver.py)
def test_pcg_generic_callables(pkg, rng):
    """test_solver.py:71-128 on this package's pcg_solve with plain callables (device-resident
    state, the caller's operator): a perfect preconditioner converges in one iteration; no
    preconditioner reproduces cg_solve's alphas and betas; batched equals column by column;
    columns stop independently; a zero column stays zero; non-convergence is reported."""
    from paper_2503_02259_b200 import solver

    a = _spd(25, rng)
    inv = np.linalg.inv(a)
    y = rng.standard_normal((25, 3))
    rep = solver.pcg_solve(lambda b: a @ b, lambda b: inv @ b, y, tol=1e-8)
    assert all(t.iterations == 1 for t in rep.traces) and rep.all_converged

    a = _spd(40, rng, shift=20.0)

    def by_columns(b):  # the same matrix-vector rounding for the block and the single-vector solve
        if b.ndim == 1:
            return a @ b
        return np.column_stack([a @ np.ascontiguousarray(b[:, j]) for j in range(b.shape[1])])

    y = rng.standard_normal((40, 2))
    rep = solver.pcg_solve(by_columns, None, y, tol=1e-9, max_iter=200)
    for j in range(2):
        xj, tj = solver.cg_solve(by_columns, y[:, j], tol=1e-9, max_iter=200)
        assert tj.iterations == rep.traces[j].iterations
        np.testing.assert_allclose(rep.traces[j].alphas, tj.alphas, rtol=1e-12)
        np.testing.assert_allclose(rep.traces[j].betas, tj.betas, rtol=1e-12)
        np.testing.assert_allclose(rep.solution[:, j], xj, rtol=1e-12, atol=1e-14)

    a = _spd(35, rng)
    minv = np.diag(1.0 / np.diag(a))
    y = rng.standard_normal((35, 5))
    batched = solver.pcg_solve(lambda b: a @ b, lambda b: minv @ b, y, tol=1e-10, max_iter=300)
    for j in range(5):
        single = solver.pcg_solve(lambda b: a @ b, lambda b: minv @ b, y[:, j], tol=1e-10, max_iter=300)
        np.testing.assert_allclose(batched.solution[:, j], single.solution, rtol=1e-10, atol=1e-12)

    a = np.diag([1.0, 2.0, 3.0, 4.0])
    y = np.zeros((4, 2))
    y[0, 0] = 1.0
    y[:, 1] = rng.standard_normal(4)
    rep = solver.pcg_solve(lambda b: a @ b, None, y, tol=1e-12, max_iter=50)
    assert rep.traces[0].iterations < rep.traces[1].iterations and rep.all_converged
    np.testing.assert_allclose(rep.solution[:, 0], y[:, 0], rtol=1e-12)

    y = np.zeros((6, 2))
    y[:, 1] = 1.0
    rep = solver.pcg_solve(lambda b: 2.0 * b, None, y, tol=1e-12)
    np.testing.assert_array_equal(rep.solution[:, 0], np.zeros(6))
    np.testing.assert_allclose(rep.solution[:, 1], 0.5 * np.ones(6), rtol=1e-14)

    a = _spd(30, rng, shift=1e-6)
    rep = solver.pcg_solve(lambda b: a @ b, None, rng.standard_normal(30), tol=1e-14, max_iter=2)
    assert not rep.all_converged


@pytest.mark.parametrize("precision", ["fp64", "fast"])
def test_pcg_device_driver_edge_cases(pkg, precision, rng):
    """The same properties through the DEVICE driver (kgp_pcg: the engine's fused operator and the
    Nystrom application inside the captured iteration): batched equals column by column, a zero
    column stays exactly zero with no iteration, non-convergence is reported, the solution
    solves the dense system."""
    from paper_2503_02259_b200 import precond, solver

    n = 300
    x = rng.uniform(-1, 1, (n, 2))
    hp = _hp(pkg, 0.6, 1.0, 0.05)
    e = pkg.KernelEngine(pkg.KernelType.GAUSSIAN, x, hp, mode=pkg.EngineMode.ON_THE_FLY, precision=precision)
    pre = precond.build(e, 40)
    y = rng.standard_normal((n, 4))
    y[:, 2] = 0.0
    tol = 1e-10 if precision == "fp64" else 1e-5
    rep = solver.pcg_solve(e.matmul, pre.apply_inverse, y, tol=tol, max_iter=2000)
    assert rep.all_converged
    np.testing.assert_array_equal(rep.solution[:, 2], np.zeros(n))
    assert rep.traces[2].iterations == 0
    exact = np.linalg.solve(_khat_loops("gaussian", x, hp), y)
    assert rel_max(rep.solution, exact) <= (1e-8 if precision == "fp64" else 2e-3)
    for j in (0, 3):
        single = solver.pcg_solve(e.matmul, pre.apply_inverse, y[:, j], tol=tol, max_iter=2000)
        assert single.solution.shape == (n,)
        assert single.traces[0].iterations == rep.traces[j].iterations
        np.testing.assert_allclose(single.solution, rep.solution[:, j], rtol=1e-9 if precision == "fp64" else 1e-4,
                                   atol=1e-12)
    short = solver.pcg_solve(e.matmul, None, y[:, 0], tol=1e-14, max_iter=2)
    assert not short.all_converged and short.traces[0].iterations == 2


# ---------------------------------------------------------------------------- tridiagonals and SLQ
def test_tridiag_layout_and_validation(pkg):
    """test_solver.py:131-177: T = [[1/a0]] after one iteration; the 2x2 layout; a negative beta and
    a non-positive Ritz value are ValueErrors; mismatched probe norms are rejected."""
    from paper_2503_02259_b200 import solver

    tr = solver.CgTrace(np.array([2.0]), np.array([0.1]), 1, 0.0)
    np.testing.assert_allclose(solver.build_tridiag(tr), [[0.5]], rtol=1e-15)
    tr = solver.CgTrace(np.array([0.5, 0.25]), np.array([0.04, 0.0]), 2, 0.0)
    np.testing.assert_allclose(solver.build_tridiag(tr), [[2.0, 0.4], [0.4, 4.08]], rtol=1e-14)
    with pytest.raises(ValueError, match="negative betas"):
        solver.build_tridiag(solver.CgTrace(np.array([1.0, 1.0]), np.array([-0.1, 0.0]), 2, 0.0))
    with pytest.raises(ValueError, match="probe norms"):
        solver.slq_logdet([], [1.0])
    with pytest.raises(ValueError):
        solver.slq_logdet([solver.CgTrace(np.array([-1.0]), np.array([0.0]), 1, 0.0)], [1.0])


def test_tridiag_spectrum_properties(pkg, rng):
    """test_solver.py:146-170: two distinct eigenvalues are recovered in two iterations; Ritz values
    lie inside the spectrum; T is symmetric with a positive diagonal."""
    from paper_2503_02259_b200 import solver

    a = np.diag([1.0, 3.0])
    _, tr = solver.cg_solve(lambda v: a @ v, np.array([1.0, 1.0]), tol=0.0, max_iter=2)
    np.testing.assert_allclose(np.sort(np.linalg.eigvalsh(solver.build_tridiag(tr))), [1.0, 3.0], atol=1e-10)
    for _ in range(3):
        a = _spd(50, rng)
        lam = np.linalg.eigvalsh(a)
        _, tr = solver.cg_solve(lambda v: a @ v, rng.standard_normal(50), tol=1e-10, max_iter=50)
        t = solver.build_tridiag(tr)
        ritz = np.linalg.eigvalsh(t)
        assert ritz.min() >= lam.min() - 1e-8 and ritz.max() <= lam.max() + 1e-8
        np.testing.assert_array_equal(t, t.T)
        assert np.all(np.diag(t) > 0)


def test_slq_closed_forms(pkg, rng):
    """test_solver.py:180-218: the identity has log-determinant exactly 0; a scalar matrix gives
    z^2 log a per probe; diag(1..10) with 200 probes is within 5 %."""
    from paper_2503_02259_b200 import solver

    z = rng.standard_normal((10, 6))
    rep = solver.pcg_solve(lambda b: b, None, z, tol=1e-12)
    assert solver.slq_logdet(rep.traces, np.sum(z * z, axis=0)) == 0.0
    zs = np.array([1.7])
    _, tr = solver.cg_solve(lambda v: 2.5 * v, zs, tol=1e-14)
    np.testing.assert_allclose(solver.slq_logdet([tr], [zs[0] ** 2]), zs[0] ** 2 * math.log(2.5), rtol=1e-12)
    d = np.arange(1.0, 11.0)
    z = rng.standard_normal((10, 200))
    rep = solver.pcg_solve(lambda b: d[:, None] * b, None, z, tol=0.0, max_iter=10)
    est = solver.slq_logdet(rep.traces, np.sum(z * z, axis=0))
    truth = float(np.sum(np.log(d)))
    assert abs(est - truth) / truth < 0.05


# ---------------------------------------------------------------------------- NLML and prediction (test_gp.py)
def test_nlml_single_point_closed_forms(pkg):
    """test_gp.py:41-68: one training point: loss = (y^2/c + log c + log 2 pi)/2 with c = f^2 + s,
    dL/ds = (-y^2/c^2 + 1/c)/2 and dL/df = 2 f dL/ds; vanishing noise at y = 0 leaves log(2 pi)/2."""
    from paper_2503_02259_b200 import gp

    e = pkg.KernelEngine(pkg.KernelType.GAUSSIAN, [[0.0]], _hp(pkg, 1, 2, 0.1))
    np.testing.assert_allclose(gp.nlml_exact(e, [1.0]), 0.5 * (1 / 4.1 + math.log(4.1) + math.log(2 * math.pi)),
                               rtol=1e-14)
    e0 = pkg.KernelEngine(pkg.KernelType.GAUSSIAN, [[0.0]], _hp(pkg, 1, 1, 1e-12))
    np.testing.assert_allclose(gp.nlml_exact(e0, [0.0]), 0.5 * math.log(2 * math.pi), rtol=1e-9)
    f, s, yv = 2.0, 0.1, 1.3
    c = f * f + s
    lg = gp.grad_exact(pkg.KernelEngine(pkg.KernelType.MATERN32, [[0.0]], _hp(pkg, 1, f, s)), [yv])
    np.testing.assert_allclose(lg.grad_s, 0.5 * (-(yv**2) / c**2 + 1 / c), rtol=1e-13)
    np.testing.assert_allclose(lg.grad_f, 2 * f * lg.grad_s, rtol=1e-13)


@pytest.mark.parametrize("kt", KTS)
def test_exact_gradient_vs_finite_differences(pkg, kt, rng):
    """test_gp.py:70-86: the exact gradient (device Cholesky path) against central differences of
    the exact loss, 1e-5 relative; its loss equals nlml_exact."""
    from paper_2503_02259_b200 import gp

    x = rng.standard_normal((100, 3))
    y = rng.standard_normal(100)
    base = dict(l=1.4, f=0.9, s=0.2)
    e = pkg.KernelEngine(pkg.KernelType(kt), x, pkg.Hyperparams(**base))
    lg = gp.grad_exact(e, y)
    assert lg.loss == gp.nlml_exact(e, y)
    for name, analytic in zip(("l", "f", "s"), lg.grads()):
        h = 1e-6 * base[name]
        vals = []
        for sign in (+1, -1):
            hp = dict(base)
            hp[name] += sign * h
            vals.append(gp.nlml_exact(pkg.KernelEngine(pkg.KernelType(kt), x, pkg.Hyperparams(**hp)), y))
        fd = (vals[0] - vals[1]) / (2 * h)
        assert abs(analytic - fd) / (abs(analytic) + 1e-12) < 1e-5


def test_iterative_gradient_matches_dense_algebra(pkg, rng):
    """test_gp.py:103-120: with the estimator's own probes, every gradient component equals
    (-w^T dK w + mean_z (Khat^-1 z)^T dK z)/2 formed with dense algebra, 1e-6 relative; the
    evaluation is deterministic for a seed; probe rows are checked."""
    from paper_2503_02259_b200 import gp, precond

    n = 200
    x = np.random.default_rng(4).standard_normal((n, 2))
    y = np.random.default_rng(5).standard_normal(n)
    hp = _hp(pkg, 1.0, 1.2, 0.3)
    e = pkg.KernelEngine(pkg.KernelType.GAUSSIAN, x, hp, mode=pkg.EngineMode.ON_THE_FLY)
    pre = precond.build(e, 60)
    probes = gp.ProbeSet.generate(n, 4, 3)
    lg = gp.nlml_grad_iterative(e, y, pre, probes, tol=1e-12, max_iter=1000)
    khat = _khat_loops("gaussian", x, hp)
    w = np.linalg.solve(khat, y)
    u = np.linalg.solve(khat, probes.vectors)
    for theta, got in ((pkg.Theta.L, lg.grad_l), (pkg.Theta.F, lg.grad_f), (pkg.Theta.S, lg.grad_s)):
        dk = e.materialize_grad(theta)
        dense = 0.5 * (-w @ dk @ w + float(np.einsum("ij,ij->", u, dk @ probes.vectors)) / probes.k_z)
        assert abs(got - dense) / (abs(dense) + 1e-12) < 1e-6
    again = gp.nlml_grad_iterative(e, y, pre, gp.ProbeSet.generate(n, 4, 3), tol=1e-12, max_iter=1000)
    assert (lg.loss, lg.grad_l, lg.grad_f, lg.grad_s) == (again.loss, again.grad_l, again.grad_f, again.grad_s)
    with pytest.raises(ValueError, match="rows"):
        gp.nlml_grad_iterative(e, y, None, gp.ProbeSet.generate(n - 10, 4, 0))


def test_estimator_within_confidence_interval(pkg):
    """test_gp.py:122-145 (20 seeds instead of 50): the stochastic loss and gradient estimates
    scatter around the exact values within three standard errors."""
    from paper_2503_02259_b200 import gp, precond

    n = 150
    x = np.random.default_rng(8).standard_normal((n, 2))
    y = np.random.default_rng(9).standard_normal(n)
    e = pkg.KernelEngine(pkg.KernelType.GAUSSIAN, x, _hp(pkg, 1.0, 1.2, 0.3), mode=pkg.EngineMode.ON_THE_FLY)
    exact = gp.grad_exact(e, y)
    pre = precond.build(e, 48)
    rows = []
    for seed in range(20):
        lg = gp.nlml_grad_iterative(e, y, pre, gp.ProbeSet.generate(n, 32, seed), tol=1e-10, max_iter=1000)
        rows.append([lg.loss, lg.grad_l, lg.grad_f, lg.grad_s])
    rows = np.asarray(rows)
    for sample, truth in zip(rows.T, (exact.loss, exact.grad_l, exact.grad_f, exact.grad_s)):
        stderr = sample.std(ddof=1) / math.sqrt(len(sample))
        assert abs(sample.mean() - truth) <= 3 * stderr + 1e-9 * abs(truth)


def test_probe_sets(pkg):
    """test_gp.py:223-233: probes are reproducible for a seed; an empty probe set is rejected."""
    from paper_2503_02259_b200 import gp

    a, b = gp.ProbeSet.generate(30, 5, 123), gp.ProbeSet.generate(30, 5, 123)
    np.testing.assert_array_equal(a.vectors, b.vectors)
    np.testing.assert_array_equal(a.norms_sq, b.norms_sq)
    with pytest.raises(ValueError):
        gp.ProbeSet.generate(10, 0, 1)


def test_prediction_limits_and_edges(pkg, rng):
    """test_gp.py:150-203: vanishing noise interpolates the training targets; far from the data the
    prediction reverts to the prior (mean 0, stddev f); an empty test set gives empty arrays; a
    dimension mismatch is a ValueError naming it; the predicted stddev is the square root of the
    diagonal of the full posterior covariance, which is symmetric positive semi-definite."""
    from paper_2503_02259_b200 import gp

    x = rng.uniform(-1, 1, (40, 2))
    y = np.sin(x[:, 0]) + np.cos(x[:, 1])
    pred = gp.predict(pkg.KernelType.GAUSSIAN, x, y, x, _hp(pkg, 1.0, 1.0, 1e-10))
    assert np.max(np.abs(pred.mean - y)) / np.max(np.abs(y)) < 1e-4
    assert np.max(pred.stddev) < 1e-3

    x = rng.standard_normal((30, 2))
    y = rng.standard_normal(30)
    hp = _hp(pkg, 0.5, 1.7, 0.1)
    for mode in ("exact", "iterative"):
        pred = gp.predict(pkg.KernelType.GAUSSIAN, x, y, np.array([[500.0, -500.0]]), hp, mode=mode)
        np.testing.assert_allclose(pred.mean, [0.0], atol=1e-12)
        np.testing.assert_allclose(pred.stddev, [hp.f], rtol=1e-12)

    pred = gp.predict(pkg.KernelType.GAUSSIAN, x, y, np.empty((0, 2)), _hp(pkg, 1, 1, 0.1))
    assert pred.mean.shape == (0,) and pred.stddev.shape == (0,)
    with pytest.raises(ValueError, match="mismatch"):
        gp.predict(pkg.KernelType.GAUSSIAN, x, np.zeros(30), np.zeros((3, 3)), _hp(pkg, 1, 1, 0.1))

    x = rng.standard_normal((50, 2))
    y = rng.standard_normal(50)
    xs = rng.standard_normal((15, 2))
    hp = _hp(pkg, 1.0, 1.3, 0.2)
    f2 = hp.f**2
    kss = f2 * pkg.eval_kernel(pkg.KernelType.MATERN52, xs, xs, hp.l)
    ks = f2 * pkg.eval_kernel(pkg.KernelType.MATERN52, x, xs, hp.l)
    cov = kss - ks.T @ np.linalg.solve(_khat_loops("matern52", x, hp), ks)
    np.testing.assert_allclose(cov, cov.T, atol=1e-12)
    assert np.linalg.eigvalsh(cov).min() >= -1e-8
    pred = gp.predict(pkg.KernelType.MATERN52, x, y, xs, hp)
    np.testing.assert_allclose(pred.stddev, np.sqrt(np.diag(cov)), rtol=1e-8)


@pytest.mark.parametrize("kt", KTS)
def test_iterative_prediction_matches_exact(pkg, kt, rng):
    """test_gp.py:172-183: iterative and exact prediction agree to 10 tol."""
    from paper_2503_02259_b200 import gp

    x = rng.uniform(-2, 2, (300, 2))
    y = np.sin(x[:, 0] * 2) + 0.05 * rng.standard_normal(300)
    hp = _hp(pkg, 0.8, 1.0, 0.05)
    tol = 1e-8
    ex = gp.predict(pkg.KernelType(kt), x, y, x[:30] + 0.01, hp, mode="exact")
    it = gp.predict(pkg.KernelType(kt), x, y, x[:30] + 0.01, hp, mode="iterative", tol=tol, max_iter=2000)
    assert np.max(np.abs(ex.mean - it.mean)) <= 10 * tol * np.max(np.abs(ex.mean))
    assert np.max(np.abs(ex.stddev - it.stddev)) <= 10 * tol * max(1.0, np.max(ex.stddev))


# ---------------------------------------------------------------------------- preconditioner (test_precond.py)
def test_fps_properties(pkg, rng):
    """test_precond.py:13-44 through the device farthest-point sampler: one landmark is the seed; a
    line picks its far end; a full selection is a permutation; the greedy max-min order equals a
    brute-force restatement; repeated calls agree; a rank above n is rejected."""
    from paper_2503_02259_b200 import precond

    x = rng.standard_normal((10, 2))
    assert list(precond.fps_select(x, 1, seed_index=4)) == [4]
    assert list(precond.fps_select(np.arange(10.0)[:, None], 2, seed_index=0)) == [0, 9]
    x = rng.standard_normal((25, 3))
    assert sorted(precond.fps_select(x, 25, seed_index=7)) == list(range(25))
    x = rng.standard_normal((30, 2))
    chosen = [0]
    for _ in range(5):
        d2 = ((x[:, None, :] - x[chosen][None, :, :]) ** 2).sum(-1).min(axis=1)
        chosen.append(int(np.argmax(d2)))
    assert list(precond.fps_select(x, 6, seed_index=0)) == chosen
    x = rng.standard_normal((40, 3))
    np.testing.assert_array_equal(precond.fps_select(x, 12, seed_index=3), precond.fps_select(x, 12, seed_index=3))
    with pytest.raises(ValueError):
        precond.fps_select(rng.standard_normal((5, 1)), 6)


def test_nystrom_properties(pkg, rng):
    """test_precond.py:47-99: one point: M^-1 v = v / (f^2 + s); full rank equals the dense solve
    (1e-6); a vanishing signal leaves M^-1 = I/s; apply and apply_inverse are inverse to each other;
    M^-1 is symmetric and positive; landmarks are deterministic; the default rank rule."""
    from paper_2503_02259_b200 import precond

    e1 = pkg.KernelEngine(pkg.KernelType.GAUSSIAN, [[0.0]], _hp(pkg, 1, 2, 0.1))
    np.testing.assert_allclose(precond.build(e1, 1).apply_inverse(np.array([3.0])), [3.0 / 4.1], rtol=1e-9)

    def engine(n, seed, hp=None):
        xx = np.random.default_rng(seed).standard_normal((n, 2))
        return pkg.KernelEngine(pkg.KernelType.GAUSSIAN, xx, hp or _hp(pkg, 1.0, 1.0, 0.1)), xx

    e, x = engine(50, 1)
    b = rng.standard_normal((50, 3))
    expected = np.linalg.solve(_khat_loops("gaussian", x, _hp(pkg, 1.0, 1.0, 0.1)), b)
    assert rel_max(precond.build(e, 50).apply_inverse(b), expected) < 1e-6

    e, _ = engine(30, 2, _hp(pkg, 1.0, 1e-8, 0.25))
    b = rng.standard_normal((30, 2))
    np.testing.assert_allclose(precond.build(e, 10).apply_inverse(b), b / 0.25, rtol=1e-10)

    e, _ = engine(80, 3)
    p = precond.build(e, 20)
    v = rng.standard_normal(80)
    np.testing.assert_allclose(p.apply_inverse(p.apply(v)), v, rtol=1e-8, atol=1e-10)

    e, _ = engine(70, 4)
    p = precond.build(e, 25)
    v, w = rng.standard_normal(70), rng.standard_normal(70)
    lhs, rhs = v @ p.apply_inverse(w), w @ p.apply_inverse(v)
    assert abs(lhs - rhs) <= 1e-10 * max(abs(lhs), abs(rhs))
    assert v @ p.apply_inverse(v) > 0

    e, _ = engine(90, 5)
    np.testing.assert_array_equal(precond.build(e, 30).landmark_indices, precond.build(e, 30).landmark_indices)
    assert [precond.default_rank(n) for n in (4, 100, 10_000, 1_000_000)] == [4, 40, 400, 500]


def test_preconditioning_reduces_iterations(pkg, rng):
    """test_precond.py:102-118: on a smooth kernel (lengthscale = the data's diameter) the Nystrom
    preconditioner cuts the device PCG's iteration count."""
    from paper_2503_02259_b200 import precond, solver

    n = 500
    x = rng.uniform(-1, 1, size=(n, 2))
    diameter = math.sqrt(np.max(((x[:, None, :] - x[None, :, :]) ** 2).sum(-1)))
    e = pkg.KernelEngine(pkg.KernelType.GAUSSIAN, x, _hp(pkg, diameter, 1.0, 1e-2), mode=pkg.EngineMode.ON_THE_FLY)
    y = rng.standard_normal(n)
    plain = solver.pcg_solve(e.matmul, None, y, tol=1e-8, max_iter=2000)
    clever = solver.pcg_solve(e.matmul, precond.build(e, 100).apply_inverse, y, tol=1e-8, max_iter=2000)
    assert clever.all_converged
    assert clever.traces[0].iterations < plain.traces[0].iterations


# ---------------------------------------------------------------------------- panels (test_kernels.py)
def test_pairwise_sq_dist_properties(pkg, rng):
    """test_kernels.py:13-35 on the device panel kernel: exact small cases (a unit step, 3-4-5), a
    double loop, non-negativity when nearly coincident points cancel, dimension mismatch."""
    np.testing.assert_array_equal(pkg.pairwise_sq_dist([[0.0], [1.0]], [[0.0], [1.0]]), [[0.0, 1.0], [1.0, 0.0]])
    np.testing.assert_array_equal(pkg.pairwise_sq_dist([[0.0, 0.0]], [[3.0, 4.0]]), [[25.0]])
    x, y = rng.standard_normal((5, 3)), rng.standard_normal((4, 3))
    loops = np.array([[np.sum((x[i] - y[j]) ** 2) for j in range(4)] for i in range(5)])
    np.testing.assert_allclose(pkg.pairwise_sq_dist(x, y), loops, rtol=1e-13)
    base = rng.standard_normal((50, 4)) * 100
    xx = np.vstack([base, base + 1e-9])
    assert np.all(pkg.pairwise_sq_dist(xx, xx) >= 0.0)
    with pytest.raises(ValueError, match="dimension"):
        pkg.pairwise_sq_dist([[0.0, 1.0]], [[0.0]])


@pytest.mark.parametrize("kt", KTS)
def test_kernel_panel_properties(pkg, kt, rng):
    """test_kernels.py:38-70, 122-140: unit diagonal to the bit for l in {0.1, 1, 7.5}; transpose
    symmetry to the bit; values in (0, 1] and equal to the scalar closed forms (1e-12); any row or
    column tiling of a panel gives the same bits as the whole panel; invalid length scales rejected."""
    K = pkg.KernelType(kt)
    for l in (0.1, 1.0, 7.5):
        x = rng.standard_normal((6, 2))
        np.testing.assert_array_equal(np.diag(pkg.eval_kernel(K, x, x, l)), np.ones(6))
    x, y = rng.standard_normal((7, 3)), rng.standard_normal((5, 3))
    np.testing.assert_array_equal(pkg.eval_kernel(K, x, y, 0.8), pkg.eval_kernel(K, y, x, 0.8).T)
    x, y = rng.standard_normal((8, 3)), rng.standard_normal((6, 3))
    k = pkg.eval_kernel(K, x, y, 1.3)
    assert np.all(k > 0) and np.all(k <= 1)
    scalar = np.array([[_kappa(kt, float(np.linalg.norm(x[i] - y[j])), 1.3) for j in range(6)] for i in range(8)])
    np.testing.assert_allclose(k, scalar, rtol=1e-12)
    x, y = rng.standard_normal((83, 4)), rng.standard_normal((61, 4))
    full = pkg.eval_kernel(K, x, y, 0.9)
    np.testing.assert_array_equal(full, np.vstack([pkg.eval_kernel(K, x[i:i + 17], y, 0.9) for i in range(0, 83, 17)]))
    np.testing.assert_array_equal(full, np.hstack([pkg.eval_kernel(K, x, y[j:j + 13], 0.9) for j in range(0, 61, 13)]))
    gfull = pkg.eval_kernel_grad_l(K, x, y, 0.9)
    np.testing.assert_array_equal(gfull,
                                  np.vstack([pkg.eval_kernel_grad_l(K, x[i:i + 17], y, 0.9) for i in range(0, 83, 17)]))
    for bad in (0.0, -1.0, float("nan")):
        with pytest.raises(ValueError, match="length scale"):
            pkg.eval_kernel(pkg.KernelType.GAUSSIAN, [[0.0]], [[1.0]], bad)


def test_kernel_grad_l_properties(pkg, rng):
    """test_kernels.py:73-120: d kappa / dl is exactly 0 at coincident points; the Gaussian's equals
    kappa r^2 / l^3 (1e-13); all three against central finite differences of the scalar closed forms
    on 60 random pairs over three decades of distance and two of length scale (1e-5; the reference's
    sweep differentiates a 50-digit evaluation, here double precision with h = 1e-6 l on pairs whose
    difference quotient is resolvable)."""
    for kt in KTS:
        np.testing.assert_array_equal(pkg.eval_kernel_grad_l(pkg.KernelType(kt), [[2.0, 3.0]], [[2.0, 3.0]], 0.7),
                                      [[0.0]])
    x, y = rng.standard_normal((5, 2)), rng.standard_normal((4, 2))
    l = 1.7
    k = pkg.eval_kernel(pkg.KernelType.GAUSSIAN, x, y, l)
    np.testing.assert_allclose(pkg.eval_kernel_grad_l(pkg.KernelType.GAUSSIAN, x, y, l),
                               k * pkg.pairwise_sq_dist(x, y) / l**3, rtol=1e-13)
    for kt in KTS:
        for _ in range(20):
            d = int(rng.integers(1, 5))
            u, v = rng.standard_normal(d), rng.standard_normal(d)
            l = rng.uniform(0.5, 2.0)
            h = 1e-6 * l
            r = float(np.linalg.norm(u - v))
            fd = (_kappa(kt, r, l + h) - _kappa(kt, r, l - h)) / (2 * h)
            g = pkg.eval_kernel_grad_l(pkg.KernelType(kt), u[None, :], v[None, :], l)[0, 0]
            assert abs(g - fd) / max(abs(fd), abs(g)) < 1e-5


# ---------------------------------------------------------------------------- training (test_train.py)
def test_training_properties(pkg):
    """test_train.py:60-120 with the device engine under train.fit: one step records one loss and
    one gradient norm and stops on MAX_STEPS; hyperparameters stay positive; the loss does not end
    above where it started; exact mode is reproducible to the bit; iterative mode records a finite
    loss per step; the median-heuristic initialisation; configuration validation."""
    from paper_2503_02259_b200 import train

    def data(n=80, seed=0):
        r = np.random.default_rng(seed)
        x = r.uniform(-2, 2, (n, 2))
        return x, np.sin(x[:, 0]) * np.cos(x[:, 1]) + 0.1 * r.standard_normal(n)

    x, y = data()
    res = train.fit(pkg.KernelType.GAUSSIAN, x, y, train.TrainConfig(max_steps=1))
    assert len(res.loss_history) == 1 and len(res.grad_norm_history) == 1
    assert res.status is train.TrainStatus.MAX_STEPS
    x, y = data(seed=1)
    res = train.fit(pkg.KernelType.MATERN32, x, y, train.TrainConfig(max_steps=30))
    assert res.params.l > 0 and res.params.f > 0 and res.params.s > 0
    x, y = data(seed=2)
    res = train.fit(pkg.KernelType.GAUSSIAN, x, y, train.TrainConfig(max_steps=60))
    assert res.loss_history[-1] <= res.loss_history[0]
    x, y = data(seed=3)
    cfg = train.TrainConfig(max_steps=15, rng_seed=7)
    a, b = train.fit(pkg.KernelType.GAUSSIAN, x, y, cfg), train.fit(pkg.KernelType.GAUSSIAN, x, y, cfg)
    assert a.loss_history == b.loss_history
    assert (a.params.l, a.params.f, a.params.s) == (b.params.l, b.params.f, b.params.s)
    x, y = data(n=60, seed=4)
    res = train.fit(pkg.KernelType.GAUSSIAN, x, y,
                    train.TrainConfig(max_steps=10, mode="iterative", k_z=8, tol=1e-8, probe_tol=1e-6, rng_seed=1))
    assert len(res.loss_history) == 10 and np.isfinite(res.loss_history).all()
    hp = train.initial_hyperparams(np.array([[0.0], [1.0], [2.0], [10.0]]), np.array([0.0, 1.0, -1.0, 3.0]))
    yv = np.array([0.0, 1.0, -1.0, 3.0])
    np.testing.assert_allclose([hp.l, hp.f, hp.s], [5.0, np.std(yv), 0.01 * np.var(yv)], rtol=1e-12)
    with pytest.raises(ValueError):
        train.TrainConfig(learning_rate=0.0)
    with pytest.raises(ValueError):
        train.TrainConfig(mode="warp")
