"""CPU-only checks of the boundary and the host logic (no compute calls without a GPU)."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import REPO


def test_library_loads_and_exports_every_header_symbol():
    from paper_2503_02259_b200 import _lib

    lib = _lib.load()
    header = open(os.path.join(REPO, "include", "kgp.h")).read()
    declared = set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(kgp_\w+)\s*\(", header, re.M))
    assert declared, "no declarations parsed"
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(_lib.EXPORTED), declared ^ set(_lib.EXPORTED)
    assert lib.kgp_version() == 1


def test_error_codes_map_to_reference_exceptions():
    from paper_2503_02259_b200 import _lib
    from paper_2503_02259_b200.errors import BreakdownError, KernelGpError, NumericalError, ResourceLimitError

    lib = _lib.load()
    # an invalid call fails in argument validation, before touching a device
    rc = lib.kgp_fps(0, 1, None, 1, 0, None, None)
    assert rc == _lib.ERR_INVALID
    assert "1 <= m <= n" in _lib.last_error()
    with pytest.raises(ValueError):
        _lib.check(rc)
    for code, exc in ((2, ResourceLimitError), (3, BreakdownError), (4, NumericalError), (6, KernelGpError)):
        with pytest.raises(exc):
            _lib.check(code)
    assert issubclass(BreakdownError, NumericalError)


def test_double_destroy_is_an_error_not_a_crash():
    from paper_2503_02259_b200 import _lib

    lib = _lib.load()
    assert lib.kgp_engine_destroy(ctypes.c_void_p(12345)) == _lib.ERR_STATE
    assert lib.kgp_precond_destroy(None) == _lib.ERR_STATE


def test_engine_argument_validation_without_gpu():
    from paper_2503_02259_b200 import _lib

    lib = _lib.load()
    h = ctypes.c_void_p()
    x = np.zeros((4, 2))
    assert lib.kgp_engine_create(ctypes.byref(h), 0, 7, 0, 4, 2, x.ctypes.data, 0, 1.0, 1.0, 1.0, None) == 1
    assert lib.kgp_engine_create(ctypes.byref(h), 0, 0, 0, 4, 2, x.ctypes.data, 0, -1.0, 1.0, 1.0, None) == 1
    assert "length" in _lib.last_error() or "hyperparameter l" in _lib.last_error()


def test_hyperparams_and_train_helpers():
    from paper_2503_02259_b200 import train
    from paper_2503_02259_b200.kmat import Hyperparams

    for bad in (dict(l=0), dict(f=-1), dict(s=0), dict(l=np.nan)):
        args = dict(l=1.0, f=1.0, s=1.0)
        args.update(bad)
        with pytest.raises(ValueError):
            Hyperparams(**args)
    hp = Hyperparams(l=0.37, f=2.4, s=1e-5)
    back = train.RawParams.from_hyperparams(hp).to_hyperparams()
    np.testing.assert_allclose([back.l, back.f, back.s], [hp.l, hp.f, hp.s], rtol=1e-12)
    np.testing.assert_allclose(train.RawParams(0, 0, 0).to_hyperparams().l, np.log(2.0), rtol=1e-15)
    adam = train.Adam(0.1)
    np.testing.assert_allclose(adam.step(np.zeros(3), np.array([5.0, -2.0, 0.5])), [-0.1, 0.1, -0.1], rtol=1e-6)
    with pytest.raises(ValueError):
        train.TrainConfig(mode="bogus")


def test_train_helpers_match_reference_golden():
    """softplus/Adam host arithmetic against the reference run's recorded trajectory inputs."""
    from paper_2503_02259_b200 import train

    rho = np.array([-40.0, -1.0, 0.0, 1.0, 40.0])
    np.testing.assert_allclose(train.softplus(rho), np.log1p(np.exp(rho)), rtol=1e-12)
    np.testing.assert_allclose(train.softplus_inv(train.softplus(rho[1:4])), rho[1:4], rtol=1e-12)
    np.testing.assert_allclose(train.sigmoid(rho), 1 / (1 + np.exp(-rho)), rtol=1e-12)


def test_workload_shapes():
    from paper_2503_02259_b200 import workloads

    w = workloads.cfg2(n=1024)
    assert w.x.shape == (1024, 8) and w.z.shape == (1024, 32)
    assert np.array_equal(w.x, w.x.astype(np.float32).astype(np.float64))  # fp32-representable
    w = workloads.cfg3(n=512)
    assert w.kernel == "matern32" and w.x.shape == (512, 4) and w.k_z == 32
    w = workloads.cfg5(n=256, m_test=64)
    assert w.extra["xstar"].shape == (64, 2)


def test_lazy_exports_match_reference_surface():
    import paper_2503_02259_b200 as p

    ref_names = {"KernelType", "pairwise_sq_dist", "eval_kernel", "eval_kernel_grad_l", "Hyperparams", "Theta",
                 "EngineMode", "KernelEngine", "fps_select", "NystromPreconditioner", "CgTrace", "SolveReport",
                 "cg_solve", "pcg_solve", "build_tridiag", "slq_logdet", "LossGrad", "Prediction", "ProbeSet",
                 "nlml_exact", "grad_exact", "nlml_grad_iterative", "predict", "RawParams", "TrainConfig",
                 "TrainResult", "fit"}
    # north-star additions beyond kernelgp/__init__.py:16-44: AFN, and HiGP's Listing-1 GPR
    # problem API
    extensions = {"AFNPreconditioner", "GPRProblem", "GPRModel", "GPROptions", "gpr_prediction"}
    assert set(p.__all__) == ref_names | extensions
    for name in ref_names:
        getattr(p, name)


def test_build_tridiag_and_bands():
    from paper_2503_02259_b200 import solver

    t = solver.build_tridiag(solver.CgTrace(np.array([2.0]), np.array([0.1]), 1, 0.0))
    np.testing.assert_allclose(t, [[0.5]], rtol=1e-15)
    a, b = np.array([2.0, 4.0]), np.array([0.25, 0.5])
    t = solver.build_tridiag(solver.CgTrace(a, b, 2, 0.0))
    np.testing.assert_allclose(t, [[0.5, 0.25], [0.25, 0.25 + 0.125]], rtol=1e-15)
    with pytest.raises(ValueError):
        solver.build_tridiag(solver.CgTrace(np.array([-1.0]), np.array([0.1]), 1, 0.0))
    with pytest.raises(ValueError):
        solver.slq_logdet([], [])


def test_row_range_alignment():
    """Row blocks of the fused all-gather operator start on column-block (32-row) boundaries
    and still cover [0, n) in order; align=1 is the plain balanced split."""
    from paper_2503_02259_b200 import dist as kdist

    for n, world in ((3000, 3), (4100, 2), (65536, 8), (100, 8)):
        rs = [kdist.row_range(n, world, q, 32) for q in range(world)]
        assert rs[0][0] == 0 and rs[-1][1] == n
        assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
        assert all(r0 % 32 == 0 for r0, _ in rs)
        assert [kdist.row_range(n, world, q) for q in range(world)] == [
            (q * n // world, (q + 1) * n // world) for q in range(world)]


def test_gpr_setup_host_contract():
    """SPEC.md:523-528 / 546-547: setup copies the data (no aliasing), a label-length mismatch
    raises, empty test_x gives empty arrays, releasing twice is a no-op (never a crash).
    No device work happens in setup, so this runs on the CPU."""
    from paper_2503_02259_b200 import gpr

    rng = np.random.default_rng(0)
    x, y = rng.standard_normal((10, 2)), rng.standard_normal(10)
    prob = gpr.setup(data=x, label=y, kernel_type="gaussian")
    x[0, 0] = 99.0
    y[0] = 99.0
    assert prob.x[0, 0] != 99.0 and prob.y[0] != 99.0 and prob.n == 10
    assert not prob.x.flags.writeable
    with pytest.raises(ValueError, match="mismatch"):
        gpr.setup(data=x, label=y[:9])
    with pytest.raises(ValueError):
        gpr.setup(data=x, label=y, mode="bogus")
    pred = gpr.gpr_prediction(x, y, np.empty((0, 2)), "gaussian", (1.0, 1.0, 0.1))
    assert pred.prediction_mean.shape == (0,) and pred.prediction_stddev.shape == (0,)
    assert prob.release() is True
    assert prob.release() is False
