"""GPU tests of the Dirichlet GP classification path (gpc.py, kgp_gpc_nlml_grad,
kgp_engine_set_diag, kgp_pcg_grouped).

No reference GPC exists, so the checks are against the numpy statement in
tests/gpc_ref.py: the dense loss/gradient (1e-9), and the iterative path against the
dense same-probe estimator (1e-6, the FP64-mode bar; the reference makes the same
iterative-vs-dense-with-the-same-probes comparison for GPR, test_gp.py:104-119).
"""

import numpy as np
import pytest

from conftest import rel_max

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2503_02259_b200 as p

    return p


def _data(n=400, d=2, c=3, seed=0):
    from paper_2503_02259_b200 import gpc

    x = np.random.default_rng(seed).uniform(0.0, 1.0, (n, d))
    lab = gpc.sample_latent_labels(x, c, l=0.3, seed=seed)
    return x, lab


def test_engine_diag_matmul(pkg):
    import torch

    from oracle import kgp_oracle as orc
    from paper_2503_02259_b200 import _lib, gpc

    x, lab = _data()
    prob = gpc.setup(x, lab)
    l, f, s = 0.3, 1.2, 0.05
    e = pkg.KernelEngine(pkg.KernelType.MATERN52, x, pkg.Hyperparams(l=l, f=f, s=s), precision="fp64")
    b = np.random.default_rng(2).standard_normal((400, 5))
    cmap = [2, 0, 1, 1, 0]
    dn = torch.from_numpy(prob.noise).cuda()
    import ctypes

    _lib.call("kgp_engine_set_diag", e.handle, 3, dn.data_ptr(), 5, (ctypes.c_int32 * 5)(*cmap), None)
    got = e.matmul(b)
    kh = orc.khat_dense("matern52", x, l, f, s)
    want = kh @ b + prob.noise[cmap].T * b
    assert rel_max(got, want) <= 1e-12
    # derivative outputs ignore the diagonal
    assert rel_max(e.grad_matmul(pkg.Theta.F, b), 2 * f * orc.eval_kernel("matern52", x, x, l) @ b) <= 1e-12
    with pytest.raises(ValueError):
        e.matmul(np.ones((400, 6)))  # more columns than the map covers
    _lib.call("kgp_engine_set_diag", e.handle, 0, None, 0, None, None)
    assert rel_max(e.matmul(b), kh @ b) <= 1e-12


@pytest.mark.parametrize("kt", ["gaussian", "matern32"])
def test_gpc_exact_matches_numpy(pkg, kt):
    import gpc_ref
    from paper_2503_02259_b200 import gpc

    x, lab = _data()
    prob = gpc.setup(x, lab)
    l, f, s = 0.25, 1.1, 0.02
    e = pkg.KernelEngine(pkg.KernelType(kt), x, pkg.Hyperparams(l=l, f=f, s=s), precision="fp64")
    got = gpc.grad_exact(e, prob)
    loss, g = gpc_ref.exact(kt, x, prob.targets, prob.noise, l, f, s)
    np.testing.assert_allclose([got.loss, got.grad_l, got.grad_f, got.grad_s], [loss, *g], rtol=1e-9)


@pytest.mark.parametrize("kind", ["afn", "none"])
def test_gpc_iterative_matches_same_probe_estimator(pkg, kind):
    import gpc_ref
    from paper_2503_02259_b200 import gpc

    x, lab = _data()
    prob = gpc.setup(x, lab)
    l, f, s = 0.25, 1.1, 0.02
    e = pkg.KernelEngine(pkg.KernelType.MATERN32, x, pkg.Hyperparams(l=l, f=f, s=s), precision="fp64")
    probes = gpc.generate_probes(400, 3, 8, 5)
    pcs = gpc.build_preconditioners(e, prob, 40, kind, fsai_npt=8)
    lg = gpc.nlml_grad_iterative(e, prob, pcs, probes, tol=1e-10, max_iter=2000, probe_tol=1e-10)
    loss, g = gpc_ref.estimator("matern32", x, prob.targets, prob.noise, l, f, s, probes)
    got = np.array([lg.loss, lg.grad_l, lg.grad_f, lg.grad_s])
    ref = np.array([loss, *g])
    assert lg.converged
    assert np.all(np.abs(got - ref) <= 1e-6 * np.abs(ref)), (got, ref)
    # the engine's diagonal is cleared afterwards
    b = np.ones((400, 2))
    assert rel_max(e.matmul(b), pkg.KernelEngine(pkg.KernelType.MATERN32, x, e.params, precision="fp64").matmul(b)) \
        <= 1e-14


def test_gpc_predict(pkg):
    import torch

    from oracle import kgp_oracle as orc
    from paper_2503_02259_b200 import gpc

    x, lab = _data()
    prob = gpc.setup(x, lab)
    hp = pkg.Hyperparams(l=0.25, f=1.1, s=0.02)
    xs = np.random.default_rng(9).uniform(0.0, 1.0, (50, 2))
    ex = gpc.predict(pkg.KernelType.GAUSSIAN, prob, xs, hp, mode="exact", precision="fp64")
    it = gpc.predict(pkg.KernelType.GAUSSIAN, prob, xs, hp, mode="iterative", tol=1e-10, rank=40,
                     precision="fp64")
    kb = orc.khat_dense("gaussian", x, hp.l, hp.f, hp.s)
    cross = hp.f ** 2 * orc.eval_kernel("gaussian", xs, x, hp.l)
    for c in range(3):
        kc = kb + np.diag(prob.noise[c])
        mean = cross @ np.linalg.solve(kc, prob.targets[c]) + prob.means[c]
        var = hp.f ** 2 - np.einsum("ij,ji->i", cross, np.linalg.solve(kc, cross.T))
        assert rel_max(ex.mean[:, c], mean) <= 1e-10
        assert rel_max(ex.variance[:, c], var) <= 1e-8
        assert rel_max(it.mean[:, c], mean) <= 1e-7
    np.testing.assert_allclose(ex.probabilities.sum(axis=1), 1.0, rtol=1e-12)
    np.testing.assert_array_equal(ex.labels, np.argmax(ex.mean, axis=1))
    # the latent-mean classifier reproduces most training labels on its own data
    tr = gpc.predict(pkg.KernelType.GAUSSIAN, prob, x, hp, mode="exact", precision="fp64")
    assert (tr.labels == lab).mean() > 0.9


def test_gpc_fit_runs(pkg):
    from paper_2503_02259_b200 import gpc

    x, lab = _data(n=600)
    prob = gpc.setup(x, lab)
    res = gpc.fit(pkg.KernelType.GAUSSIAN, prob, pkg.Hyperparams(l=0.5, f=1.0, s=0.1), steps=4, k_z=8, rank=50,
                  tol=1e-8, max_iter=1000, probe_tol=1e-6, precision="fp64")
    assert len(res.loss_history) == 4 and np.all(np.isfinite(res.loss_history))
    assert res.params.l > 0 and res.params.f > 0 and res.params.s > 0
    assert res.loss_history[-1] < res.loss_history[0]


def test_gpc_preconditioned_probes_estimator(pkg):
    """Per-class AFN draws z_c ~ N(0, M_c): the device estimator equals the dense same-probe
    formula (sum over classes of the GPR preconditioned estimator), 1e-6."""
    from oracle import kgp_oracle as orc
    from paper_2503_02259_b200 import gpc

    x, lab = _data()
    prob = gpc.setup(x, lab)
    l, f, s = 0.25, 1.1, 0.02
    e = pkg.KernelEngine(pkg.KernelType.MATERN32, x, pkg.Hyperparams(l=l, f=f, s=s), precision="fp64")
    probes = gpc.generate_probes(400, 3, 4, 7)
    pcs = gpc.build_preconditioners(e, prob, 40, "afn", fsai_npt=8)
    lg = gpc.nlml_grad_iterative(e, prob, pcs, probes, tol=1e-11, max_iter=2000, probe_tol=1e-11,
                                 preconditioned_probes=True)
    n = 400
    kap = orc.eval_kernel("matern32", x, x, l)
    kb = f * f * kap + s * np.eye(n)
    dks = [f * f * orc.eval_kernel_grad_l("matern32", x, x, l), 2 * f * kap, np.eye(n)]
    loss, g = 0.0, np.zeros(3)
    for c in range(3):
        kh = kb + np.diag(prob.noise[c])
        m = np.linalg.inv(pcs[c].apply_inverse(np.eye(n)))
        m = 0.5 * (m + m.T)
        z = pcs[c].sample(probes[c * 4:(c + 1) * 4].T).cpu().numpy().T
        ev, vec = np.linalg.eigh(m)
        mh = (vec / np.sqrt(ev)) @ vec.T
        ea, va = np.linalg.eigh(mh @ kh @ mh)
        zh = mh @ z
        w = np.linalg.solve(kh, prob.targets[c])
        loss += 0.5 * (prob.targets[c] @ w + pcs[c].logdet + np.einsum("ij,ij->", zh, ((va * np.log(ea)) @ va.T) @ zh)
                       / 4 + n * np.log(2 * np.pi))
        u = np.linalg.solve(kh, z)
        mz = np.linalg.solve(m, z)
        for i, dk in enumerate(dks):
            g[i] += 0.5 * (-w @ dk @ w + np.einsum("ij,ij->", mz, dk @ u) / 4)
    got = np.array([lg.loss, lg.grad_l, lg.grad_f, lg.grad_s])
    ref = np.array([loss, *g])
    assert lg.converged
    assert np.all(np.abs(got - ref) <= 1e-6 * np.abs(ref)), (got, ref)
