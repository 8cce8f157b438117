"""GPU tests of the AFN preconditioner (afn.cu + precond.build_afn).

AFN has no reference implementation, so:
* the device factors/applications are checked against the numpy statement of the same
  algorithm (tests/afn_ref.py): knn pattern exact, M^-1 B to 1e-8 of max|ref|
  (different Cholesky/TRSM rounding: cuSOLVER vs LAPACK);
* the solves it preconditions are pinned to the reference: converged PCG solutions and
  tolerance-mode NLML/gradient against the reference's golden values (<= 1e-6, the
  FP64-mode bar), with AFN replacing the Nystrom preconditioner of the w-solve;
* its purpose is checked by iteration counts against Nystrom at equal rank.
"""

import os

import numpy as np
import pytest

from conftest import golden, rel_max

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2503_02259_b200 as p

    return p


def _problem(kt, n, d, l, s, seed=0):
    rng = np.random.default_rng(seed)
    x = rng.uniform(0.0, 1.0, (n, d))
    y = np.sin(3.0 * x).sum(axis=1) + 0.05 * rng.standard_normal(n)
    return x, y


def test_knn_prev_matches_numpy(pkg):
    import torch

    import afn_ref
    from paper_2503_02259_b200 import precond

    for d, npt in ((1, 5), (3, 12), (8, 40)):
        x = np.random.default_rng(d).uniform(0.0, 1.0, (700, d))
        got = precond.knn_prev_device(torch.from_numpy(x).cuda(), npt).cpu().numpy()
        np.testing.assert_array_equal(got, afn_ref.knn_prev(x, npt))


def test_knn_prev_ties_to_lower_index(pkg):
    import torch

    from paper_2503_02259_b200 import precond

    x = np.zeros((6, 2))  # all coincident: every earlier point ties at distance 0
    got = precond.knn_prev_device(torch.from_numpy(x).cuda(), 3).cpu().numpy()
    want = np.array([[-1, -1, -1], [0, -1, -1], [0, 1, -1], [0, 1, 2], [0, 1, 2], [0, 1, 2]])
    np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("kt", ["gaussian", "matern32", "matern52"])
def test_afn_apply_matches_numpy(pkg, kt):
    import afn_ref
    from paper_2503_02259_b200 import precond

    x, _ = _problem(kt, 900, 3, 0.2, 1e-3)
    l, f, s = 0.2, 1.3, 1e-3
    e = pkg.KernelEngine(pkg.KernelType(kt), x, pkg.Hyperparams(l=l, f=f, s=s))
    pre = precond.build_afn(e, 64, fsai_npt=10)
    ref = afn_ref.AFN(kt, x, l, f, s, 64, 10)
    np.testing.assert_array_equal(pre.landmark_indices, ref.perm[:64])
    b = np.random.default_rng(1).standard_normal((900, 5))
    assert rel_max(pre.apply_inverse(b), ref.apply_inverse(b)) <= 1e-8
    # 1-D in, 1-D out; strided device input
    assert rel_max(pre.apply_inverse(b[:, 2]), ref.apply_inverse(b[:, 2])) <= 1e-8
    # run-to-run bitwise determinism (no atomics in the application)
    np.testing.assert_array_equal(pre.apply_inverse(b), pre.apply_inverse(b))
    # k > 8: the point-major application (transposed cuBLAS products, coalesced G gathers)
    b12 = np.random.default_rng(2).standard_normal((900, 12))
    assert rel_max(pre.apply_inverse(b12), ref.apply_inverse(b12)) <= 1e-8
    np.testing.assert_array_equal(pre.apply_inverse(b12), pre.apply_inverse(b12))


@pytest.mark.parametrize("n,m,k", [(900, 64, 9), (900, 130, 17), (900, 64, 33), (1337, 130, 40),
                                   (900, 66, 51), (900, 64, 64), (6000, 512, 33), (900, 63, 33)])
def test_afn_apply_wide_blocks(pkg, n, m, k):
    """Point-major application with the DMMA W products (wgemm.cu): ragged row counts, landmark
    counts off the 32/64-element tiles (odd m takes the cuBLAS path), every column-tile count
    1..8, several row splits and staged chunks; against the numpy statement of the same
    algebra, deterministic run to run."""
    import afn_ref
    from paper_2503_02259_b200 import precond

    x, _ = _problem("matern32", n, 3, 0.2, 1e-3)
    l, f, s = 0.2, 1.3, 1e-3
    e = pkg.KernelEngine(pkg.KernelType.MATERN32, x, pkg.Hyperparams(l=l, f=f, s=s))
    pre = precond.build_afn(e, m, fsai_npt=10)
    ref = afn_ref.AFN("matern32", x, l, f, s, m, 10)
    b = np.random.default_rng(k).standard_normal((n, k))
    want = ref.apply_inverse(b)
    # default dispatch (DMMA streams for 33..40 columns), then forced for every width
    for mode in ("1", "2"):
        os.environ["KGP_AFN_WGEMM"] = mode
        try:
            got = pre.apply_inverse(b)
            assert rel_max(got, want) <= 1e-8, mode
            np.testing.assert_array_equal(got, pre.apply_inverse(b))
        finally:
            del os.environ["KGP_AFN_WGEMM"]


def test_afn_preconditioned_pcg(pkg):
    """High-rank Matern problem: AFN cuts PCG iterations vs Nystrom at equal rank, and the
    converged solution matches the dense solve."""
    from oracle import kgp_oracle as orc
    from paper_2503_02259_b200 import precond, solver

    kt, n, l, s = "matern32", 3000, 0.2, 1e-3
    x, y = _problem(kt, n, 4, l, s)
    e = pkg.KernelEngine(pkg.KernelType(kt), x, pkg.Hyperparams(l=l, f=1.0, s=s))
    afn = precond.build_afn(e, 128, fsai_npt=16)
    nys = precond.build(e, 128)
    rep_a = solver.pcg_solve(e.matmul, afn.apply_inverse, y, tol=1e-8, max_iter=3000)
    rep_n = solver.pcg_solve(e.matmul, nys.apply_inverse, y, tol=1e-8, max_iter=3000)
    it_a, it_n = rep_a.iteration_counts()[0], rep_n.iteration_counts()[0]
    assert rep_a.converged[0] and rep_n.converged[0]
    assert it_a * 4 <= it_n, (it_a, it_n)  # numpy statement: 26 vs 273
    ref = np.linalg.solve(orc.khat_dense(kt, x, l, 1.0, s), y)
    assert rel_max(rep_a.solution, ref) <= 1e-5
    # rep_a ran the device driver (kgp_pcg with the AFN handle); the host-loop PCG over the
    # same application (a non-method callable) agrees
    gen = solver.pcg_solve(e.matmul, lambda b: afn.apply_inverse(b), y, tol=1e-8, max_iter=3000)
    assert gen.converged[0] and abs(gen.iteration_counts()[0] - it_a) <= 2
    assert rel_max(gen.solution, ref) <= 1e-5


@pytest.mark.parametrize("kt", ["matern32", "matern52"])
def test_afn_nlml_matches_reference(pkg, kt):
    """Tolerance-mode NLML+gradient with AFN in the w-solve equals the reference's
    (Nystrom-preconditioned) golden result within the FP64 bar."""
    from paper_2503_02259_b200 import gp, precond

    g = golden("nlml.npz")
    e = pkg.KernelEngine(pkg.KernelType(kt), g[f"{kt}_x"], pkg.Hyperparams(l=0.25, f=1.5, s=1e-2))
    pre = precond.build_afn(e, 40, fsai_npt=16)
    lg = gp.nlml_grad_iterative(e, g[f"{kt}_y"], pre, gp.ProbeSet(g[f"{kt}_probes"]),
                                tol=1e-10, max_iter=3000, probe_tol=1e-10)
    got = np.array([lg.loss, lg.grad_l, lg.grad_f, lg.grad_s])
    ref = g[f"{kt}_res"]
    assert np.all(np.abs(got - ref) <= 1e-6 * np.abs(ref)), (got, ref)


def test_build_adaptive_choice(pkg):
    from paper_2503_02259_b200 import precond, workloads

    w = workloads.cfg1(n=2048)  # smooth Gaussian, l=0.3: numerically low rank
    e = pkg.KernelEngine(pkg.KernelType.GAUSSIAN, w.x, pkg.Hyperparams(l=w.l, f=w.f, s=w.s))
    assert isinstance(precond.build_adaptive(e, 256), precond.NystromPreconditioner)
    x, _ = _problem("matern32", 2048, 4, 0.2, 1e-3)
    e = pkg.KernelEngine(pkg.KernelType.MATERN32, x, pkg.Hyperparams(l=0.2, f=1.0, s=1e-3))
    assert isinstance(precond.build_adaptive(e, 128), precond.AFNPreconditioner)


def test_afn_errors(pkg):
    from paper_2503_02259_b200 import precond

    x, _ = _problem("gaussian", 100, 2, 0.3, 1e-2)
    e = pkg.KernelEngine(pkg.KernelType.GAUSSIAN, x, pkg.Hyperparams(l=0.3, f=1.0, s=1e-2))
    with pytest.raises(ValueError):
        precond.build_afn(e, 100)
    with pytest.raises(ValueError):
        precond.build_afn(e, 10, fsai_npt=65)
    pre = precond.build_afn(e, 10, fsai_npt=4)
    with pytest.raises(ValueError):
        pre.apply_inverse(np.ones(99))


def test_afn_sampling_and_logdet(pkg):
    """kgp_afn_sample draws exactly N(0, M) (covariance of the linear map = M) and
    AFNPreconditioner.logdet = log|M|, M = (the application's inverse)^-1."""
    from paper_2503_02259_b200 import precond

    x, _ = _problem("matern32", 500, 3, 0.2, 1e-3)
    e = pkg.KernelEngine(pkg.KernelType.MATERN32, x, pkg.Hyperparams(l=0.2, f=1.1, s=1e-3))
    pre = precond.build_afn(e, 40, fsai_npt=8)
    minv = pre.apply_inverse(np.eye(500))
    m = np.linalg.inv(minv)
    z = pre.sample(np.eye(500)).cpu().numpy()            # row r = L F e_r
    np.testing.assert_allclose(z.T @ z, m, atol=1e-8 * np.abs(m).max())
    assert abs(pre.logdet - np.linalg.slogdet(m)[1]) <= 1e-9 * abs(pre.logdet)


def test_afn_preconditioned_probes_estimator(pkg):
    """preconditioned_probes=True with AFN equals its dense same-probe formula."""
    from oracle import kgp_oracle as orc
    from paper_2503_02259_b200 import gp, precond

    n, kt, l, f, s = 300, "matern52", 0.2, 1.2, 5e-3
    x, y = _problem(kt, n, 2, l, s, seed=4)
    e = pkg.KernelEngine(pkg.KernelType(kt), x, pkg.Hyperparams(l=l, f=f, s=s))
    pre = precond.build_afn(e, 30, fsai_npt=10)
    probes = gp.ProbeSet.generate(n, 5, 9)
    lg = gp.nlml_grad_iterative(e, y, pre, probes, tol=1e-11, max_iter=3000, probe_tol=1e-11,
                                preconditioned_probes=True)
    z = pre.sample(probes.vectors).cpu().numpy().T
    kh = orc.khat_dense(kt, x, l, f, s)
    m = np.linalg.inv(pre.apply_inverse(np.eye(n)))
    m = 0.5 * (m + m.T)
    ev, vec = np.linalg.eigh(m)
    mh = (vec / np.sqrt(ev)) @ vec.T
    ea, va = np.linalg.eigh(mh @ kh @ mh)
    loga = (va * np.log(ea)) @ va.T
    zh = mh @ z
    w = np.linalg.solve(kh, y)
    loss = 0.5 * (y @ w + pre.logdet + np.einsum("ij,ij->", zh, loga @ zh) / 5 + n * np.log(2 * np.pi))
    kap = orc.eval_kernel(kt, x, x, l)
    dks = [f * f * orc.eval_kernel_grad_l(kt, x, x, l), 2 * f * kap, np.eye(n)]
    u = np.linalg.solve(kh, z)
    mz = np.linalg.solve(m, z)
    grads = [0.5 * (-w @ dk @ w + np.einsum("ij,ij->", mz, dk @ u) / 5) for dk in dks]
    got = np.array([lg.loss, lg.grad_l, lg.grad_f, lg.grad_s])
    ref = np.array([loss, *grads])
    assert lg.converged
    assert np.all(np.abs(got - ref) <= 1e-6 * np.abs(ref)), (got, ref)
