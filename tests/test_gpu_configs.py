"""Parity at the BASELINE.json configuration sizes (configs[2..4]) and on configs[2]'s
generator through the reference's own estimator.

* Operator (kmat.py:165-189) at FULL n: Khat.Z and dKhat/dl.Z of the device engine on
  sampled rows against the C oracle (oracle/kgp_oracle.c, the reference's streamed operator
  restated, pinned to the reference's goldens in tests/test_oracle.py). The fast (3xTF32)
  product is computed for ALL rows exactly as a solver would (full column sweep, the
  launch's own column split), then subsampled; fp64 computes only the sampled row blocks.
  Bars: fp64 <= 1e-12 of max|ref| (test_kmat.py:49); fast Khat.Z <= 2e-5 and dKhat/dl.Z
  <= 2e-4 (the same bars as the cfg2 test).
* NLML + gradient (gp.py:133-179) on configs[2]'s generator at n = 16384 (or 8192) (Matern-3/2, d=4,
  l=0.2, f=1.5, s=1e-3, 32 probes, Nystrom rank 1024), tolerance mode tol = probe_tol =
  1e-10, against tests/golden/cfg3_small.npz made by the unmodified reference
  (make_golden.py cfg3). Bars: fp64 operator <= 1e-6 relative (north star FP64 mode), fast
  operator <= 1e-3 (north star tensor-core mode).
"""

import numpy as np
import pytest

from conftest import golden, rel_max

pytestmark = pytest.mark.gpu

# (name, kernel, n, d, k, l, f, s, generator) -- workloads.cfg3/cfg4/cfg5 shapes
CONFIGS = {
    "cfg3": ("matern32", 262144, 4, 33),
    "cfg4": ("gaussian", 131072, 8, 51),
    "cfg5": ("matern52", 1048576, 2, 64),
}
ROW_BLOCKS = 2
ROWS_PER_BLOCK = 256


@pytest.fixture(scope="module")
def pkg():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2503_02259_b200 as p

    return p


_CACHE = {}


def _problem(name):
    """Seeded inputs (workloads.*), the sampled row blocks and the C-oracle outputs there."""
    if name in _CACHE:
        return _CACHE[name]
    from oracle import kgp_oracle_c as oc
    from paper_2503_02259_b200 import workloads

    kt, n, d, k = CONFIGS[name]
    w = {"cfg3": workloads.cfg3, "cfg4": workloads.cfg4, "cfg5": lambda n: workloads.cfg5(n=n, m_test=1)}[name](n=n)
    assert w.x.shape == (n, d) and w.kernel == kt
    rng = np.random.default_rng(1000 + n)
    z = rng.standard_normal((n, k))
    starts = np.sort(rng.choice(n // ROWS_PER_BLOCK, ROW_BLOCKS, replace=False)) * ROWS_PER_BLOCK
    starts[-1] = n - ROWS_PER_BLOCK  # include the ragged end of the column sweep's last rows
    refk, refl = [], []
    for r0 in starts:
        a, b = oc.matmul(kt, w.x, w.l, w.f, w.s, z, row0=int(r0), nrows=ROWS_PER_BLOCK, want_dl=True)
        refk.append(a)
        refl.append(b)
    _CACHE[name] = (w, z, starts, np.vstack(refk), np.vstack(refl))
    return _CACHE[name]


@pytest.mark.parametrize("name", list(CONFIGS))
def test_config_operator_fast_full_n(pkg, name):
    import torch

    w, z, starts, refk, refl = _problem(name)
    e = pkg.KernelEngine(pkg.KernelType(w.kernel), w.x, pkg.Hyperparams(w.l, w.f, w.s), precision="fast")
    zd = torch.from_numpy(z).cuda()
    kk, dl, _ = e.apply(zd, True, True, False)
    rows = np.concatenate([np.arange(r0, r0 + ROWS_PER_BLOCK) for r0 in starts])
    idx = torch.from_numpy(rows).cuda()
    gk = kk.index_select(0, idx).cpu().numpy()
    gl = dl.index_select(0, idx).cpu().numpy()
    e.close()
    ek, el = rel_max(gk, refk), rel_max(gl, refl)
    print(f"{name} fast: Khat.Z {ek:.2e}  dKhat/dl.Z {el:.2e}")
    assert ek <= 2e-5
    assert el <= 2e-4


@pytest.mark.parametrize("name", list(CONFIGS))
def test_config_operator_fp64_row_blocks(pkg, name):
    import torch

    from paper_2503_02259_b200 import _lib

    w, z, starts, refk, refl = _problem(name)
    e = pkg.KernelEngine(pkg.KernelType(w.kernel), w.x, pkg.Hyperparams(w.l, w.f, w.s), precision="fp64")
    zd = torch.from_numpy(z).cuda()
    gk, gl = [], []
    for r0 in starts:
        _lib.call("kgp_engine_set_rows", e.handle, int(r0), ROWS_PER_BLOCK)
        kk, dl, _ = e.apply(zd, True, True, False)  # (n, k) buffers; rows [0, 256) = the block
        gk.append(kk[:ROWS_PER_BLOCK].cpu().numpy())
        gl.append(dl[:ROWS_PER_BLOCK].cpu().numpy())
    e.close()
    ek, el = rel_max(np.vstack(gk), refk), rel_max(np.vstack(gl), refl)
    print(f"{name} fp64: Khat.Z {ek:.2e}  dKhat/dl.Z {el:.2e}")
    assert ek <= 1e-12
    assert el <= 1e-12


def _cfg3_small():
    from paper_2503_02259_b200 import gp, workloads

    import os

    from conftest import GOLDEN

    # n = 16384 when its (1 h) reference run has been made, else the n = 8192 fixture
    g = golden("cfg3_small.npz" if os.path.exists(os.path.join(GOLDEN, "cfg3_small.npz"))
               else "cfg3_small_n8192.npz")
    n = int(g["n"])
    w = workloads.cfg3(n=n)
    probes = gp.ProbeSet.generate(n, w.k_z, w.probe_seed)
    chk = np.array([np.sum(w.x ** 2), np.sum(w.y ** 2), np.sum(probes.vectors ** 2)])
    np.testing.assert_allclose(chk, g["checksum"], rtol=1e-13)  # same seeded inputs as the reference's run
    assert bool(g["converged"])
    return g, w, probes


@pytest.mark.parametrize("precision,bar", [("fp64", 1e-6), ("fast", 1e-3)])
def test_cfg3_generator_nlml_reference_estimator(pkg, precision, bar):
    from paper_2503_02259_b200 import gp, precond

    g, w, probes = _cfg3_small()
    e = pkg.KernelEngine(pkg.KernelType.MATERN32, w.x, pkg.Hyperparams(w.l, w.f, w.s), precision=precision)
    pre = precond.build(e, w.rank)
    lg = gp.nlml_grad_iterative(e, w.y, pre, probes, tol=1e-10, max_iter=6000, probe_tol=1e-10)
    ref = g["iter_tight"]
    got = np.array([lg.loss, lg.grad_l, lg.grad_f, lg.grad_s])
    rel = np.abs(got - ref) / np.abs(ref)
    print(f"cfg3-generator n={w.n} {precision}: rel err loss/l/f/s = {rel}, converged={lg.converged}")
    assert np.all(rel <= bar), (got, ref, rel)
    if precision == "fp64":
        assert lg.converged


def test_cfg3_generator_fast_true_residual(pkg):
    """What 'converged' means for the fast operator at s = 1e-3: the
    recursive residual of the fast w-solve reaches tol while the TRUE residual against the fp64
    operator stalls at the operator's error times the solution's size. Measured and bounded
    here, so the fast NLML's converged flag is never read as fp64 convergence."""
    import torch

    from paper_2503_02259_b200 import precond, solver

    g, w, probes = _cfg3_small()
    hp = pkg.Hyperparams(w.l, w.f, w.s)
    ef = pkg.KernelEngine(pkg.KernelType.MATERN32, w.x, hp, precision="fast")
    e64 = pkg.KernelEngine(pkg.KernelType.MATERN32, w.x, hp, precision="fp64")
    rep = solver.pcg_solve(ef.matmul, precond.build(ef, w.rank).apply_inverse, w.y, tol=1e-6, max_iter=6000)
    assert rep.converged[0]
    true_rel = np.linalg.norm(w.y - e64.matmul(rep.solution)) / np.linalg.norm(w.y)
    ref = solver.pcg_solve(e64.matmul, precond.build(e64, w.rank).apply_inverse, w.y, tol=1e-10, max_iter=6000)
    sol_rel = np.linalg.norm(rep.solution - ref.solution) / np.linalg.norm(ref.solution)
    print(f"fast w-solve: recursive rel {rep.traces[0].final_rel_residual:.2e}, true rel {true_rel:.2e}, "
          f"solution rel err vs fp64 {sol_rel:.2e}")
    assert true_rel <= 1e-4
    assert sol_rel <= 1e-3
    del torch


def test_cfg5_generator_local_variance_vs_exact(pkg):
    """configs[4]'s predictive variance: at m = 262144 correlated test points the Hutchinson
    diagonal is noise-dominated, and a truncated-spectrum (LOVE-style) cache
    would need every mode of Khat above s because the posterior variance is ~1e-4 f^2. The
    variance path is local kriging (gp.predict_local): var = f^2 - c^T Khat_NN^-1 c over the k
    nearest training points, an upper bound of the exact variance that tightens as k grows.
    Checked here against the exact variance (gp.py:240-243, dense Cholesky on the device) on the
    configs[4] generator at reduced n = 16384, m = 1024: the error must shrink with k and be
    <= 3 % in stddev at k = 128 (measured 34 % / 17 % / 2.1 % at k = 32 / 64 / 128); the mean
    is the iterative solve's (1e-6). The bound loosens as the data get denser relative to l
    (at full n the 128 neighbours cover a radius l / 16): DESIGN.md 3.4b states the limits."""
    from paper_2503_02259_b200 import gp, workloads

    w = workloads.cfg5(n=16384, m_test=1024)
    xs = w.extra["xstar"]
    hp = pkg.Hyperparams(w.l, w.f, w.s)
    ex = gp.predict(pkg.KernelType.MATERN52, w.x, w.y, xs, hp, mode="exact")
    errs = {}
    for knn in (32, 64, 128):
        lo = gp.predict_local(pkg.KernelType.MATERN52, w.x, w.y, xs, hp, tol=1e-10, max_iter=3000, k_nn=knn,
                              precision="fp64", preconditioner="afn", precond_rank=512)
        errs[knn] = float(np.max(np.abs(lo.stddev - ex.stddev) / ex.stddev))
        assert np.all(lo.stddev >= ex.stddev * (1 - 1e-6))  # conditioning on fewer points: an upper bound
        if knn == 128:
            assert rel_max(lo.mean, ex.mean) <= 1e-6
    print("cfg5-generator local-variance max rel stddev error by k:", errs)
    assert errs[128] <= errs[64] <= errs[32]
    assert errs[128] <= 3e-2, errs
