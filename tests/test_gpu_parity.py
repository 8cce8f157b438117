"""GPU parity: the CUDA path (through the C ABI) against the reference's golden vectors
and the CPU oracle. Tolerances are written next to each check:

* fp64 operator vs reference outputs: <= 1e-12 of max|ref| (test_kmat.py:49's bar)
* fast (3xTF32) operator: <= 2e-5 of max|ref|; tf32 operator: <= 1e-3 (north star)
* NLML/gradient in tolerance mode (tol = probe_tol = 1e-10): <= 1e-6 relative (north star, FP64 mode)
"""

import numpy as np
import pytest

from conftest import golden, rel_max

pytestmark = pytest.mark.gpu

KTS = ("gaussian", "matern32", "matern52")


@pytest.fixture(scope="module")
def pkg():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2503_02259_b200 as p

    return p


def _hp(pkg, l, f, s):
    return pkg.Hyperparams(l=l, f=f, s=s)


# ---------------------------------------------------------------------------- panels
def test_panels_match_reference(pkg):
    g = golden("panels.npz")
    x, y, l = g["panel_x"], g["panel_y"], float(g["panel_l"])
    np.testing.assert_allclose(pkg.pairwise_sq_dist(x, y), g["sqdist_numba"], rtol=1e-15, atol=0)
    for kt in KTS:
        k = pkg.eval_kernel(pkg.KernelType(kt), x, y, l)
        gl = pkg.eval_kernel_grad_l(pkg.KernelType(kt), x, y, l)
        np.testing.assert_allclose(k, g[f"K_{kt}_numba"], rtol=1e-13, atol=1e-15)
        np.testing.assert_allclose(gl, g[f"G_{kt}_numba"], rtol=1e-12, atol=1e-15)
        assert gl[0, 0] == 0.0  # coincident pair (test_kernels.py:80-83)


def test_known_answers(pkg):
    kt = pkg.KernelType.GAUSSIAN
    assert abs(pkg.eval_kernel(kt, [[0.0]], [[1.0]], 1.0)[0, 0] - 0.6065306597126334) <= 1e-15
    e = pkg.KernelEngine(kt, [[0.0]], _hp(pkg, 1, 2, 0.1))
    np.testing.assert_allclose(e.matmul([[1.0]]), [[4.1]], rtol=1e-15)
    np.testing.assert_allclose(e.grad_matmul(pkg.Theta.F, np.array([[3.0]])), [[12.0]], rtol=1e-15)
    b = np.random.default_rng(0).standard_normal((1, 2))
    np.testing.assert_array_equal(e.grad_matmul(pkg.Theta.S, b), b)


# ---------------------------------------------------------------------------- operator
@pytest.mark.parametrize("tag", list("abcdefg"))
def test_engine_fp64_matches_reference(pkg, tag):
    g = golden("engine.npz")
    n, d, k, l, f, s, bs = g[f"{tag}_meta"]
    e = pkg.KernelEngine(pkg.KernelType(str(g[f"{tag}_kt"])), g[f"{tag}_x"], _hp(pkg, l, f, s),
                         precision="fp64")
    b = g[f"{tag}_b"]
    assert rel_max(e.matmul(b), g[f"{tag}_K"]) <= 1e-12
    for th in ("l", "f"):
        assert rel_max(e.grad_matmul(pkg.Theta(th), b), g[f"{tag}_d{th}"]) <= 1e-12
    np.testing.assert_array_equal(e.grad_matmul(pkg.Theta.S, b), g[f"{tag}_ds"])
    kk, dl, df = e.matmul_with_grads(b)
    assert rel_max(kk, g[f"{tag}_K"]) <= 1e-12
    assert rel_max(dl, g[f"{tag}_dl"]) <= 1e-12
    assert rel_max(df, g[f"{tag}_df"]) <= 1e-12


@pytest.mark.parametrize("precision,bar", [("fast", 2e-5), ("tf32", 1e-3), ("bf16x3", 5e-5)])
@pytest.mark.parametrize("tag", list("abcdefg"))
def test_engine_tensorcore_matches_reference(pkg, tag, precision, bar):
    g = golden("engine.npz")
    n, d, k, l, f, s, bs = g[f"{tag}_meta"]
    if precision == "bf16x3" and d <= 4:
        pytest.skip("bf16x3 runs with the tensor-core distance only (d > 4)")
    e = pkg.KernelEngine(pkg.KernelType(str(g[f"{tag}_kt"])), g[f"{tag}_x"], _hp(pkg, l, f, s),
                         precision=precision)
    b = g[f"{tag}_b"]
    kk, dl, df = e.matmul_with_grads(b)
    assert rel_max(kk, g[f"{tag}_K"]) <= bar
    assert rel_max(dl, g[f"{tag}_dl"]) <= 10 * bar  # derivative entries vanish at r=0: larger relative spread
    assert rel_max(df, g[f"{tag}_df"]) <= bar
    assert rel_max(e.matmul(b), g[f"{tag}_K"]) <= bar


@pytest.mark.parametrize("kt", KTS)
@pytest.mark.parametrize("d", [1, 2, 3, 4, 5, 8, 11, 16])
@pytest.mark.parametrize("k", [1, 16, 17, 33, 64, 130])
def test_fast_operator_shapes(pkg, kt, d, k):
    """Every tcgen05 instantiation (padded d, KP, NOUT) against the fp64 engine."""
    rng = np.random.default_rng(d * 1000 + k)
    n = 300 + 7 * d
    x = rng.standard_normal((n, d))
    b = rng.standard_normal((n, k))
    hp = _hp(pkg, 0.9 * np.sqrt(d), 1.3, 0.2)
    ref = pkg.KernelEngine(pkg.KernelType(kt), x, hp, precision="fp64").matmul_with_grads(b)
    got = pkg.KernelEngine(pkg.KernelType(kt), x, hp, precision="fast").matmul_with_grads(b)
    assert rel_max(got[0], ref[0]) <= 2e-5
    assert rel_max(got[1], ref[1]) <= 2e-4
    assert rel_max(got[2], ref[2]) <= 2e-5


@pytest.mark.parametrize("kt", KTS)
@pytest.mark.parametrize("d", [5, 8, 11, 16])
@pytest.mark.parametrize("k", [1, 16, 17, 33, 64, 130])
def test_bf16x3_operator_shapes(pkg, kt, d, k):
    """The bf16x3 contraction (two round-to-nearest bf16 terms per operand, A0B0 + A0B1 + A1B0)
    against the fp64 engine: 5e-5 (2.5x the 3xTF32 bar: its two-term bf16 splits keep 16
    mantissa bits, the tf32 hi/lo ones 22; single-column products reach 2.4e-5) and 5e-4 for
    dKhat/dl."""
    rng = np.random.default_rng(d * 1000 + k + 7)
    n = 300 + 7 * d
    x = rng.standard_normal((n, d))
    b = rng.standard_normal((n, k))
    hp = _hp(pkg, 0.9 * np.sqrt(d), 1.3, 0.2)
    ref = pkg.KernelEngine(pkg.KernelType(kt), x, hp, precision="fp64").matmul_with_grads(b)
    got = pkg.KernelEngine(pkg.KernelType(kt), x, hp, precision="bf16x3").matmul_with_grads(b)
    assert rel_max(got[0], ref[0]) <= 5e-5
    assert rel_max(got[1], ref[1]) <= 5e-4
    assert rel_max(got[2], ref[2]) <= 5e-5


def test_bf16x3_rejects_direct_distance(pkg):
    x = np.random.default_rng(0).standard_normal((100, 3))
    e = pkg.KernelEngine(pkg.KernelType.GAUSSIAN, x, _hp(pkg, 1, 1, 0.1), precision="bf16x3")
    with pytest.raises(ValueError, match="d > 4"):
        e.matmul(np.ones((100, 2)))


@pytest.mark.parametrize("kt", KTS)
@pytest.mark.parametrize("n,k", [(1, 1), (127, 1), (129, 2), (1000, 3), (2049, 4), (300, 5)])
def test_fp64_symmetric_small_k(pkg, kt, n, k):
    """The fp64 square operator with k <= 4 evaluates each entry once for both row blocks
    (kmm_f64_sym_kernel, transpose-butterfly column sums, partner-ordered partials): equal to
    the oracle's streamed operator to the fp64 bar, including ragged last blocks; k = 5 takes
    the ordinary path. ON_THE_FLY so the products are not the DENSE-mode DGEMM."""
    from oracle import kgp_oracle as orc

    rng = np.random.default_rng(n + 31 * k)
    x = rng.uniform(0, 1, (n, 3))
    b = rng.standard_normal((n, k))
    hp = _hp(pkg, 0.4, 1.3, 0.05)
    e = pkg.KernelEngine(pkg.KernelType(kt), x, hp, mode=pkg.EngineMode.ON_THE_FLY, precision="fp64")
    ref = orc.khat_matmul(kt, x, hp.l, hp.f, hp.s, b)
    assert rel_max(e.matmul(b), ref) <= 1e-12
    assert rel_max(e.grad_matmul(pkg.Theta.F, b), orc.khat_matmul(kt, x, hp.l, hp.f, hp.s, b, theta="f")) <= 1e-12
    got = e.matmul(b)
    assert np.array_equal(got, e.matmul(b))  # run-to-run identical


@pytest.mark.parametrize("kt", KTS)
@pytest.mark.parametrize("n,d,k", [(301, 3, 29), (257, 8, 32), (300, 4, 33), (130, 2, 40), (259, 8, 51), (200, 3, 64),
                                   (190, 9, 65), (150, 5, 100), (140, 2, 130)])
def test_fp64_lane_split_wide_k(pkg, kt, n, d, k):
    """The fp64 operator's wide-k passes (kmm_f64_split_kernel: 2 or 4 lanes share a row and every
    kernel-entry evaluation, each lane contracting its own columns of the slice): one output
    (k > 48) and two outputs (k > 28), every (G, KQ) layout, ragged rows / columns / tiles,
    against the oracle's streamed operator (kmat.py:165-189) at the fp64 bar, run-to-run identical."""
    from oracle import kgp_oracle as orc

    rng = np.random.default_rng(n + 31 * k)
    x = rng.uniform(0, 1, (n, d))
    b = rng.standard_normal((n, k))
    hp = _hp(pkg, 0.4, 1.3, 0.05)
    e = pkg.KernelEngine(pkg.KernelType(kt), x, hp, mode=pkg.EngineMode.ON_THE_FLY, precision="fp64")
    ref_k = orc.khat_matmul(kt, x, hp.l, hp.f, hp.s, b)
    ref_l = orc.khat_matmul(kt, x, hp.l, hp.f, hp.s, b, theta="l")
    ref_f = orc.khat_matmul(kt, x, hp.l, hp.f, hp.s, b, theta="f")
    got_k, got_l, got_f = e.matmul_with_grads(b)
    assert rel_max(got_k, ref_k) <= 1e-12 and rel_max(got_l, ref_l) <= 1e-12 and rel_max(got_f, ref_f) <= 1e-12
    one = e.matmul(b)
    assert rel_max(one, ref_k) <= 1e-12
    assert np.array_equal(one, e.matmul(b))
    assert rel_max(one, got_k) <= 1e-13  # different layouts and column splits, the same entries


def test_cfg2_row_subsample(pkg):
    """configs[1] at full size: fast K.Z and dK/dl.Z against the C oracle on 512 rows."""
    import torch

    from oracle import kgp_oracle_c as oc
    from paper_2503_02259_b200 import workloads

    w = workloads.cfg2()
    zd = torch.from_numpy(w.z).cuda()
    rows = np.random.default_rng(7).choice(w.n, 512, replace=False)
    rows.sort()
    refk = np.empty((512, w.z.shape[1]))
    refd = np.empty_like(refk)
    for i, gi in enumerate(rows):
        a, bb = oc.matmul("gaussian", w.x, w.l, w.f, w.s, w.z, row0=int(gi), nrows=1, want_dl=True)
        refk[i], refd[i] = a[0], bb[0]
    for precision in ("fast", "bf16x3"):
        e = pkg.KernelEngine(pkg.KernelType.GAUSSIAN, w.x, _hp(pkg, w.l, w.f, w.s), precision=precision)
        kk, dl, _ = e.apply(zd, True, True, False)
        kk, dl = kk.cpu().numpy()[rows], dl.cpu().numpy()[rows]
        assert rel_max(kk, refk) <= 2e-5, precision
        assert rel_max(dl, refd) <= 2e-4, precision
        e.close()


def test_cross_matmul_matches_panel(pkg):
    import torch

    rng = np.random.default_rng(3)
    x = rng.uniform(-1, 1, (500, 3))
    xs = rng.uniform(-1, 1, (77, 3))
    b = rng.standard_normal((500, 5))
    for prec, bar in (("fp64", 1e-12), ("fast", 2e-5)):
        for kt in KTS:
            hp = _hp(pkg, 0.6, 1.2, 0.1)
            e = pkg.KernelEngine(pkg.KernelType(kt), x, hp, precision=prec)
            got = e.cross_matmul(torch.from_numpy(xs).cuda(), torch.from_numpy(b).cuda()).cpu().numpy()
            ref = 1.44 * pkg.eval_kernel(pkg.KernelType(kt), xs, x, 0.6) @ b
            assert rel_max(got, ref) <= bar


# ---------------------------------------------------------------------------- preconditioner
def test_fps_matches_reference(pkg):
    g = golden("precond.npz")
    np.testing.assert_array_equal(pkg.fps_select(g["fps_x"], 50, 0), g["fps_idx"])
    np.testing.assert_array_equal(pkg.fps_select(g["fps_x"], 20, 7), g["fps_idx_seed7"])
    np.testing.assert_array_equal(pkg.fps_select(g["fps_tie_x"], 6, 0), g["fps_tie_idx"])


@pytest.mark.parametrize("kt", KTS)
def test_nystrom_matches_reference(pkg, kt):
    from paper_2503_02259_b200 import precond

    g = golden("precond.npz")
    e = pkg.KernelEngine(pkg.KernelType(kt), g["fps_x"], _hp(pkg, 0.8, 1.1, 0.02))
    p = precond.build(e, 60)
    np.testing.assert_array_equal(p.landmark_indices, g[f"{kt}_idx"])
    b = g[f"{kt}_b"]
    assert rel_max(p.apply_inverse(b), g[f"{kt}_minv"]) <= 1e-8
    assert rel_max(p.apply(b), g[f"{kt}_m"]) <= 1e-10


# ---------------------------------------------------------------------------- solvers
def test_pcg_matches_reference(pkg):
    from paper_2503_02259_b200 import precond, solver

    g = golden("solver.npz")
    l, f, s = g["hp"]
    e = pkg.KernelEngine(pkg.KernelType.GAUSSIAN, g["x"], _hp(pkg, l, f, s))
    pre = precond.build(e, 40)
    for tag, minv in (("plain", None), ("nys", pre.apply_inverse)):
        rep = solver.pcg_solve(e.matmul, minv, g["y"], tol=1e-8, max_iter=500)
        # CG counts at tol=1e-8 are chaotic under rounding changes even inside the reference
        # (DENSE vs ON_THE_FLY: [62,60,0,62] vs [56,61,0,62]): counts within 15%, solution 100 x tol
        its = np.array(rep.iteration_counts())
        ref_its = g[f"{tag}_iters"]
        assert np.all(np.abs(its - ref_its) <= np.maximum(1, np.ceil(0.15 * ref_its))), (its, ref_its)
        assert rel_max(rep.solution, g[f"{tag}_sol"]) <= 1e-6
        assert list(rep.converged) == list(g[f"{tag}_conv"])
        for j, t in enumerate(rep.traces):
            m = min(t.iterations, int(g[f"{tag}_iters"][j]), 8)
            np.testing.assert_allclose(t.alphas[:m], g[f"{tag}_alphas"][j, :m], rtol=1e-9)
            np.testing.assert_allclose(t.betas[:m], g[f"{tag}_betas"][j, :m], rtol=1e-9)
        assert rep.traces[2].iterations == 0 and np.all(rep.solution[:, 2] == 0.0)


def test_slq_matches_reference(pkg):
    from paper_2503_02259_b200 import solver

    g = golden("solver.npz")
    # SLQ on the reference's own coefficients: isolates the device eigensolver (stev)
    traces = [solver.CgTrace(g["probe_alphas"][j, :m], g["probe_betas"][j, :m], int(m), 0.0)
              for j, m in enumerate(g["probe_iters"])]
    got = solver.slq_logdet(traces, g["probe_norms"])
    assert abs(got - float(g["slq_logdet"])) <= 1e-12 * abs(float(g["slq_logdet"]))
    traces = [solver.CgTrace(g["fixed_alphas"][j, :7], g["fixed_betas"][j, :7], 7, 0.0) for j in range(6)]
    got = solver.slq_logdet(traces, g["probe_norms"])
    assert abs(got - float(g["fixed_slq"])) <= 1e-12 * abs(float(g["fixed_slq"]))


def test_slq_known_answers(pkg):
    from paper_2503_02259_b200 import solver

    rng = np.random.default_rng(5)
    d = np.arange(1.0, 11.0)
    z = rng.standard_normal((10, 200))
    rep = solver.pcg_solve(lambda b: d[:, None] * b, None, z, tol=0.0, max_iter=10)
    est = solver.slq_logdet(rep.traces, np.sum(z * z, axis=0))
    assert abs(est - np.sum(np.log(d))) / np.sum(np.log(d)) < 0.05
    t = solver.CgTrace(np.array([2.0]), np.array([0.1]), 1, 0.0)
    assert abs(solver.slq_logdet([t], [3.0]) - 3.0 * np.log(0.5)) < 1e-15


def test_pcg_breakdown_raises(pkg):
    from paper_2503_02259_b200 import solver

    from paper_2503_02259_b200.errors import BreakdownError

    a = -np.eye(5)
    with pytest.raises(BreakdownError):
        solver.pcg_solve(lambda b: a @ b, None, np.ones(5), tol=1e-8)


# ---------------------------------------------------------------------------- NLML
def test_nlml_iterative_matches_reference(pkg):
    from paper_2503_02259_b200 import gp, precond

    g = golden("nlml.npz")
    l, f, s = g["hp"]
    e = pkg.KernelEngine(pkg.KernelType.GAUSSIAN, g["x"], _hp(pkg, l, f, s))
    pre = precond.build(e, int(g["rank"]))
    probes = gp.ProbeSet(g["probes"])
    lg = gp.nlml_grad_iterative(e, g["y"], pre, probes, tol=1e-10, max_iter=3000, probe_tol=1e-10)
    ref = g["iter_tight"][:4]
    got = np.array([lg.loss, lg.grad_l, lg.grad_f, lg.grad_s])
    assert np.all(np.abs(got - ref) <= 1e-6 * np.abs(ref)), (got, ref)
    assert lg.converged
    ex = gp.grad_exact(e, g["y"])
    np.testing.assert_allclose([ex.loss, ex.grad_l, ex.grad_f, ex.grad_s], g["exact"], rtol=1e-9)


@pytest.mark.parametrize("kt", ["matern32", "matern52"])
def test_nlml_matern_matches_reference(pkg, kt):
    from paper_2503_02259_b200 import gp, precond

    g = golden("nlml.npz")
    e = pkg.KernelEngine(pkg.KernelType(kt), g[f"{kt}_x"], _hp(pkg, 0.25, 1.5, 1e-2))
    lg = gp.nlml_grad_iterative(e, g[f"{kt}_y"], precond.build(e, 40), gp.ProbeSet(g[f"{kt}_probes"]),
                                tol=1e-10, max_iter=3000, probe_tol=1e-10)
    got = np.array([lg.loss, lg.grad_l, lg.grad_f, lg.grad_s])
    ref = g[f"{kt}_res"]
    assert np.all(np.abs(got - ref) <= 1e-6 * np.abs(ref)), (got, ref)


def test_cfg1_full_matches_reference(pkg):
    """configs[0] at full size (n=4096) in tolerance mode, same seeds as the reference run."""
    from paper_2503_02259_b200 import gp, precond, workloads

    g = golden("cfg1_full.npz")
    w = workloads.cfg1()
    probes = gp.ProbeSet.generate(w.n, w.k_z, w.probe_seed)
    chk = np.array([np.sum(w.x ** 2), np.sum(w.y ** 2), np.sum(probes.vectors ** 2)])
    np.testing.assert_allclose(chk, g["checksum"], rtol=1e-14)
    e = pkg.KernelEngine(pkg.KernelType.GAUSSIAN, w.x, _hp(pkg, w.l, w.f, w.s))
    lg = gp.nlml_grad_iterative(e, w.y, precond.build(e, w.rank), probes, tol=1e-10, max_iter=3000,
                                probe_tol=1e-10)
    got = np.array([lg.loss, lg.grad_l, lg.grad_f, lg.grad_s])
    ref = g["iter_tight"]
    assert np.all(np.abs(got - ref) <= 1e-6 * np.abs(ref)), (got, ref)


def test_cfg1_fast_mode_within_tf32_bar(pkg):
    """North star: NLML and gradient within 1e-3 of the reference in the TF32 (tensor-core)
    mode. The 3xTF32 operator gives 3e-6 (loss) .. 6e-4 (grad_s) at configs[0] in tolerance
    mode (measured, tools/nlml_precision.py); the single-pass tf32 operator does not meet it
    (grad_f/grad_s amplify operator error ~1e4x) and is a throughput mode only."""
    from paper_2503_02259_b200 import gp, precond, workloads

    g = golden("cfg1_full.npz")
    w = workloads.cfg1()
    probes = gp.ProbeSet.generate(w.n, w.k_z, w.probe_seed)
    e = pkg.KernelEngine(pkg.KernelType.GAUSSIAN, w.x, _hp(pkg, w.l, w.f, w.s), precision="fast")
    lg = gp.nlml_grad_iterative(e, w.y, precond.build(e, w.rank), probes, tol=1e-10, max_iter=3000,
                                probe_tol=1e-10)
    got = np.array([lg.loss, lg.grad_l, lg.grad_f, lg.grad_s])
    ref = g["iter_tight"][:4]
    assert lg.converged
    assert np.all(np.abs(got - ref) <= 1e-3 * np.abs(ref)), (got, ref)


def test_nlml_deterministic(pkg):
    from paper_2503_02259_b200 import gp, precond

    rng = np.random.default_rng(6)
    x, y = rng.standard_normal((80, 2)), rng.standard_normal(80)
    e = pkg.KernelEngine(pkg.KernelType.GAUSSIAN, x, _hp(pkg, 1.0, 1.2, 0.3))
    pre = precond.build(e, 25)
    a = gp.nlml_grad_iterative(e, y, pre, gp.ProbeSet.generate(80, 8, 99), tol=1e-8)
    b = gp.nlml_grad_iterative(e, y, pre, gp.ProbeSet.generate(80, 8, 99), tol=1e-8)
    assert (a.loss, a.grad_l, a.grad_f, a.grad_s) == (b.loss, b.grad_l, b.grad_f, b.grad_s)


# ---------------------------------------------------------------------------- prediction, training
@pytest.mark.parametrize("kt", KTS)
def test_predict_matches_reference(pkg, kt):
    from paper_2503_02259_b200 import gp

    g = golden("predict.npz")
    hp = _hp(pkg, 0.8, 1.0, 0.05)
    ex = gp.predict(pkg.KernelType(kt), g["x"], g["y"], g["xs"], hp, mode="exact")
    np.testing.assert_allclose(ex.mean, g[f"{kt}_exact_mean"], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(ex.stddev, g[f"{kt}_exact_sd"], rtol=1e-7, atol=1e-9)
    it = gp.predict(pkg.KernelType(kt), g["x"], g["y"], g["xs"], hp, mode="iterative", tol=1e-10,
                    max_iter=2000)
    np.testing.assert_allclose(it.mean, g[f"{kt}_iter_mean"], rtol=1e-7, atol=1e-9)
    np.testing.assert_allclose(it.stddev, g[f"{kt}_iter_sd"], rtol=1e-6, atol=1e-7)


def test_train_matches_reference(pkg):
    from paper_2503_02259_b200 import train

    g = golden("train.npz")
    init = train.initial_hyperparams(g["x"], g["y"], 3)
    np.testing.assert_allclose([init.l, init.f, init.s], g["init"], rtol=1e-15)
    res = train.fit(pkg.KernelType.MATERN52, g["x"], g["y"],
                    train.TrainConfig(learning_rate=0.1, max_steps=15, mode="exact", rng_seed=3))
    np.testing.assert_allclose(res.loss_history, g["exact_loss"], rtol=1e-9)
    np.testing.assert_allclose([res.params.l, res.params.f, res.params.s], g["exact_params"], rtol=1e-8)
    res = train.fit(pkg.KernelType.MATERN52, g["x"], g["y"],
                    train.TrainConfig(learning_rate=0.1, max_steps=6, mode="iterative", rng_seed=3,
                                      tol=1e-10, probe_tol=1e-10, max_iter=2000))
    np.testing.assert_allclose(res.loss_history, g["iter_loss"], rtol=1e-7)


def test_errors_and_handles(pkg):
    from paper_2503_02259_b200 import _lib
    from paper_2503_02259_b200.errors import KernelGpError, ResourceLimitError

    e = pkg.KernelEngine(pkg.KernelType.GAUSSIAN, np.zeros((30, 2)) + np.arange(30)[:, None],
                         _hp(pkg, 1, 1, 0.5), dense_budget=25, mode=pkg.EngineMode.ON_THE_FLY)
    with pytest.raises(ResourceLimitError, match="25"):
        e.materialize()
    with pytest.raises(ValueError, match="rows"):
        e.matmul(np.ones((9, 2)))
    h = e.handle
    e.close()
    with pytest.raises(KernelGpError):
        _lib.call("kgp_engine_destroy", h)  # double destroy is an error, not a crash


def test_fixed_recipe_matches_reference(pkg):
    """configs[0]'s fixed recipe on the device: PCG 50 (preconditioned) + 20-step probe CG + SLQ.
    Fixed-step SLQ is chaotic under rounding changes (reference self-spread 1.5e-6): bar 1e-5."""
    from paper_2503_02259_b200 import gp, precond, workloads

    g = golden("cfg1_full.npz")
    w = workloads.cfg1()
    probes = gp.ProbeSet.generate(w.n, w.k_z, w.probe_seed)
    e = pkg.KernelEngine(pkg.KernelType.GAUSSIAN, w.x, _hp(pkg, w.l, w.f, w.s))
    lg = gp.nlml_grad_iterative(e, w.y, precond.build(e, w.rank), probes, tol=0.0, max_iter=50, probe_tol=0.0,
                                probe_max_iter=20)
    from oracle import kgp_oracle as orc

    ny = orc.Nystrom("gaussian", w.x, w.l, w.f, w.s, w.rank)
    ref = orc.nlml_grad("gaussian", w.x, w.y, w.l, w.f, w.s, probes.vectors, ny, tol=0.0, max_iter=50,
                        probe_tol=0.0, dense=True, probe_max_iter=20)
    got = np.array([lg.loss, lg.grad_l, lg.grad_f, lg.grad_s])
    # Bars = 2x the reference's OWN spread between its DENSE and ON_THE_FLY modes on exactly this
    # recipe and these seeds (measured with kernelgp: loss 4.5e-6, grad_l 2.4e-3, grad_f 1.4e-2,
    # grad_s 3.4e-5): 20 CG steps amplify summation-order rounding into the probe solutions.
    bars = np.array([1e-5, 5e-3, 3e-2, 7e-5])
    rel = np.abs(got - np.array(ref[:4])) / np.abs(np.array(ref[:4]))
    assert np.all(rel <= bars), (got, ref, rel)
    assert not lg.converged  # tol = 0: the solves stop on the iteration caps by construction


def _dist_gpu_worker(rank, world, port, errfile):
    import os

    import torch
    import torch.distributed as tdist

    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        # gloo: the collectives run on the host, so two ranks may share one GPU safely
        tdist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        import paper_2503_02259_b200 as kgp
        from paper_2503_02259_b200 import dist as kdist
        from paper_2503_02259_b200 import gp, precond

        g = golden("nlml.npz")
        l, f, s = g["hp"]
        n = g["x"].shape[0]
        e = kgp.KernelEngine(kgp.KernelType.GAUSSIAN, g["x"], kgp.Hyperparams(l, f, s))
        wt = kdist.build_precond_factor(e, int(g["rank"]))
        r0, r1 = kdist.row_range(n, world, rank)
        ops = kdist.CudaRowOps(e, r0, r1, wt)
        comm = kdist.Comm(n)
        y = torch.from_numpy(g["y"][r0:r1].copy()).cuda()
        z = torch.from_numpy(np.ascontiguousarray(g["probes"].T[:, r0:r1])).cuda()
        got = kdist.dist_nlml_grad(ops, comm, y, z, np.einsum("ij,ij->j", g["probes"], g["probes"]), 1e-10, 3000,
                                   precondition=True, shift=s)
        ref = g["iter_tight"][:4]
        assert np.all(np.abs(np.array(got[:4]) - ref) <= 1e-6 * np.abs(ref)), (got, ref)
        single = gp.nlml_grad_iterative(e, g["y"], precond.build(e, int(g["rank"])), gp.ProbeSet(g["probes"]),
                                        tol=1e-10, max_iter=3000)
        assert abs(got[0] - single.loss) <= 1e-9 * abs(single.loss)
        tdist.barrier()
        tdist.destroy_process_group()
    except Exception as exc:
        with open(errfile, "a") as fh:
            fh.write(f"rank {rank}: {type(exc).__name__}: {exc}\n")
        raise


def test_row_partitioned_nlml_on_device(pkg, tmp_path):
    """dist.CudaRowOps (libkgp row-block operator + sharded Woodbury) with 2 ranks on one GPU."""
    import os
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    errfile = str(tmp_path / "err.txt")
    mp.spawn(_dist_gpu_worker, args=(2, port, errfile), nprocs=2, join=True)
    assert not os.path.exists(errfile), open(errfile).read()


def _dist_gpc_gpu_worker(rank, world, port, errfile):
    import os

    import torch
    import torch.distributed as tdist

    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        tdist.init_process_group("gloo", rank=rank, world_size=world)  # host collectives: one GPU is safe
        torch.cuda.set_device(0)
        import paper_2503_02259_b200 as kgp
        from paper_2503_02259_b200 import dist as kdist
        from paper_2503_02259_b200 import gpc

        rng = np.random.default_rng(7)
        n, c, kz = 400, 3, 4
        x = rng.uniform(0, 1, (n, 2))
        lab = gpc.sample_latent_labels(x, c, l=0.3, seed=7)
        prob = gpc.setup(x, lab)
        hp = kgp.Hyperparams(l=0.25, f=1.1, s=0.02)
        e = kgp.KernelEngine(kgp.KernelType.MATERN32, x, hp, precision="fp64")
        probes = gpc.generate_probes(n, c, kz, 5)
        r0, r1 = kdist.row_range(n, world, rank)
        ops = kdist.CudaRowOps(e, r0, r1)
        comm = kdist.Comm(n)
        cuda = lambda a: torch.from_numpy(np.ascontiguousarray(a[:, r0:r1])).cuda()  # noqa: E731
        got = kdist.dist_gpc_nlml_grad(ops, comm, cuda(prob.targets), cuda(prob.noise), cuda(probes),
                                       np.einsum("ij,ij->i", probes, probes), 1e-11, 3000)
        single = gpc.nlml_grad_iterative(e, prob, [], probes, tol=1e-11, max_iter=3000)
        ref = np.array([single.loss, single.grad_l, single.grad_f, single.grad_s])
        assert got[4] and single.converged
        assert np.all(np.abs(np.array(got[:4]) - ref) <= 1e-8 * np.abs(ref)), (got, ref)
        xs = rng.uniform(0, 1, (33, 2))
        alpha = rng.standard_normal((2, n))
        mean = kdist.dist_predict_mean(ops, comm, xs, cuda(alpha))
        want = e.cross_matmul(torch.from_numpy(xs).cuda(), torch.from_numpy(alpha.T.copy()).cuda())
        assert rel_max(mean.T.cpu().numpy(), want.cpu().numpy()) <= 1e-12
        var = kdist.dist_local_variance(comm, xs, lambda q: ops.local_variance(q, 32))
        np.testing.assert_array_equal(var.cpu().numpy(), ops.local_variance(xs, 32).cpu().numpy())
        tdist.barrier()
        tdist.destroy_process_group()
    except Exception as exc:
        with open(errfile, "a") as fh:
            fh.write(f"rank {rank}: {type(exc).__name__}: {exc}\n")
        raise


def test_row_partitioned_gpc_and_predict_on_device(pkg, tmp_path):
    """dist.dist_gpc_nlml_grad / dist_predict_mean over dist.CudaRowOps, 2 ranks on one GPU,
    against the single-GPU GPC estimator (same probes) and the full cross-kernel product."""
    import os
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    errfile = str(tmp_path / "err.txt")
    mp.spawn(_dist_gpc_gpu_worker, args=(2, port, errfile), nprocs=2, join=True)
    assert not os.path.exists(errfile), open(errfile).read()


def _dist_fit_gpu_worker(rank, world, port, errfile):
    import os

    import torch
    import torch.distributed as tdist

    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        tdist.init_process_group("gloo", rank=rank, world_size=world)  # host collectives: one GPU is safe
        torch.cuda.set_device(0)
        import paper_2503_02259_b200 as kgp
        from paper_2503_02259_b200 import dist as kdist
        from paper_2503_02259_b200 import train

        rng = np.random.default_rng(11)
        n = 500
        x = rng.uniform(0, 1, (n, 2))
        y = np.sin(4 * x[:, 0]) + 0.1 * rng.standard_normal(n)
        cfg = train.TrainConfig(learning_rate=0.05, max_steps=3, mode="iterative", k_z=6, tol=1e-10,
                                probe_tol=1e-10, max_iter=3000, precond_rank=40, rng_seed=4, precision="fp64")
        comm = kdist.Comm(n)
        r0, r1 = kdist.row_range(n, world, rank)
        hp0 = train.initial_hyperparams(x, y, cfg.rng_seed)
        res = kdist.dist_fit(comm, torch.from_numpy(y[r0:r1].copy()).cuda(), cfg, hp0,
                             kdist.cuda_ops_factory(kgp.KernelType.MATERN52, x, comm, 40, "fp64"))
        single = train.fit(kgp.KernelType.MATERN52, x, y, cfg)
        np.testing.assert_allclose(res.loss_history, single.loss_history, rtol=1e-8)
        np.testing.assert_allclose(res.raw.as_array(), single.raw.as_array(), rtol=1e-6)
        tdist.barrier()
        tdist.destroy_process_group()
    except Exception as exc:
        with open(errfile, "a") as fh:
            fh.write(f"rank {rank}: {type(exc).__name__}: {exc}\n")
        raise


def test_row_partitioned_fit_on_device(pkg, tmp_path):
    """dist.dist_fit over dist.CudaRowOps (2 ranks on one GPU) follows train.fit's trajectory."""
    import os
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    errfile = str(tmp_path / "err.txt")
    mp.spawn(_dist_fit_gpu_worker, args=(2, port, errfile), nprocs=2, join=True)
    assert not os.path.exists(errfile), open(errfile).read()


def test_predict_hutchinson_variance(pkg):
    """configs[4]'s estimator (no reference oracle): the mean equals the exact posterior mean,
    the Hutchinson variance is unbiased -- within 5 sigma of the exact diagonal, sigma from the
    exact off-diagonal mass of C^T Khat^-1 C (Rademacher probes)."""
    from oracle import kgp_oracle as orc
    from paper_2503_02259_b200 import gp

    rng = np.random.default_rng(12)
    x = rng.uniform(0, 1, (400, 2))
    y = np.sin(4 * np.pi * x[:, 0]) + np.cos(4 * np.pi * x[:, 1]) + 0.1 * rng.standard_normal(400)
    xs = rng.uniform(0, 1, (30, 2))
    hp = _hp(pkg, 0.1, 1.0, 1e-2)
    S = 4096
    got = gp.predict_hutchinson(pkg.KernelType.MATERN52, x, y, xs, hp, tol=1e-10, max_iter=3000,
                                precond_rank=40, num_probes=S, seed=5)
    mean, sd = orc.predict("matern52", x, y, xs, 0.1, 1.0, 1e-2)
    np.testing.assert_allclose(got.mean, mean, rtol=1e-7, atol=1e-9)
    c = orc.eval_kernel("matern52", x, xs, 0.1)
    a = c.T @ np.linalg.solve(orc.khat_dense("matern52", x, 0.1, 1.0, 1e-2), c)
    sigma = np.sqrt((a ** 2).sum(axis=1) - np.diag(a) ** 2) / np.sqrt(S)
    var_got = got.stddev ** 2
    var_ref = sd ** 2
    assert np.all(np.abs(var_got - var_ref) <= 5 * sigma + 1e-9), (var_got - var_ref, sigma)


@pytest.mark.parametrize("precision", ["fast", "fp64"])
def test_matmul_host_matches_device(pkg, precision):
    """kgp_engine_matmul_host (row-chunked, output transfer pipelined) equals the device product."""
    import torch

    from paper_2503_02259_b200 import _lib

    n, k = (80000, 32) if precision == "fast" else (3000, 5)  # the fast case is large enough to chunk
    rng = np.random.default_rng(3)
    x = rng.standard_normal((n, 8))
    b = rng.standard_normal((n, k))
    e = pkg.KernelEngine(pkg.KernelType.GAUSSIAN, x, _hp(pkg, 1.0, 1.2, 0.1), precision=precision)
    ref_k, ref_l, _ = e.apply(torch.from_numpy(b).cuda(), True, True, False)
    bh = torch.from_numpy(b).pin_memory()
    ok = torch.empty((n, k), dtype=torch.float64).pin_memory()
    ol = torch.empty_like(ok).pin_memory()
    _lib.call("kgp_engine_matmul_host", e.handle, k, bh.data_ptr(), ok.data_ptr(), ol.data_ptr(), None,
              torch.cuda.current_stream().cuda_stream)
    bar = 1e-5 if precision == "fast" else 1e-13  # chunking changes the column split (summation order)
    assert rel_max(ok.numpy(), ref_k.cpu().numpy()) <= bar
    assert rel_max(ol.numpy(), ref_l.cpu().numpy()) <= bar
    # pageable host memory works too (synchronous staging by the driver)
    ok2 = np.empty((n, k))
    _lib.call("kgp_engine_matmul_host", e.handle, k, b.ctypes.data, ok2.ctypes.data, None, None, None)
    assert rel_max(ok2, ref_k.cpu().numpy()) <= bar


@pytest.mark.parametrize("zchunks,ratio", [(2, 1), (5, 3), (8, 4)])
def test_matmul_host_input_chunks(pkg, zchunks, ratio, monkeypatch):
    """The host entry's input pipelining: B copied in `zchunks` chunks (sizes growing by `ratio`)
    while the first row chunk runs as column-chunked launches sharing one partial buffer; ragged n
    (not a multiple of 32) and a k that needs the 16-column padding."""
    import torch

    from paper_2503_02259_b200 import _lib

    n, k = 70001, 21
    rng = np.random.default_rng(zchunks)
    x = rng.standard_normal((n, 8))
    b = rng.standard_normal((n, k))
    e = pkg.KernelEngine(pkg.KernelType.GAUSSIAN, x, _hp(pkg, 1.0, 1.2, 0.1), precision="fast")
    ref_k, ref_l, _ = e.apply(torch.from_numpy(b).cuda(), True, True, False)
    monkeypatch.setenv("KGP_HOST_ZCHUNKS", str(zchunks))
    monkeypatch.setenv("KGP_HOST_ZRATIO", str(ratio))
    bh = torch.from_numpy(b).pin_memory()
    ok = torch.empty((n, k), dtype=torch.float64).pin_memory()
    ol = torch.empty_like(ok).pin_memory()
    for _ in range(2):  # the second call reuses the engine's buffers and events
        _lib.call("kgp_engine_matmul_host", e.handle, k, bh.data_ptr(), ok.data_ptr(), ol.data_ptr(), None,
                  torch.cuda.current_stream().cuda_stream)
        assert rel_max(ok.numpy(), ref_k.cpu().numpy()) <= 1e-5
        assert rel_max(ol.numpy(), ref_l.cpu().numpy()) <= 1e-5


def test_preconditioned_probes_estimator(pkg):
    """preconditioned_probes=True (extension): log|M| and the N(0, M) draws are exact, and the
    device estimator equals its dense same-probe formula (1e-6 at tight tolerances)."""
    import torch

    from oracle import kgp_oracle as orc
    from paper_2503_02259_b200 import gp, precond

    rng = np.random.default_rng(11)
    n, kt, l, f, s = 300, "matern32", 0.25, 1.3, 2e-2
    x = rng.uniform(0, 1, (n, 2))
    y = np.sin(5 * x[:, 0]) + 0.1 * rng.standard_normal(n)
    e = pkg.KernelEngine(pkg.KernelType(kt), x, _hp(pkg, l, f, s))
    pre = precond.build(e, 40)
    m_dense = pre.apply(np.eye(n))
    assert abs(pre.logdet - np.linalg.slogdet(m_dense)[1]) <= 1e-9 * abs(pre.logdet)
    zv = pre.sample(np.zeros((n, 40)), np.eye(40)).cpu().numpy()        # rows: f V e_i
    np.testing.assert_allclose(zv.T @ zv, m_dense - s * np.eye(n), atol=1e-10 * np.abs(m_dense).max())
    probes = gp.ProbeSet.generate(n, 6, 3)
    lg = gp.nlml_grad_iterative(e, y, pre, probes, tol=1e-11, max_iter=2000, probe_tol=1e-11,
                                preconditioned_probes=True)
    w2 = np.random.default_rng([3, gp.PP_TAIL_SEED]).standard_normal((40, 6))
    z = pre.sample(probes.vectors, w2).cpu().numpy().T                   # (n, k_z) ~ N(0, M)
    kh = orc.khat_dense(kt, x, l, f, s)
    mi = np.linalg.inv(m_dense)
    ev, vec = np.linalg.eigh(m_dense)
    mh = (vec / np.sqrt(ev)) @ vec.T                                    # M^-1/2
    ah = mh @ kh @ mh
    ea, va = np.linalg.eigh(ah)
    loga = (va * np.log(ea)) @ va.T
    zh = mh @ z
    w = np.linalg.solve(kh, y)
    loss = 0.5 * (y @ w + pre.logdet + np.einsum("ij,ij->", zh, loga @ zh) / 6 + n * np.log(2 * np.pi))
    kap = orc.eval_kernel(kt, x, x, l)
    dks = [f * f * orc.eval_kernel_grad_l(kt, x, x, l), 2 * f * kap, np.eye(n)]
    u = np.linalg.solve(kh, z)
    grads = [0.5 * (-w @ dk @ w + np.einsum("ij,ij->", mi @ z, dk @ u) / 6) for dk in dks]
    got = np.array([lg.loss, lg.grad_l, lg.grad_f, lg.grad_s])
    ref = np.array([loss, *grads])
    assert lg.converged
    assert np.all(np.abs(got - ref) <= 1e-6 * np.abs(ref)), (got, ref)


def test_preconditioned_probes_unbiased(pkg):
    """Averaged over probe sets the preconditioned estimator approaches the exact gradient."""
    from paper_2503_02259_b200 import gp, precond

    rng = np.random.default_rng(5)
    n = 400
    x = rng.uniform(0, 1, (n, 3))
    y = np.cos(4 * x[:, 1]) + 0.1 * rng.standard_normal(n)
    e = pkg.KernelEngine(pkg.KernelType.GAUSSIAN, x, _hp(pkg, 0.3, 1.0, 1e-2))
    pre = precond.build(e, 60)
    ex = gp.grad_exact(e, y)
    est = np.array([gp.nlml_grad_iterative(e, y, pre, gp.ProbeSet.generate(n, 32, r), tol=1e-10, max_iter=2000,
                                           probe_tol=1e-8, preconditioned_probes=True).grads() for r in range(8)])
    mean, sem = est.mean(axis=0), est.std(axis=0, ddof=1) / np.sqrt(len(est))
    assert np.all(np.abs(mean - ex.grads()) <= 4 * sem + 1e-9 * np.abs(ex.grads())), (mean, ex.grads(), sem)



def test_predict_local_variance(pkg):
    """predict_local: exact when the neighbourhood is the whole training set; the cross kNN
    matches a numpy search; a 64-neighbour variance is close to the exact one for a short
    length scale."""
    import torch

    from oracle import kgp_oracle as orc
    from paper_2503_02259_b200 import _lib, gp

    rng = np.random.default_rng(21)
    x = rng.uniform(0, 1, (60, 2))
    y = np.sin(4 * x[:, 0]) + 0.05 * rng.standard_normal(60)
    xs = rng.uniform(0, 1, (25, 2))
    hp = _hp(pkg, 0.3, 1.2, 1e-2)
    ex = gp.predict(pkg.KernelType.MATERN52, x, y, xs, hp, mode="exact")
    lo = gp.predict_local(pkg.KernelType.MATERN52, x, y, xs, hp, tol=1e-12, max_iter=500, k_nn=64,
                          preconditioner="nystrom", precond_rank=20)
    assert rel_max(lo.stddev, ex.stddev) <= 1e-8
    assert rel_max(lo.mean, ex.mean) <= 1e-8
    # cross kNN against numpy (distances, ties to the lower index)
    nbr = torch.empty((25, 7), dtype=torch.int64, device="cuda")
    xd, xsd = torch.from_numpy(x).cuda(), torch.from_numpy(xs).cuda()
    _lib.call("kgp_knn_cross", 25, xsd.data_ptr(), 60, xd.data_ptr(), 2, 7, nbr.data_ptr(), None)
    d2 = orc.sqdist(xs, x)
    want = np.array([np.lexsort((np.arange(60), r))[:7] for r in d2])
    np.testing.assert_array_equal(nbr.cpu().numpy(), want)
    # short length scale, 3000 points: 64 neighbours carry almost all the information
    x = rng.uniform(0, 1, (3000, 2))
    y = np.cos(6 * x[:, 1]) + 0.05 * rng.standard_normal(3000)
    xs = rng.uniform(0, 1, (200, 2))
    hp = _hp(pkg, 0.05, 1.0, 1e-2)
    ex = gp.predict(pkg.KernelType.MATERN32, x, y, xs, hp, mode="exact")
    lo = gp.predict_local(pkg.KernelType.MATERN32, x, y, xs, hp, tol=1e-10, max_iter=2000, k_nn=64)
    assert np.max(np.abs(lo.stddev - ex.stddev) / ex.stddev) <= 0.05, np.max(np.abs(lo.stddev - ex.stddev) / ex.stddev)
    assert rel_max(lo.mean, ex.mean) <= 1e-6


@pytest.mark.parametrize("n", [1, 2, 31, 33, 127, 129, 4097])
@pytest.mark.parametrize("d", [1, 3, 8])
def test_fast_operator_tiny_and_ragged_n(pkg, n, d):
    """Row/column counts off the 32-column block and 128-row CTA tiles, down to one point."""
    rng = np.random.default_rng(n * 31 + d)
    x = rng.standard_normal((n, d))
    b = rng.standard_normal((n, 5))
    hp = _hp(pkg, 0.8 * np.sqrt(d), 1.1, 0.3)
    ref = pkg.KernelEngine(pkg.KernelType.MATERN52, x, hp, precision="fp64").matmul_with_grads(b)
    for prec, bar in (("fast", 2e-5), ("tf32", 1e-3)):
        got = pkg.KernelEngine(pkg.KernelType.MATERN52, x, hp, precision=prec).matmul_with_grads(b)
        assert rel_max(got[0], ref[0]) <= bar, prec
        assert rel_max(got[2], ref[2]) <= bar, prec
        if n > 1:
            assert rel_max(got[1], ref[1]) <= 10 * bar, prec


@pytest.mark.parametrize("precision", ["fp64", "fast"])
def test_grouped_pcg_narrow_tail(pkg, precision):
    """kgp_pcg_grouped with the probe group capped early: after the probes stop, the driver
    switches to a graph over the w prefix only. Column 0 must equal a standalone
    preconditioned solve of the same length and the probe columns a standalone capped solve."""
    import ctypes

    import torch

    from paper_2503_02259_b200 import _device, _lib, precond, solver

    rng = np.random.default_rng(17)
    n, kz, it1, it2 = 700, 6, 25, 6
    x = rng.uniform(0, 1, (n, 3))
    e = pkg.KernelEngine(pkg.KernelType.MATERN32, x, _hp(pkg, 0.4, 1.1, 1e-2), precision=precision,
                         mode=pkg.EngineMode.ON_THE_FLY)
    pre = precond.build(e, 40)
    yt = torch.from_numpy(rng.standard_normal((1 + kz, n))).cuda()
    k = 1 + kz
    xo = torch.empty((k, n), dtype=torch.float64, device="cuda")
    al = torch.zeros((k, it1), dtype=torch.float64, device="cuda")
    be = torch.zeros_like(al)
    it = torch.empty(k, dtype=torch.int32, device="cuda")
    rel = torch.empty(k, dtype=torch.float64, device="cuda")
    conv = torch.empty(k, dtype=torch.int32, device="cuda")
    arr = (ctypes.c_void_p * 1)(pre.handle)
    _lib.call("kgp_pcg_grouped", e.handle, arr, 1, k, 1, yt.data_ptr(), 0.0, it1, 0.0, it2, xo.data_ptr(),
              al.data_ptr(), be.data_ptr(), it.data_ptr(), rel.data_ptr(), conv.data_ptr(), _device.stream_ptr())
    its = it.cpu().numpy()
    assert its[0] == it1 and np.all(its[1:] == it2)
    w = solver.pcg_device(e, pre, yt[:1].contiguous(), 0.0, it1)
    z = solver.pcg_device(e, None, yt[1:].contiguous(), 0.0, it2)
    tol = 1e-9 if precision == "fp64" else 1e-4
    assert rel_max(xo[0].cpu().numpy(), w[0][0].cpu().numpy()) <= tol
    assert rel_max(al[0].cpu().numpy(), w[1][0].cpu().numpy()) <= tol
    assert rel_max(xo[1:].cpu().numpy(), z[0].cpu().numpy()) <= tol
    assert rel_max(al[1:, :it2].cpu().numpy(), z[1].cpu().numpy()) <= tol


@pytest.mark.parametrize("precision", ["fast", "fp64"])
def test_operator_workspace_linear_in_n(pkg, precision):
    """The on-the-fly operator never stores a kernel panel: its device workspace grows like
    n (k + d), not n^2 (the reference's scratch bound, test_kmat.py:157-182)."""
    import torch

    from paper_2503_02259_b200 import _lib

    used = []
    for n in (32768, 65536):
        torch.cuda.synchronize()
        free0 = torch.cuda.mem_get_info()[0]
        x = np.random.default_rng(n).standard_normal((n, 8))
        e = pkg.KernelEngine(pkg.KernelType.GAUSSIAN, x, _hp(pkg, 1.0, 1.0, 1e-2), precision=precision,
                             mode=pkg.EngineMode.ON_THE_FLY)
        z = torch.randn((33, n), dtype=torch.float64, device="cuda")
        o = torch.empty_like(z)
        _lib.call("kgp_engine_matmul", e.handle, 33, z.data_ptr(), 1, n, o.data_ptr(), None, None, 1, n,
                  torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        used.append(free0 - torch.cuda.mem_get_info()[0])
        e.close()
        del z, o
    n2 = 65536
    assert used[1] <= 64 * n2 * (33 + 8) * 8 + (64 << 20), used  # far below one n x n panel (34 GB)
    assert used[1] <= 2.5 * used[0] + (32 << 20), used


@pytest.mark.gpu
@pytest.mark.parametrize("n", [1, 63, 1000, 4097])
@pytest.mark.parametrize("k", [1, 3, 4, 5])
def test_dense_mode_products_match_on_the_fly(pkg, n, k):
    """DENSE mode (kmat.py:93-94): the packed symmetric product (k <= 4, symv.cu) and the
    cuBLAS product (k > 4) both equal the fp64 on-the-fly operator (kmat.py:165-189)."""
    rng = np.random.default_rng(n + 10 * k)
    x = rng.uniform(0, 1, (n, 3))
    b = rng.standard_normal((n, k))
    hp = _hp(pkg, 0.3, 1.2, 1e-2)
    import torch

    dense = pkg.KernelEngine(pkg.KernelType.MATERN52, x, hp, mode=pkg.EngineMode.DENSE)
    otf = pkg.KernelEngine(pkg.KernelType.MATERN52, x, hp, mode=pkg.EngineMode.ON_THE_FLY)
    # column-major device blocks, the PCG state's layout (the DENSE product's operand layout)
    bd = torch.from_numpy(np.ascontiguousarray(b.T)).cuda().T

    def run(e):
        out = torch.empty((k, n), dtype=torch.float64, device="cuda").T
        e.apply(bd, outs=(out, None, None))
        torch.cuda.synchronize()
        return out.cpu().numpy()

    got, ref = run(dense), run(otf)
    assert rel_max(got, ref) <= 1e-13
    assert np.array_equal(got, run(dense))  # fixed-order partial sums: run-to-run identical


@pytest.mark.gpu
@pytest.mark.parametrize("world,n,k,nout", [(3, 3000, 16, 1), (2, 4100, 33, 2), (4, 8192, 32, 2)])
def test_fused_allgather_operator_simulated_ranks(pkg, world, n, k, nout):
    """The fused all-gather operator (kgp_engine_set_peers / peer_publish / peer_matmul): every
    rank reads the other ranks' published RHS tiles inside its kernel. Ranks simulated on one
    device (all buffers local, published before any rank multiplies): each rank's rows equal
    its row block of the ordinary product -- bitwise when both use the same tile layout (same
    kernel, same column split) -- over several epochs (the ready/done flag protocol). No kernel
    here waits for a launch that has not run yet: all ranks publish before any multiplies."""
    import ctypes

    import torch

    from paper_2503_02259_b200 import _lib, dist as kdist

    rng = np.random.default_rng(world * 100 + k)
    x = rng.standard_normal((n, 8))
    hp = _hp(pkg, 1.1, 1.3, 0.05)
    starts = [kdist.row_range(n, world, q, 32)[0] for q in range(world)] + [n]
    engines, bases = [], []
    for q in range(world):
        e = pkg.KernelEngine(pkg.KernelType.GAUSSIAN, x, hp, precision="fast")
        _lib.call("kgp_engine_set_rows", e.handle, starts[q], starts[q + 1] - starts[q])
        nb, ptr = ctypes.c_int64(), ctypes.c_void_p()
        _lib.call("kgp_engine_peer_buffer_bytes", e.handle, k, starts[q + 1] - starts[q], ctypes.byref(nb))
        _lib.call("kgp_peer_alloc", nb.value, ctypes.byref(ptr), None)
        engines.append(e)
        bases.append(ptr.value)
    tiles = [kdist.PeerTiles(engines[q].handle, world, q, starts, k, bases=bases) for q in range(world)]
    st = torch.cuda.current_stream().cuda_stream
    try:
        for epoch in (1, 2, 3):
            b = torch.randn(k, n, dtype=torch.float64, device="cuda")  # (k, n): column-major blocks
            locs = [b[:, starts[q]:starts[q + 1]].contiguous() for q in range(world)]
            for q in range(world):
                nl = starts[q + 1] - starts[q]
                _lib.call("kgp_engine_peer_publish", engines[q].handle, k, locs[q].data_ptr(), 1, nl, epoch, st)
            for q in range(world):
                nl = starts[q + 1] - starts[q]
                outk = torch.empty((k, nl), dtype=torch.float64, device="cuda")
                outl = torch.empty_like(outk) if nout == 2 else None
                _lib.call("kgp_engine_peer_matmul", engines[q].handle, k, epoch, outk.data_ptr(),
                          outl.data_ptr() if outl is not None else None, None, 1, nl, st)
                ref_k = torch.empty_like(outk)
                ref_l = torch.empty_like(outk) if nout == 2 else None
                _lib.call("kgp_engine_matmul", engines[q].handle, k, b.data_ptr(), 1, n, ref_k.data_ptr(),
                          ref_l.data_ptr() if ref_l is not None else None, None, 1, nl, st)
                torch.cuda.synchronize()
                if nout == 2 and k > 32:
                    # the ordinary two-output product uses the LB layout here (bf16 lo parts);
                    # published tiles are all-tf32: same precision class, not the same bits
                    assert rel_max(outk.cpu().numpy(), ref_k.cpu().numpy()) <= 2e-5, (epoch, q)
                    assert rel_max(outl.cpu().numpy(), ref_l.cpu().numpy()) <= 2e-4, (epoch, q)
                else:
                    assert torch.equal(outk, ref_k), (epoch, q)
                    if nout == 2:
                        assert torch.equal(outl, ref_l), (epoch, q)
        # derivative-only outputs (dist_nlml_grad's grads_local: out_k NULL, dL and dF)
        epoch = 4
        b = torch.randn(k, n, dtype=torch.float64, device="cuda")
        locs = [b[:, starts[q]:starts[q + 1]].contiguous() for q in range(world)]
        for q in range(world):
            nl = starts[q + 1] - starts[q]
            _lib.call("kgp_engine_peer_publish", engines[q].handle, k, locs[q].data_ptr(), 1, nl, epoch, st)
        for q in range(world):
            nl = starts[q + 1] - starts[q]
            dl, df = (torch.empty((k, nl), dtype=torch.float64, device="cuda") for _ in range(2))
            _lib.call("kgp_engine_peer_matmul", engines[q].handle, k, epoch, None, dl.data_ptr(), df.data_ptr(), 1,
                      nl, st)
            rl, rf = torch.empty_like(dl), torch.empty_like(df)
            _lib.call("kgp_engine_matmul", engines[q].handle, k, b.data_ptr(), 1, n, None, rl.data_ptr(),
                      rf.data_ptr(), 1, nl, st)
            torch.cuda.synchronize()
            tol_l = 2e-4 if k > 32 else 0.0  # LB layout in the ordinary two-output product for k > 32
            assert rel_max(dl.cpu().numpy(), rl.cpu().numpy()) <= tol_l, q
            assert rel_max(df.cpu().numpy(), rf.cpu().numpy()) <= (2e-5 if k > 32 else 0.0), q
    finally:
        for t in tiles:
            t.close()
        for p in bases:
            _lib.call("kgp_peer_free", p)


@pytest.mark.gpu
def test_fused_allgather_operator_errors(pkg):
    import ctypes

    from paper_2503_02259_b200 import _lib
    from paper_2503_02259_b200.errors import KernelGpError

    x = np.random.default_rng(0).standard_normal((256, 3))
    e64 = pkg.KernelEngine(pkg.KernelType.GAUSSIAN, x, _hp(pkg, 1, 1, 0.1), precision="fp64")
    starts = (ctypes.c_int64 * 3)(0, 128, 256)
    ptrs = (ctypes.c_void_p * 2)(1, 1)
    with pytest.raises(ValueError, match="tensor-core"):
        _lib.call("kgp_engine_set_peers", e64.handle, 2, 0, starts, ptrs, 4)
    ef = pkg.KernelEngine(pkg.KernelType.GAUSSIAN, x, _hp(pkg, 1, 1, 0.1), precision="fast")
    with pytest.raises(KernelGpError, match="no peer configuration"):
        _lib.call("kgp_engine_peer_publish", ef.handle, 4, 1, 1, 256, 1, None)
    _lib.call("kgp_engine_set_rows", ef.handle, 0, 128)
    bad = (ctypes.c_int64 * 3)(0, 100, 256)
    with pytest.raises(ValueError, match="multiples of 32"):
        _lib.call("kgp_engine_set_peers", ef.handle, 2, 0, bad, ptrs, 4)
    with pytest.raises(ValueError, match="not rank 1"):
        _lib.call("kgp_engine_set_peers", ef.handle, 2, 1, starts, ptrs, 4)
    # a peer configuration is valid only for the precision and row block it was made with
    # (ADVICE r1): a later set_precision / set_rows makes publish and peer_matmul refuse
    import ctypes as ct

    nb, ptr = ct.c_int64(), ct.c_void_p()
    one = (ct.c_int64 * 2)(0, 256)
    _lib.call("kgp_engine_set_rows", ef.handle, 0, 256)
    _lib.call("kgp_engine_peer_buffer_bytes", ef.handle, 4, 256, ct.byref(nb))
    _lib.call("kgp_peer_alloc", nb.value, ct.byref(ptr), None)
    try:
        _lib.call("kgp_engine_set_peers", ef.handle, 1, 0, one, (ct.c_void_p * 1)(ptr.value), 4)
        _lib.call("kgp_engine_set_precision", ef.handle, 2)  # tf32
        with pytest.raises(KernelGpError, match="precision changed"):
            _lib.call("kgp_engine_peer_publish", ef.handle, 4, 1, 1, 256, 1, None)
        _lib.call("kgp_engine_set_precision", ef.handle, 1)
        _lib.call("kgp_engine_set_rows", ef.handle, 0, 128)
        with pytest.raises(KernelGpError, match="rows changed"):
            _lib.call("kgp_engine_peer_matmul", ef.handle, 4, 1, 1, None, None, 1, 128, None)
    finally:
        _lib.call("kgp_peer_free", ptr.value)
