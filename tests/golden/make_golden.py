"""Generate golden fixtures by running the REAL reference (kernelgp, /root/reference/pkg).

Run in the build container only (the reference does not exist on the GPU box):

    python tests/golden/make_golden.py

The reference is imported from a scratch copy under /tmp because numba's
``cache=True`` writes next to the source. Every fixture stores its
inputs next to the reference outputs, so tests never need the reference or
numpy's RNG stream to match. Outputs go to ``tests/golden/*.npz``.
"""

from __future__ import annotations

import os
import shutil
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF_PKG = "/root/reference/pkg"


def _import_reference():
    scratch = os.path.join(tempfile.gettempdir(), "kgp_ref_golden")
    if not os.path.isdir(scratch):
        shutil.copytree(REF_PKG, scratch)
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tempfile.gettempdir(), "kgp_numba"))
    sys.path.insert(0, os.path.join(scratch, "src"))
    import kernelgp  # noqa: F401
    return scratch


def _pad_traces(traces, width=None):
    m = max([t.iterations for t in traces] + [1])
    width = width or m
    a = np.full((len(traces), width), np.nan)
    b = np.full((len(traces), width), np.nan)
    it = np.zeros(len(traces), dtype=np.int64)
    rel = np.zeros(len(traces))
    for j, t in enumerate(traces):
        a[j, : t.iterations] = t.alphas
        b[j, : len(t.betas)] = t.betas
        it[j] = t.iterations
        rel[j] = t.final_rel_residual
    return a, b, it, rel


def main():
    _import_reference()
    from kernelgp import backends, gp, precond, solver, train
    from kernelgp.kernels import KernelType, eval_kernel, eval_kernel_grad_l, pairwise_sq_dist
    from kernelgp.kmat import EngineMode, Hyperparams, KernelEngine, Theta

    sys.path.insert(0, REPO)
    from paper_2503_02259_b200 import workloads

    kts = [KernelType.GAUSSIAN, KernelType.MATERN32, KernelType.MATERN52]
    out = {}

    # --- panels: both reference backends (kernels.py:79-94, _panels_*.py) -----------
    rng = np.random.default_rng(1)
    x = rng.standard_normal((23, 3))
    y = rng.standard_normal((17, 3))
    y[0] = x[0]  # a coincident pair: dk/dl must be exactly 0 there
    out["panel_x"], out["panel_y"], out["panel_l"] = x, y, 0.7
    for bname in ("numba", "numpy"):
        os.environ["KERNELGP_BACKEND"] = bname
        out[f"sqdist_{bname}"] = pairwise_sq_dist(x, y)
        for kt in kts:
            out[f"K_{kt.value}_{bname}"] = eval_kernel(kt, x, y, 0.7)
            out[f"G_{kt.value}_{bname}"] = eval_kernel_grad_l(kt, x, y, 0.7)
    os.environ.pop("KERNELGP_BACKEND")
    np.savez_compressed(os.path.join(HERE, "panels.npz"), **out)

    # --- engine: OTF matmul / grad_matmul (kmat.py:145-189) ---------------------------
    out = {}
    cases = [
        ("a", 300, 3, 5, KernelType.GAUSSIAN, (0.9, 1.3, 0.2), 64, 11),
        ("b", 300, 3, 5, KernelType.MATERN32, (0.9, 1.3, 0.2), 64, 11),
        ("c", 300, 3, 5, KernelType.MATERN52, (0.9, 1.3, 0.2), 64, 11),
        ("d", 257, 1, 1, KernelType.MATERN52, (0.5, 0.8, 0.05), 256, 12),
        ("e", 130, 8, 17, KernelType.GAUSSIAN, (2.0, 0.7, 1e-2), 41, 13),
        ("f", 97, 2, 33, KernelType.MATERN32, (0.2, 1.5, 1e-3), 256, 14),
        ("g", 1, 1, 1, KernelType.GAUSSIAN, (1.0, 2.0, 0.1), 256, 15),
    ]
    for tag, n, d, k, kt, (l, f, s), bs, seed in cases:
        r = np.random.default_rng(seed)
        xx = r.standard_normal((n, d))
        bb = r.standard_normal((n, k))
        hp = Hyperparams(l=l, f=f, s=s)
        e = KernelEngine(kt, xx, hp, mode=EngineMode.ON_THE_FLY, block_size=bs)
        out[f"{tag}_x"], out[f"{tag}_b"] = xx, bb
        out[f"{tag}_meta"] = np.array([n, d, k, l, f, s, bs])
        out[f"{tag}_kt"] = np.array(kt.value)
        out[f"{tag}_K"] = e.matmul(bb)
        for th in (Theta.L, Theta.F, Theta.S):
            out[f"{tag}_d{th.value}"] = e.grad_matmul(th, bb)
    np.savez_compressed(os.path.join(HERE, "engine.npz"), **out)

    # --- solver: batched PCG with/without Nystrom, SLQ (solver.py:122-265) -----------
    out = {}
    r = np.random.default_rng(21)
    n = 200
    xx = r.standard_normal((n, 2))
    hp = Hyperparams(l=1.1, f=1.2, s=0.05)
    e = KernelEngine(KernelType.GAUSSIAN, xx, hp, mode=EngineMode.ON_THE_FLY)
    yy = r.standard_normal((n, 4))
    yy[:, 2] = 0.0  # zero column: zero-iteration trace
    pre = precond.build(e, 40)
    out["x"], out["y"], out["hp"] = xx, yy, np.array([hp.l, hp.f, hp.s])
    for tag, minv in (("plain", None), ("nys", pre.apply_inverse)):
        rep = solver.pcg_solve(e.matmul, minv, yy, tol=1e-8, max_iter=500)
        a, b, it, rel = _pad_traces(rep.traces)
        out[f"{tag}_sol"], out[f"{tag}_alphas"], out[f"{tag}_betas"] = rep.solution, a, b
        out[f"{tag}_iters"], out[f"{tag}_rel"] = it, rel
        out[f"{tag}_conv"] = np.array(rep.converged)
    z = gp.ProbeSet.generate(n, 6, 5)
    rep = solver.pcg_solve(e.matmul, None, z.vectors, tol=1e-10, max_iter=500)
    out["probes"], out["probe_norms"] = z.vectors, z.norms_sq
    a, b, it, rel = _pad_traces(rep.traces)
    out["probe_alphas"], out["probe_betas"], out["probe_iters"] = a, b, it
    out["slq_logdet"] = solver.slq_logdet(rep.traces, z.norms_sq)
    out["logdet_exact"] = np.linalg.slogdet(e.materialize())[1]
    # fixed-iteration mode (tol=0) on the same system
    rep = solver.pcg_solve(e.matmul, None, z.vectors, tol=0.0, max_iter=7)
    a, b, it, rel = _pad_traces(rep.traces)
    out["fixed_alphas"], out["fixed_betas"], out["fixed_sol"] = a, b, rep.solution
    out["fixed_slq"] = solver.slq_logdet(rep.traces, z.norms_sq)
    np.savez_compressed(os.path.join(HERE, "solver.npz"), **out)

    # --- preconditioner: FPS + Woodbury (precond.py:39-126) --------------------------
    out = {}
    r = np.random.default_rng(31)
    xx = r.standard_normal((500, 3))
    out["fps_x"] = xx
    out["fps_idx"] = precond.fps_select(xx, 50, seed_index=0)
    out["fps_idx_seed7"] = precond.fps_select(xx, 20, seed_index=7)
    grid = np.repeat(np.arange(6.0), 3)[:, None]  # many exact ties
    out["fps_tie_x"], out["fps_tie_idx"] = grid, precond.fps_select(grid, 6, seed_index=0)
    for kt in kts:
        hp = Hyperparams(l=0.8, f=1.1, s=0.02)
        e = KernelEngine(kt, xx, hp)
        p = precond.build(e, 60)
        bb = r.standard_normal((500, 3))
        out[f"{kt.value}_b"] = bb
        out[f"{kt.value}_idx"] = p.landmark_indices
        out[f"{kt.value}_minv"] = p.apply_inverse(bb)
        out[f"{kt.value}_m"] = p.apply(bb)
    np.savez_compressed(os.path.join(HERE, "precond.npz"), **out)

    # --- NLML + gradient (gp.py:107-179) ----------------------------------------------
    out = {}
    w = workloads.cfg1(n=1024, seed=0)
    hp = Hyperparams(l=w.l, f=w.f, s=w.s)
    e = KernelEngine(KernelType.GAUSSIAN, w.x, hp, mode=EngineMode.ON_THE_FLY)
    probes = gp.ProbeSet.generate(w.n, w.k_z, w.probe_seed)
    pre = precond.build(e, 128)
    out["x"], out["y"], out["probes"] = w.x, w.y, probes.vectors
    out["hp"] = np.array([hp.l, hp.f, hp.s])
    out["rank"] = 128
    ex = gp.grad_exact(KernelEngine(KernelType.GAUSSIAN, w.x, hp, mode=EngineMode.DENSE), w.y)
    out["exact"] = np.array([ex.loss, ex.grad_l, ex.grad_f, ex.grad_s])
    for tag, tol, ptol in (("tight", 1e-10, 1e-10), ("default", 1e-6, 1e-2)):
        lg = gp.nlml_grad_iterative(e, w.y, pre, probes, tol=tol, max_iter=3000, probe_tol=ptol)
        out[f"iter_{tag}"] = np.array([lg.loss, lg.grad_l, lg.grad_f, lg.grad_s, lg.converged])
    # the fixed recipe of configs[0]: PCG 50 + 20-step probe CG + SLQ
    wr = solver.pcg_solve(e.matmul, pre.apply_inverse, w.y, tol=0.0, max_iter=50)
    ur = solver.pcg_solve(e.matmul, None, probes.vectors, tol=0.0, max_iter=20)
    out["fixed_logdet"] = solver.slq_logdet(ur.traces, probes.norms_sq)
    out["fixed_w"] = wr.solution
    # Matern kernels at a smaller size, tight tolerance
    for kt in (KernelType.MATERN32, KernelType.MATERN52):
        r = np.random.default_rng(41)
        xx = r.uniform(0, 1, (400, 2))
        yy = np.sin(3 * xx).sum(1) + 0.05 * r.standard_normal(400)
        hp2 = Hyperparams(l=0.25, f=1.5, s=1e-2)
        e2 = KernelEngine(kt, xx, hp2, mode=EngineMode.ON_THE_FLY)
        pr2 = gp.ProbeSet.generate(400, 8, 3)
        lg = gp.nlml_grad_iterative(e2, yy, precond.build(e2, 40), pr2, tol=1e-10,
                                    max_iter=3000, probe_tol=1e-10)
        out[f"{kt.value}_x"], out[f"{kt.value}_y"], out[f"{kt.value}_probes"] = xx, yy, pr2.vectors
        out[f"{kt.value}_res"] = np.array([lg.loss, lg.grad_l, lg.grad_f, lg.grad_s])
        ex2 = gp.grad_exact(KernelEngine(kt, xx, hp2), yy)
        out[f"{kt.value}_exact"] = np.array([ex2.loss, ex2.grad_l, ex2.grad_f, ex2.grad_s])
    np.savez_compressed(os.path.join(HERE, "nlml.npz"), **out)

    # full configs[0] size, tolerance mode: inputs are regenerated from the seed by
    # workloads.cfg1 (checksummed here), outputs pinned
    out = {}
    w = workloads.cfg1(n=4096, seed=0)
    hp = Hyperparams(l=w.l, f=w.f, s=w.s)
    e = KernelEngine(KernelType.GAUSSIAN, w.x, hp, mode=EngineMode.DENSE)
    probes = gp.ProbeSet.generate(w.n, w.k_z, w.probe_seed)
    pre = precond.build(e, w.rank)
    lg = gp.nlml_grad_iterative(e, w.y, pre, probes, tol=1e-10, max_iter=3000, probe_tol=1e-10)
    out["checksum"] = np.array([np.sum(w.x ** 2), np.sum(w.y ** 2), np.sum(probes.vectors ** 2)])
    out["iter_tight"] = np.array([lg.loss, lg.grad_l, lg.grad_f, lg.grad_s])
    wr = solver.pcg_solve(e.matmul, pre.apply_inverse, w.y, tol=0.0, max_iter=50)
    ur = solver.pcg_solve(e.matmul, None, probes.vectors, tol=0.0, max_iter=20)
    out["fixed_logdet"] = solver.slq_logdet(ur.traces, probes.norms_sq)
    ex = gp.grad_exact(e, w.y)
    out["exact"] = np.array([ex.loss, ex.grad_l, ex.grad_f, ex.grad_s])
    np.savez_compressed(os.path.join(HERE, "cfg1_full.npz"), **out)

    # --- prediction (gp.py:182-244) ----------------------------------------------------
    out = {}
    r = np.random.default_rng(51)
    xx = r.uniform(-2, 2, (300, 2))
    yy = np.sin(xx[:, 0] * 2) + 0.05 * r.standard_normal(300)
    xs = np.vstack([xx[:30] + 0.01, r.uniform(-2, 2, (10, 2))])
    out["x"], out["y"], out["xs"] = xx, yy, xs
    hp = Hyperparams(l=0.8, f=1.0, s=0.05)
    for kt in kts:
        ex = gp.predict(kt, xx, yy, xs, hp, mode="exact")
        it = gp.predict(kt, xx, yy, xs, hp, mode="iterative", tol=1e-10, max_iter=2000)
        out[f"{kt.value}_exact_mean"], out[f"{kt.value}_exact_sd"] = ex.mean, ex.stddev
        out[f"{kt.value}_iter_mean"], out[f"{kt.value}_iter_sd"] = it.mean, it.stddev
    np.savez_compressed(os.path.join(HERE, "predict.npz"), **out)

    # --- training (train.py:176-240) ---------------------------------------------------
    out = {}
    r = np.random.default_rng(61)
    xx = r.uniform(-2, 2, (120, 2))
    yy = np.sin(xx[:, 0]) + 0.1 * r.standard_normal(120)
    out["x"], out["y"] = xx, yy
    res = train.fit(KernelType.MATERN52, xx, yy,
                    train.TrainConfig(learning_rate=0.1, max_steps=15, mode="exact", rng_seed=3))
    out["exact_loss"] = np.array(res.loss_history)
    out["exact_params"] = np.array([res.params.l, res.params.f, res.params.s])
    res = train.fit(KernelType.MATERN52, xx, yy,
                    train.TrainConfig(learning_rate=0.1, max_steps=6, mode="iterative",
                                      rng_seed=3, tol=1e-10, probe_tol=1e-10, max_iter=2000))
    out["iter_loss"] = np.array(res.loss_history)
    out["iter_params"] = np.array([res.params.l, res.params.f, res.params.s])
    init = train.initial_hyperparams(xx, yy, 3)
    out["init"] = np.array([init.l, init.f, init.s])
    np.savez_compressed(os.path.join(HERE, "train.npz"), **out)
    print("golden fixtures written to", HERE, "backend", backends.backend_name())


def main_cfg3(n: int = 16384):
    """configs[2]'s generator (Matern-3/2, d=4, X~U[0,1]^4 fp32, l=0.2 f=1.5 s=1e-3, 32 probes)
    at reduced n through the reference's OWN estimator (gp.py:133-179: Nystrom rank 1024
    w-solve, unpreconditioned probe CG, SLQ) in tolerance mode, tol = probe_tol = 1e-10, the
    reference's default engine mode (auto -> DENSE at n <= 20000; DENSE vs ON_THE_FLY agree to
    ~1e-11 in this mode). n = 8192: ~2 min on 8 cores; n = 16384: ~1 h (3400+
    probe CG iterations over a 2 GB dense Khat).

        python tests/golden/make_golden.py cfg3 [n]
    """
    import time

    _import_reference()
    from kernelgp import gp, precond
    from kernelgp.kernels import KernelType
    from kernelgp.kmat import Hyperparams, KernelEngine

    sys.path.insert(0, REPO)
    from paper_2503_02259_b200 import workloads

    w = workloads.cfg3(n=n)
    hp = Hyperparams(l=w.l, f=w.f, s=w.s)
    e = KernelEngine(KernelType.MATERN32, w.x, hp)
    probes = gp.ProbeSet.generate(w.n, w.k_z, w.probe_seed)
    t0 = time.time()
    pre = precond.build(e, w.rank)
    lg = gp.nlml_grad_iterative(e, w.y, pre, probes, tol=1e-10, max_iter=6000, probe_tol=1e-10)
    out = {"n": np.array(n), "mode": np.array(str(e.mode.value)),
           "checksum": np.array([np.sum(w.x ** 2), np.sum(w.y ** 2), np.sum(probes.vectors ** 2)]),
           "iter_tight": np.array([lg.loss, lg.grad_l, lg.grad_f, lg.grad_s]),
           "converged": np.array(bool(lg.converged)), "seconds": np.array(time.time() - t0)}
    name = "cfg3_small.npz" if n == 16384 else f"cfg3_small_n{n}.npz"
    np.savez_compressed(os.path.join(HERE, name), **out)
    print(name, out)


if __name__ == "__main__":
    if sys.argv[1:2] == ["cfg3"]:
        main_cfg3(int(sys.argv[2]) if len(sys.argv) > 2 else 16384)
    else:
        main()
