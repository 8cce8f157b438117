"""Validate the NLML CPU baseline against the real reference (build container only).

configs[0] fixed recipe (n=4096, Gaussian, 16 probes, Nystrom 256; PCG 50 + 20-step probe
CG + SLQ + gradient), timed three ways on this host's cores:
  * kernelgp itself (the reference, auto -> DENSE mode, numba prange panels + BLAS), the
    recipe composed from its public functions (gp.py:154-177 with the probe CG capped at 20);
  * oracle/kgp_oracle.py dense path with numpy panels (round 1's baseline);
  * oracle/kgp_oracle.py dense path with the OpenMP C panels (panels="c", bench.py's baseline).
Preconditioner builds are excluded from all three (timed separately, as bench.py does).

    python tools/cpu_nlml_baseline.py [reps]
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests", "golden"))


def best(fn, reps):
    fn()
    t = []
    for _ in range(reps):
        t0 = time.perf_counter()
        out = fn()
        t.append(time.perf_counter() - t0)
    return min(t), out


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    from oracle import kgp_oracle as orc
    from paper_2503_02259_b200 import workloads

    w = workloads.cfg1()
    probes = np.random.default_rng(w.probe_seed).standard_normal((w.n, w.k_z))
    res = {}
    try:
        import make_golden

        make_golden._import_reference()
        from kernelgp import gp, precond, solver
        from kernelgp.kernels import KernelType
        from kernelgp.kmat import Hyperparams, KernelEngine, Theta

        e = KernelEngine(KernelType.GAUSSIAN, w.x, Hyperparams(w.l, w.f, w.s))
        pre = precond.build(e, w.rank)
        pset = gp.ProbeSet(probes)

        def ref_eval():
            # a fresh engine per eval, as train.fit builds one per step (train.py:198-204): the
            # DENSE materialisation of Khat is part of every evaluation, as in the oracle's
            e = KernelEngine(KernelType.GAUSSIAN, w.x, Hyperparams(w.l, w.f, w.s))
            wr = solver.pcg_solve(e.matmul, pre.apply_inverse, w.y, tol=0.0, max_iter=50)
            ur = solver.pcg_solve(e.matmul, None, pset.vectors, tol=0.0, max_iter=20)
            logdet = solver.slq_logdet(ur.traces, pset.norms_sq)
            wv = wr.solution
            loss = 0.5 * (float(w.y @ wv) + logdet + w.n * gp.LOG_2PI)
            v = np.column_stack([wv, pset.vectors])
            for th in (Theta.L, Theta.F, Theta.S):
                dv = e.grad_matmul(th, v)
                _ = -float(wv @ dv[:, 0]) + float(np.einsum("ij,ij->", ur.solution, dv[:, 1:])) / w.k_z
            return loss

        res["kernelgp"] = best(ref_eval, reps)
        print(f"kernelgp (mode {e.mode.value}): {res['kernelgp'][0]:.3f} s  loss {res['kernelgp'][1]:.10g}")
    except Exception as exc:  # not importable (e.g. on the GPU box)
        print("kernelgp not importable:", exc)
    ny = orc.Nystrom("gaussian", w.x, w.l, w.f, w.s, w.rank)
    for panels in ("numpy", "c"):
        def ev(panels=panels):
            return orc.nlml_grad("gaussian", w.x, w.y, w.l, w.f, w.s, probes, ny, tol=0.0, max_iter=50,
                                 probe_tol=0.0, dense=True, probe_max_iter=20, panels=panels)[0]
        res[panels] = best(ev, reps)
        print(f"oracle dense, {panels} panels: {res[panels][0]:.3f} s  loss {res[panels][1]:.10g}")
    if "kernelgp" in res:
        print(f"ratio oracle(c) / kernelgp = {res['c'][0] / res['kernelgp'][0]:.2f}; "
              f"oracle(numpy) / kernelgp = {res['numpy'][0] / res['kernelgp'][0]:.2f}; cores {os.cpu_count()}")


if __name__ == "__main__":
    main()
