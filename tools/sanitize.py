"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck / initcheck).

    compute-sanitizer --tool memcheck python tools/sanitize.py [section ...]

Sections: nlml64 (kmm_f64, PCG graph, dots, Woodbury, SLQ), fast (kmm_tc + column-split
reduction, fast NLML), dense (DENSE-mode panel + packed symmetric product), afn (kNN, FSAI,
sparse G products, level solves, probe sampling), gpc (diag shift, grouped solve), local
(cross kNN + local variance), peer (fused all-gather operator with two ranks simulated on one
device: publish both, then both multiply -- no kernel waits on an unlaunched one).
Each section checks its result against numpy so a sanitizer run is also a correctness run.
"""

from __future__ import annotations

import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2503_02259_b200 as kgp  # noqa: E402
from paper_2503_02259_b200 import _lib, gp, gpc, precond, solver  # noqa: E402
from paper_2503_02259_b200 import dist as kdist  # noqa: E402


def dense_khat(kt, x, hp):
    e = kgp.KernelEngine(kt, x, hp, precision="fp64")
    return e.materialize()


def sec_nlml64():
    rng = np.random.default_rng(1)
    n = 700
    x = rng.uniform(0, 1, (n, 3))
    y = np.sin(5 * x[:, 0]) + 0.1 * rng.standard_normal(n)
    e = kgp.KernelEngine(kgp.KernelType.GAUSSIAN, x, kgp.Hyperparams(0.3, 1.0, 1e-2), precision="fp64")
    probes = gp.ProbeSet.generate(n, 4, 0)
    lg = gp.nlml_grad_iterative(e, y, precond.build(e, 40), probes, tol=1e-8, max_iter=500)
    ex = gp.grad_exact(e, y)
    assert abs(lg.loss - ex.loss) < 0.05 * abs(ex.loss) + 5, (lg, ex)
    z = rng.standard_normal((n, 3))
    a, b, c = e.matmul_with_grads(z)
    k = e.materialize()
    assert np.abs(a - k @ z).max() <= 1e-10 * np.abs(k @ z).max()
    rep = solver.cg_solve(e.matmul, y, tol=1e-10, max_iter=400)
    print("nlml64 ok", lg.loss)


def sec_fast():
    rng = np.random.default_rng(2)
    n = 1100
    x = rng.standard_normal((n, 8))
    e = kgp.KernelEngine(kgp.KernelType.GAUSSIAN, x, kgp.Hyperparams(1.0, 1.0, 1e-2), precision="fast")
    z = rng.standard_normal((n, 32))
    a, b, _ = e.matmul_with_grads(z)
    k = dense_khat(kgp.KernelType.GAUSSIAN, x, kgp.Hyperparams(1.0, 1.0, 1e-2))
    assert np.abs(a - k @ z).max() <= 2e-5 * np.abs(k @ z).max()
    x2 = rng.uniform(0, 1, (n, 4))
    e2 = kgp.KernelEngine(kgp.KernelType.MATERN32, x2, kgp.Hyperparams(0.2, 1.5, 1e-3), precision="fast")
    z2 = rng.standard_normal((n, 33))
    a2 = e2.matmul(z2)
    k2 = dense_khat(kgp.KernelType.MATERN32, x2, kgp.Hyperparams(0.2, 1.5, 1e-3))
    assert np.abs(a2 - k2 @ z2).max() <= 2e-5 * np.abs(k2 @ z2).max()
    y = rng.standard_normal(n)
    gp.nlml_grad_iterative(e2, y, precond.build(e2, 40), gp.ProbeSet.generate(n, 4, 0), tol=1e-6, max_iter=300)
    print("fast ok")


def sec_dense():
    rng = np.random.default_rng(3)
    n = 900
    x = rng.uniform(0, 1, (n, 3))
    hp = kgp.Hyperparams(0.3, 1.0, 1e-2)
    e = kgp.KernelEngine(kgp.KernelType.GAUSSIAN, x, hp, mode=kgp.EngineMode.DENSE, precision="fp64")
    v = rng.standard_normal(n)
    k = dense_khat(kgp.KernelType.GAUSSIAN, x, hp)
    assert np.abs(e.matmul(v) - k @ v).max() <= 1e-12 * np.abs(k @ v).max()
    z = rng.standard_normal((n, 17))
    assert np.abs(e.matmul(z) - k @ z).max() <= 1e-12 * np.abs(k @ z).max()
    y = np.sin(4 * x[:, 1])
    gp.nlml_grad_iterative(e, y, precond.build(e, 32), gp.ProbeSet.generate(n, 16, 0), tol=0.0, max_iter=30,
                           probe_tol=0.0, probe_max_iter=10)
    print("dense ok")


def sec_afn():
    rng = np.random.default_rng(4)
    n = 1500
    x = rng.uniform(0, 1, (n, 4))
    hp = kgp.Hyperparams(0.2, 1.5, 1e-3)
    e = kgp.KernelEngine(kgp.KernelType.MATERN32, x, hp, precision="fp64")
    afn = precond.build_afn(e, 64, fsai_npt=8)
    y = rng.standard_normal(n)
    rep = solver.pcg_solve(e.matmul, afn.apply_inverse, y, tol=1e-10, max_iter=2000)
    k = dense_khat(kgp.KernelType.MATERN32, x, hp)
    w = np.linalg.solve(k, y)
    assert rep.converged[0] and np.abs(rep.solution - w).max() <= 1e-6 * np.abs(w).max()
    yy = rng.standard_normal((n, 12))
    afn.apply_inverse(yy)
    probes = gp.ProbeSet.generate(n, 4, 0)
    gp.nlml_grad_iterative(e, y, afn, probes, tol=1e-6, max_iter=500, preconditioned_probes=True)
    print("afn ok")


def sec_gpc():
    rng = np.random.default_rng(5)
    n = 600
    x = rng.standard_normal((n, 3))
    lab = (x[:, 0] > 0).astype(int) + (x[:, 1] > 0.5).astype(int)
    prob = gpc.setup(x, lab, 3)
    e = kgp.KernelEngine(kgp.KernelType.GAUSSIAN, x, kgp.Hyperparams(1.0, 1.0, 0.1), precision="fp64")
    pres = gpc.build_preconditioners(e, prob, 32, kind="afn", fsai_npt=8)
    z = gpc.generate_probes(n, 3, 4, 0)
    lg = gpc.nlml_grad_iterative(e, prob, pres, z, tol=1e-8, max_iter=500)
    print("gpc ok", lg.loss)


def sec_local():
    rng = np.random.default_rng(6)
    n, m = 800, 50
    x = rng.uniform(0, 1, (n, 2))
    y = np.sin(4 * x[:, 0])
    xs = rng.uniform(0, 1, (m, 2))
    pr = gp.predict_local(kgp.KernelType.MATERN52, x, y, xs, kgp.Hyperparams(0.1, 1.0, 1e-2), k_nn=32,
                          precond_rank=32, precision="fp64")
    assert np.isfinite(pr.stddev).all()
    print("local ok")


def sec_peer():
    rng = np.random.default_rng(7)
    n, k, world = 2100, 16, 2
    x = rng.standard_normal((n, 8))
    hp = kgp.Hyperparams(1.1, 1.3, 0.05)
    starts = [kdist.row_range(n, world, q, 32)[0] for q in range(world)] + [n]
    engines, bases = [], []
    for q in range(world):
        e = kgp.KernelEngine(kgp.KernelType.GAUSSIAN, x, hp, precision="fast")
        _lib.call("kgp_engine_set_rows", e.handle, starts[q], starts[q + 1] - starts[q])
        nb, ptr = ctypes.c_int64(), ctypes.c_void_p()
        _lib.call("kgp_engine_peer_buffer_bytes", e.handle, k, starts[q + 1] - starts[q], ctypes.byref(nb))
        _lib.call("kgp_peer_alloc", nb.value, ctypes.byref(ptr), None)
        engines.append(e)
        bases.append(ptr.value)
    tiles = [kdist.PeerTiles(engines[q].handle, world, q, starts, k, bases=bases) for q in range(world)]
    st = torch.cuda.current_stream().cuda_stream
    for epoch in (1, 2):
        b = torch.randn(k, n, dtype=torch.float64, device="cuda")
        locs = [b[:, starts[q]:starts[q + 1]].contiguous() for q in range(world)]
        for q in range(world):
            nl = starts[q + 1] - starts[q]
            _lib.call("kgp_engine_peer_publish", engines[q].handle, k, locs[q].data_ptr(), 1, nl, epoch, st)
        for q in range(world):
            nl = starts[q + 1] - starts[q]
            outk = torch.empty((k, nl), dtype=torch.float64, device="cuda")
            _lib.call("kgp_engine_peer_matmul", engines[q].handle, k, epoch, outk.data_ptr(), None, None, 1, nl, st)
            ref = torch.empty_like(outk)
            _lib.call("kgp_engine_matmul", engines[q].handle, k, b.data_ptr(), 1, n, ref.data_ptr(), None, None,
                      1, nl, st)
            torch.cuda.synchronize()
            assert torch.equal(outk, ref)
    for t in tiles:
        t.close()
    for p in bases:
        _lib.call("kgp_peer_free", p)
    print("peer ok")


SECTIONS = {"nlml64": sec_nlml64, "fast": sec_fast, "dense": sec_dense, "afn": sec_afn, "gpc": sec_gpc,
            "local": sec_local, "peer": sec_peer}

if __name__ == "__main__":
    names = sys.argv[1:] or list(SECTIONS)
    for nm in names:
        SECTIONS[nm]()
    torch.cuda.synchronize()
    print("sanitize workloads done:", " ".join(names))
