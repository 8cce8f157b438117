"""Predictive-variance approximations vs the exact variance (gp.py:240-243) on the configs[4]
generator at reduced n, m (diagnostic): local kriging (k nearest) and DTC over FPS landmarks.
python tools/variance_methods.py [n] [m]"""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2503_02259_b200 as kgp
from paper_2503_02259_b200 import gp, precond, workloads
from paper_2503_02259_b200.kernels import device_panel

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
m = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
w = workloads.cfg5(n=n, m_test=m)
xs = w.extra["xstar"]
hp = kgp.Hyperparams(w.l, w.f, w.s)
ex = gp.predict(kgp.KernelType.MATERN52, w.x, w.y, xs, hp, mode="exact", dense_budget=max(n, 20000))
print(f"n={n} m={m}: exact stddev mean {ex.stddev.mean():.4e} min {ex.stddev.min():.4e} max {ex.stddev.max():.4e}")
for knn in (64, 128):
    lo = gp.predict_local(kgp.KernelType.MATERN52, w.x, w.y, xs, hp, tol=1e-10, max_iter=3000, k_nn=knn,
                          precision="fp64", preconditioner="afn", precond_rank=512)
    err = np.abs(lo.stddev - ex.stddev) / ex.stddev
    print(f"local k={knn}: max rel err {err.max():.3e} mean {err.mean():.3e}")
xd = torch.from_numpy(w.x).cuda()
xsd = torch.from_numpy(xs).cuda()
kid = 2
f2 = w.f ** 2
for r in (512, 1024, 2048, 4096):
    if r > n:
        continue
    idx = precond.fps_device(xd, r, 0)
    xm = xd.index_select(0, idx)
    kmm = f2 * device_panel(kid, 0, xm, xm, w.l)
    kmm.diagonal().add_(1e-10 * float(torch.trace(kmm)) / r)
    L = torch.linalg.cholesky(kmm)
    knm = f2 * device_panel(kid, 0, xd, xm, w.l)          # n x r
    U = torch.linalg.solve_triangular(L, knm.T, upper=False).T  # n x r
    A = U.T @ U
    B = A @ torch.linalg.inv(A + w.s * torch.eye(r, dtype=torch.float64, device="cuda"))
    B = 0.5 * (B + B.T)
    ksm = f2 * device_panel(kid, 0, xsd, xm, w.l)         # m x r
    us = torch.linalg.solve_triangular(L, ksm.T, upper=False)  # r x m
    var = f2 - (us * (B @ us)).sum(0)
    sd = torch.sqrt(torch.clamp(var, min=0)).cpu().numpy()
    err = np.abs(sd - ex.stddev) / ex.stddev
    print(f"DTC r={r}: max rel err {err.max():.3e} mean {err.mean():.3e}")
