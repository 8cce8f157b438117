"""BASELINE configs[4] pipeline on ONE B200 (the config targets 8): Matern-5/2, n=1048576, d=2,
64 RHS (y + 63 probes), rank 2048: AFN build, one NLML+gradient evaluation with AFN-preconditioned
probes, and the Hutchinson prediction at m_test=262144. Usage: python tools/cfg5_run.py [n] [m_test]"""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2503_02259_b200 as kgp
from paper_2503_02259_b200 import gp, precond, workloads

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1048576
mt = int(sys.argv[2]) if len(sys.argv) > 2 else 262144
w = workloads.cfg5(n=n, m_test=mt)
hp = kgp.Hyperparams(w.l, w.f, w.s)
def timed(fn):
    torch.cuda.synchronize(); t0 = time.perf_counter(); r = fn(); torch.cuda.synchronize()
    return r, time.perf_counter() - t0
e = kgp.KernelEngine(kgp.KernelType.MATERN52, w.x, hp, precision="fast")
torch.linalg.cholesky(torch.eye(8, dtype=torch.float64, device="cuda"))
pre, tb = timed(lambda: precond.build_afn(e, w.rank, 32))
print(f"n={n}: AFN build (m={w.rank}, npt=32) {tb:.2f} s, log|M| {pre.logdet:.6g}", flush=True)
probes = gp.ProbeSet.generate(n, w.k_z, 0)
lg, t = timed(lambda: gp.nlml_grad_iterative(e, w.y, pre, probes, tol=1e-6, max_iter=500,
                                             preconditioned_probes=True))
print(f"NLML+grad (AFN-preconditioned probes, k_z={w.k_z}): {t:.2f} s, loss {lg.loss:.8g}, "
      f"grad ({lg.grad_l:.6g}, {lg.grad_f:.6g}, {lg.grad_s:.6g}), converged {lg.converged}", flush=True)
del pre
torch.cuda.empty_cache()
pr, t = timed(lambda: gp.predict_hutchinson(kgp.KernelType.MATERN52, w.x, w.y, w.extra["xstar"], hp, tol=1e-6,
                                            max_iter=500, precond_rank=w.rank, num_probes=64, precision="fast",
                                            preconditioner="afn"))
truth = np.sin(4 * np.pi * w.extra["xstar"][:, 0]) + np.cos(4 * np.pi * w.extra["xstar"][:, 1])
print(f"predict (Hutchinson, m={mt}, 64 probes): {t:.2f} s, rmse vs noise-free truth "
      f"{np.sqrt(np.mean((pr.mean - truth) ** 2)):.4f}, mean stddev {pr.stddev.mean():.4f}", flush=True)

pl, t = timed(lambda: gp.predict_local(kgp.KernelType.MATERN52, w.x, w.y, w.extra["xstar"], hp, tol=1e-6,
                                       max_iter=500, precond_rank=w.rank, k_nn=64, precision="fast"))
print(f"predict (local variance, 64 neighbours, m={mt}): {t:.2f} s, rmse {np.sqrt(np.mean((pl.mean - truth) ** 2)):.4f}, "
      f"mean stddev {pl.stddev.mean():.4f} (min {pl.stddev.min():.4f}, max {pl.stddev.max():.4f})", flush=True)
# accuracy of the local variance against the exact one on a subsample of the problem
ns, ms = 8192, 512
pe = gp.predict(kgp.KernelType.MATERN52, w.x[:ns], w.y[:ns], w.extra["xstar"][:ms], hp, mode="exact")
pq = gp.predict_local(kgp.KernelType.MATERN52, w.x[:ns], w.y[:ns], w.extra["xstar"][:ms], hp, tol=1e-10, k_nn=64)
print(f"local vs exact variance (n={ns}, m={ms}): max rel err of stddev "
      f"{np.max(np.abs(pq.stddev - pe.stddev) / pe.stddev):.3e}", flush=True)
