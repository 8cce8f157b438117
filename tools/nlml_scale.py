"""NLML+gradient at the cfg3 generator (Matern-3/2, d=4, l=0.2, s=1e-3, 32 probes, tol 1e-6,
reference default probe_tol): the reference estimator (unpreconditioned probes) vs the
preconditioned-probe extension. Usage: python tools/nlml_scale.py [n] [rank] [max_iter]"""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2503_02259_b200 as kgp
from paper_2503_02259_b200 import gp, precond, solver, workloads

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
rank = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
max_iter = int(sys.argv[3]) if len(sys.argv) > 3 else 2000
w = workloads.cfg3(n=n)
e = kgp.KernelEngine(kgp.KernelType.MATERN32, w.x, kgp.Hyperparams(w.l, w.f, w.s), precision="fast")
probes = gp.ProbeSet.generate(n, w.k_z, 0)
torch.linalg.cholesky(torch.eye(8, dtype=torch.float64, device="cuda"))
def timed(fn):
    torch.cuda.synchronize(); t0 = time.perf_counter(); r = fn(); torch.cuda.synchronize()
    return r, time.perf_counter() - t0
print(f"n={n} rank={rank} tol=1e-6 probe_tol={solver.DEFAULT_PROBE_TOL} max_iter={max_iter}", flush=True)
afn, tb = timed(lambda: precond.build_afn(e, rank, 32))
lg, t = timed(lambda: gp.nlml_grad_iterative(e, w.y, afn, probes, tol=1e-6, max_iter=max_iter))
print(f"reference estimator, AFN w-solve: {t:.2f} s (+{tb:.2f} s build) loss {lg.loss:.6f} "
      f"grad ({lg.grad_l:.5g}, {lg.grad_f:.5g}, {lg.grad_s:.5g}) converged {lg.converged}", flush=True)
lg, t = timed(lambda: gp.nlml_grad_iterative(e, w.y, afn, probes, tol=1e-6, max_iter=max_iter,
                                             preconditioned_probes=True))
print(f"preconditioned probes (AFN draws, AFN everywhere): {t:.2f} s loss {lg.loss:.6f} "
      f"grad ({lg.grad_l:.5g}, {lg.grad_f:.5g}, {lg.grad_s:.5g}) converged {lg.converged}", flush=True)
ny, tb = timed(lambda: precond.build(e, rank))
lg, t = timed(lambda: gp.nlml_grad_iterative(e, w.y, afn, probes, tol=1e-6, max_iter=max_iter,
                                             preconditioned_probes=ny))
print(f"preconditioned probes (Nystrom probes, AFN w-solve): {t:.2f} s (+{tb:.2f} s build) loss {lg.loss:.6f} "
      f"grad ({lg.grad_l:.5g}, {lg.grad_f:.5g}, {lg.grad_s:.5g}) converged {lg.converged}", flush=True)
del afn
lg, t = timed(lambda: gp.nlml_grad_iterative(e, w.y, ny, probes, tol=1e-6, max_iter=max_iter,
                                             preconditioned_probes=True))
print(f"preconditioned probes (Nystrom): {t:.2f} s (+{tb:.2f} s build) loss {lg.loss:.6f} "
      f"grad ({lg.grad_l:.5g}, {lg.grad_f:.5g}, {lg.grad_s:.5g}) converged {lg.converged}", flush=True)
