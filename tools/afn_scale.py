"""cfg3-scale preconditioner comparison (BASELINE configs[2]): build time, apply time and
PCG iterations/time for Nystrom vs AFN at the same rank. Usage: python tools/afn_scale.py [n]"""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2503_02259_b200 as kgp
from paper_2503_02259_b200 import precond, solver, workloads

n = int(sys.argv[1]) if len(sys.argv) > 1 else 262144
prec = sys.argv[2] if len(sys.argv) > 2 else "fast"
w = workloads.cfg3(n=n)
e = kgp.KernelEngine(kgp.KernelType.MATERN32, w.x, kgp.Hyperparams(w.l, w.f, w.s), precision=prec)
yd = torch.from_numpy(w.y).cuda()
torch.linalg.cholesky(torch.eye(8, dtype=torch.float64, device="cuda"))
rank = w.rank
def timed(fn, reps=1):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): r = fn()
    torch.cuda.synchronize(); return r, (time.perf_counter() - t0) / reps
for name, bld in (("nystrom", lambda: precond.build(e, rank)), ("afn", lambda: precond.build_afn(e, rank, 32))):
    pre, t_first = timed(bld)
    del pre; torch.cuda.empty_cache()
    pre, t_b = timed(bld)
    b = torch.randn(n, 1, dtype=torch.float64, device="cuda")
    _, t_a = timed(lambda: pre.apply_inverse(b), 10)
    rep, t_s = timed(lambda: solver.pcg_solve(e.matmul, pre.apply_inverse, yd, tol=1e-6, max_iter=2000))
    print(f"{name}: build {t_b*1e3:.1f} ms (first {t_first*1e3:.1f}), apply {t_a*1e3:.3f} ms, "
          f"pcg iters {rep.iteration_counts()[0]} conv {rep.converged[0]} in {t_s*1e3:.1f} ms", flush=True)
    del pre; torch.cuda.empty_cache()

# NLML+gradient eval at this size (tolerance mode, tol 1e-6, reference default probe_tol), AFN w-solve
from paper_2503_02259_b200 import gp
probes = gp.ProbeSet.generate(n, w.k_z, 0)
pre = precond.build_afn(e, rank, 32)
lg, t1 = timed(lambda: gp.nlml_grad_iterative(e, w.y, pre, probes, tol=1e-6, max_iter=2000))
lg, t2 = timed(lambda: gp.nlml_grad_iterative(e, w.y, pre, probes, tol=1e-6, max_iter=2000))
print(f"nlml (afn, k_z={w.k_z}): {t2*1e3:.1f} ms (first {t1*1e3:.1f}), loss {lg.loss:.8f} grad "
      f"({lg.grad_l:.6g}, {lg.grad_f:.6g}, {lg.grad_s:.6g}) converged {lg.converged}", flush=True)
