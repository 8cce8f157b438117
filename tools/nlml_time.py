"""Time the cfg1 fixed-recipe NLML+gradient eval (diagnostic): python tools/nlml_time.py [precision] [otf|dense] [reps]"""
import sys
import time
sys.path.insert(0, ".")
import torch
import paper_2503_02259_b200 as kgp
from paper_2503_02259_b200 import gp, precond, workloads

prec = sys.argv[1] if len(sys.argv) > 1 else "fp64"
mode = kgp.EngineMode.DENSE if (len(sys.argv) > 2 and sys.argv[2] == "dense") else kgp.EngineMode.ON_THE_FLY
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
w = workloads.cfg1()
probes = gp.ProbeSet.generate(w.n, w.k_z, w.probe_seed)
e = kgp.KernelEngine(kgp.KernelType.GAUSSIAN, w.x, kgp.Hyperparams(w.l, w.f, w.s), mode=mode, precision=prec)
pre = precond.build(e, w.rank)


def ev():
    return gp.nlml_grad_iterative(e, w.y, pre, probes, tol=0.0, max_iter=50, probe_tol=0.0, probe_max_iter=20)


for _ in range(3):
    ev()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(reps):
    lg = ev()
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / reps
print(f"cfg1 fixed recipe {prec} {mode.name}: {dt * 1e3:.3f} ms/eval ({1 / dt:.1f} evals/s) loss {lg.loss:.10f}")
