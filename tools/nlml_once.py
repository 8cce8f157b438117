"""One warm cfg1 fixed-recipe NLML eval for ncu launch lists: python tools/nlml_once.py [precision] [otf|dense]"""
import sys
sys.path.insert(0, ".")
import torch
import paper_2503_02259_b200 as kgp
from paper_2503_02259_b200 import gp, precond, workloads

prec = sys.argv[1] if len(sys.argv) > 1 else "fp64"
mode = kgp.EngineMode.DENSE if (len(sys.argv) > 2 and sys.argv[2] == "dense") else kgp.EngineMode.ON_THE_FLY
w = workloads.cfg1()
probes = gp.ProbeSet.generate(w.n, w.k_z, w.probe_seed)
e = kgp.KernelEngine(kgp.KernelType.GAUSSIAN, w.x, kgp.Hyperparams(w.l, w.f, w.s), mode=mode, precision=prec)
pre = precond.build(e, w.rank)
for _ in range(2):
    lg = gp.nlml_grad_iterative(e, w.y, pre, probes, tol=0.0, max_iter=50, probe_tol=0.0, probe_max_iter=20)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("eval")
lg = gp.nlml_grad_iterative(e, w.y, pre, probes, tol=0.0, max_iter=50, probe_tol=0.0, probe_max_iter=20)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print(lg)
