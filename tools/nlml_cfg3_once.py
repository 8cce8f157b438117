"""One warm configs[2]-generator NLML eval (AFN + preconditioned probes, fast operator) inside an
NVTX range `eval`, for ncu launch lists: python tools/nlml_cfg3_once.py [n]"""
import sys, time
sys.path.insert(0, ".")
import torch
import paper_2503_02259_b200 as kgp
from paper_2503_02259_b200 import gp, precond, workloads

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
w = workloads.cfg3(n=n)
e = kgp.KernelEngine(kgp.KernelType.MATERN32, w.x, kgp.Hyperparams(w.l, w.f, w.s), precision="fast")
probes = gp.ProbeSet.generate(n, w.k_z, 0)
pre = precond.build_afn(e, w.rank, 32)


def ev():
    return gp.nlml_grad_iterative(e, w.y, pre, probes, tol=1e-6, max_iter=2000, preconditioned_probes=True)


ev()
torch.cuda.synchronize()
t0 = time.perf_counter()
torch.cuda.nvtx.range_push("eval")
lg = ev()
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("eval %.1f ms" % ((time.perf_counter() - t0) * 1e3), lg)
