"""Time one cfg4 GPC training step's parts: AFN builds (3 classes) and the grouped NLML solve."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2503_02259_b200 as kgp
from paper_2503_02259_b200 import gpc, workloads, solver

n = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
w = workloads.cfg4(n=n)
prob = gpc.setup(w.x, w.extra["labels"], 3)
e = kgp.KernelEngine(kgp.KernelType.GAUSSIAN, w.x, kgp.Hyperparams(1.0, 1.0, 0.1), precision="fast")
torch.linalg.cholesky(torch.eye(8, dtype=torch.float64, device="cuda"))
for rep in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    pcs = gpc.build_preconditioners(e, prob, w.rank, "afn")
    torch.cuda.synchronize(); t1 = time.perf_counter()
    probes = gpc.generate_probes(n, 3, w.k_z, (0, rep))
    lg = gpc.nlml_grad_iterative(e, prob, pcs, probes, tol=1e-6, max_iter=1000, probe_tol=1e-2)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    lp = gpc.nlml_grad_iterative(e, prob, pcs, probes, tol=1e-6, max_iter=1000, probe_tol=1e-2,
                                 preconditioned_probes=True)
    torch.cuda.synchronize(); t3 = time.perf_counter()
    print(f"build {1e3 * (t1 - t0):.1f} ms, nlml {1e3 * (t2 - t1):.1f} ms (loss {lg.loss:.6g}, conv {lg.converged}); "
          f"preconditioned probes {1e3 * (t3 - t2):.1f} ms (loss {lp.loss:.6g}, conv {lp.converged})", flush=True)
    for p in pcs:
        p.close()
