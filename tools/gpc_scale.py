"""BASELINE configs[3] (GPC, 3 classes, n=131072, d=8, 16 probes, AFN rank 512, 10 training
steps) on the device: per-step time of the Dirichlet-GPC training loop.
Usage: python tools/gpc_scale.py [n] [precision] [steps]"""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2503_02259_b200 as kgp
from paper_2503_02259_b200 import gpc, workloads

n = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
prec = sys.argv[2] if len(sys.argv) > 2 else "fast"
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
w = workloads.cfg4(n=n)
prob = gpc.setup(w.x, w.extra["labels"], 3)
print("class counts", np.bincount(prob.labels, minlength=3).tolist(), flush=True)
torch.linalg.cholesky(torch.eye(8, dtype=torch.float64, device="cuda"))
torch.cuda.synchronize(); t0 = time.perf_counter()
res = gpc.fit(kgp.KernelType.GAUSSIAN, prob, kgp.Hyperparams(w.l, w.f, 0.1), steps=steps, k_z=w.k_z, rank=w.rank,
              tol=1e-6, max_iter=1000, probe_tol=1e-2, precision=prec)
torch.cuda.synchronize(); t = time.perf_counter() - t0
print(f"gpc fit n={n} {prec}: {steps} steps in {t:.2f} s ({t / steps * 1e3:.1f} ms/step), "
      f"loss {res.loss_history[0]:.6g} -> {res.loss_history[-1]:.6g}, params {res.params}, "
      f"converged {res.converged}", flush=True)
