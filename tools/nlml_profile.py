"""Break down one configs[0] NLML+gradient evaluation (fixed recipe) on the device."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2503_02259_b200 as kgp
from paper_2503_02259_b200 import _lib, gp, precond, workloads

w = workloads.cfg1()
probes = gp.ProbeSet.generate(w.n, w.k_z, w.probe_seed)
torch.linalg.cholesky(torch.eye(4, dtype=torch.float64, device="cuda"))  # library init
for prec in ("fp64", "fast"):
    e = kgp.KernelEngine(kgp.KernelType.GAUSSIAN, w.x, kgp.Hyperparams(w.l, w.f, w.s), precision=prec)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    pre = precond.build(e, w.rank)
    torch.cuda.synchronize(); tb = time.perf_counter() - t0
    for k in (1, 16, 17):
        b = torch.randn(w.n, k, dtype=torch.float64, device="cuda")
        out = torch.empty_like(b)
        def run():
            _lib.call("kgp_engine_matmul", e.handle, k, b.data_ptr(), b.stride(0), b.stride(1), out.data_ptr(),
                      None, None, out.stride(0), out.stride(1), torch.cuda.current_stream().cuda_stream)
        for _ in range(3): run()
        torch.cuda.synchronize(); t0 = time.perf_counter()
        for _ in range(20): run()
        torch.cuda.synchronize(); print(prec, "matmul k=%d: %.1f us" % (k, (time.perf_counter() - t0) / 20 * 1e6))
    for _ in range(2):
        gp.nlml_grad_iterative(e, w.y, pre, probes, tol=0.0, max_iter=50, probe_tol=0.0, probe_max_iter=20)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(5):
        lg = gp.nlml_grad_iterative(e, w.y, pre, probes, tol=0.0, max_iter=50, probe_tol=0.0, probe_max_iter=20)
    torch.cuda.synchronize()
    print(prec, "build %.1f ms, eval %.2f ms, loss %.8f" % (tb * 1e3, (time.perf_counter() - t0) / 5 * 1e3, lg.loss))
