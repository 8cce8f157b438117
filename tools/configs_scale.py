"""One fused operator application (K̂·B, the PCG unit) at each BASELINE config's full size on one
GPU, vs the survey's CPU numbers for the reference (extrapolated there)."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2503_02259_b200 as kgp
from paper_2503_02259_b200 import _lib, workloads

CPU = {"cfg3": 1.13e10, "cfg4": 4.50e9, "cfg5": 1.94e10}
cases = [("cfg3", workloads.cfg3, 33, "fast"), ("cfg3", workloads.cfg3, 33, "fp64"),
         ("cfg4", workloads.cfg4, 51, "fast"), ("cfg5", workloads.cfg5, 64, "fast")]
only = sys.argv[1:] or None
for name, fn, k, prec in cases:
    if only and name not in only:
        continue
    w = fn()
    e = kgp.KernelEngine(kgp.KernelType(w.kernel), w.x, kgp.Hyperparams(w.l, w.f, w.s), precision=prec)
    b = torch.randn(w.n, k, dtype=torch.float64, device="cuda")
    out = torch.empty_like(b)
    def run():
        _lib.call("kgp_engine_matmul", e.handle, k, b.data_ptr(), b.stride(0), b.stride(1), out.data_ptr(), None,
                  None, out.stride(0), out.stride(1), torch.cuda.current_stream().cuda_stream)
    run(); torch.cuda.synchronize()
    reps = 3 if w.n * w.n * k < 1e13 else 1
    s, t = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): run()
    t.record(); t.synchronize()
    ms = s.elapsed_time(t) / reps
    rate = w.n * w.n * k / (ms / 1e3)
    print(f"{name} {w.kernel} n={w.n} d={w.d} k={k} {prec}: {ms:9.2f} ms  {rate:.3e} entries*RHS/s  "
          f"({rate / CPU[name]:.0f}x the survey's 8-core reference number)", flush=True)
    e.close()
    del b, out
    torch.cuda.empty_cache()
