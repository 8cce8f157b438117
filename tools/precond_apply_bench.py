"""Time Nystrom / AFN applications (k RHS) with CUDA events: precond_apply_bench.py n m k"""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2503_02259_b200 as kgp
from paper_2503_02259_b200 import _lib, precond

n, m, k = (int(v) for v in sys.argv[1:4])
x = np.random.default_rng(0).uniform(0, 1, (n, 4))
e = kgp.KernelEngine(kgp.KernelType.MATERN32, x, kgp.Hyperparams(0.2, 1.0, 1e-3), precision="fast")
b = torch.randn(k, n, dtype=torch.float64, device="cuda")
out = torch.empty_like(b)
for name, pre in (("nystrom", precond.build(e, m)), ("afn", precond.build_afn(e, m, 32))):
    def run():
        _lib.call("kgp_precond_apply_inverse", pre.handle, k, b.data_ptr(), 1, n, out.data_ptr(), 1, n,
                  torch.cuda.current_stream().cuda_stream)
    for _ in range(3): run()
    torch.cuda.synchronize()
    s, t = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20): run()
    t.record(); t.synchronize()
    ms = s.elapsed_time(t) / 20
    wbytes = 2 * n * m * 8
    print(f"{name} n={n} m={m} k={k}: {ms * 1e3:.1f} us  (W streamed twice: {wbytes / ms / 1e6:.0f} GB/s)", flush=True)
