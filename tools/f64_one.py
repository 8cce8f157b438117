"""Run the fp64 fused operator repeatedly (for timing / ncu): f64_one.py n k nout kernel d"""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2503_02259_b200 as kgp
from paper_2503_02259_b200 import _lib

n, k, nout, kt, d = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], int(sys.argv[5])
x = np.random.default_rng(0).uniform(0, 1, (n, d))
e = kgp.KernelEngine(kgp.KernelType(kt), x, kgp.Hyperparams(0.2, 1.5, 1e-3), precision="fp64",
                     mode=kgp.EngineMode.ON_THE_FLY)
z = torch.randn(n, k, dtype=torch.float64, device="cuda")
ok = torch.empty_like(z)
ol = torch.empty_like(z) if nout == 2 else None
st = torch.cuda.current_stream()


def run():
    _lib.call("kgp_engine_matmul", e.handle, k, z.data_ptr(), z.stride(0), z.stride(1), ok.data_ptr(),
              None if ol is None else ol.data_ptr(), None, ok.stride(0), ok.stride(1), st.cuda_stream)


for _ in range(2):
    run()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(st)
for _ in range(3):
    run()
b.record(st)
torch.cuda.synchronize()
ms = a.elapsed_time(b) / 3
print(f"{kt} d={d} n={n} k={k} nout={nout}: {ms:.2f} ms  {n * n * k * nout / ms / 1e9:.3e} entries*RHS/s")
