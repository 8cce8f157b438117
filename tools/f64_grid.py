"""Time the fp64 fused operator over a grid of shapes in one process: f64_grid.py n kernel d nout k1,k2,..."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2503_02259_b200 as kgp
from paper_2503_02259_b200 import _lib

n, kt, d, nout = int(sys.argv[1]), sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
ks = [int(v) for v in sys.argv[5].split(",")]
x = np.random.default_rng(0).uniform(0, 1, (n, d))
e = kgp.KernelEngine(kgp.KernelType(kt), x, kgp.Hyperparams(0.2, 1.5, 1e-3), precision="fp64",
                     mode=kgp.EngineMode.ON_THE_FLY)
st = torch.cuda.current_stream()
out = []
for k in ks:
    z = torch.randn(n, k, dtype=torch.float64, device="cuda")
    ok = torch.empty_like(z)
    ol = torch.empty_like(z) if nout == 2 else None

    def run():
        _lib.call("kgp_engine_matmul", e.handle, k, z.data_ptr(), z.stride(0), z.stride(1), ok.data_ptr(),
                  None if ol is None else ol.data_ptr(), None, ok.stride(0), ok.stride(1), st.cuda_stream)

    run()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(3):
        run()
    b.record(st)
    torch.cuda.synchronize()
    out.append(f"k={k}: {a.elapsed_time(b) / 3:.3f}")
print(f"{kt} d={d} n={n} nout={nout} ms: " + "  ".join(out))
