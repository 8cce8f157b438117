"""Fused-operator time across kernels / dimensions / RHS widths at one n (diagnostic).
Usage: python tools/op_matrix.py [n] [precision]"""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2503_02259_b200 as kgp
from paper_2503_02259_b200 import _lib

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
prec = sys.argv[2] if len(sys.argv) > 2 else "fast"
rng = np.random.default_rng(0)
KD = [tuple(x.split(":")) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [("gaussian", "8"), ("matern32", "4"), ("matern52", "2"), ("gaussian", "3")]
for kt, d in ((a, int(b)) for a, b in KD):
    x = rng.uniform(0, 1, (n, d))
    e = kgp.KernelEngine(kgp.KernelType(kt), x, kgp.Hyperparams(0.2, 1.0, 1e-3), precision=prec)
    for k in (1, 16, 33, 64):
        z = torch.randn(n, k, dtype=torch.float64, device="cuda")
        ok = torch.empty_like(z)
        for nout in (1, 2):
            ol = torch.empty_like(z) if nout == 2 else None
            def run():
                _lib.call("kgp_engine_matmul", e.handle, k, z.data_ptr(), z.stride(0), z.stride(1), ok.data_ptr(),
                          None if ol is None else ol.data_ptr(), None, ok.stride(0), ok.stride(1),
                          torch.cuda.current_stream().cuda_stream)
            try:
                for _ in range(3): run()
                torch.cuda.synchronize()
            except Exception as exc:
                print(f"{kt:8s} d={d:2d} k={k:3d} nout={nout} failed: {exc}", flush=True)
                continue
            s, t = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(5): run()
            t.record(); t.synchronize()
            ms = s.elapsed_time(t) / 5
            print(f"{kt:8s} d={d:2d} k={k:3d} nout={nout} {ms:8.3f} ms  {n * n * k * nout / ms / 1e9:10.1f} G entries*RHS/s  "
                  f"{n * n / ms / 1e9:8.1f} G entries/s", flush=True)
