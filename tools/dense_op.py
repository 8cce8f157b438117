"""cfg1 DENSE-mode product and eval timing (run once per env variant):
python tools/dense_op.py   (env KGP_DENSE_SYMM=0|1 selects DGEMM / DSYMM)"""
import os
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_2503_02259_b200 as kgp
from paper_2503_02259_b200 import _lib, gp, precond, workloads

w = workloads.cfg1()
probes = gp.ProbeSet.generate(w.n, w.k_z, w.probe_seed)
e = kgp.KernelEngine(kgp.KernelType.GAUSSIAN, w.x, kgp.Hyperparams(w.l, w.f, w.s), precision="fp64")
st = torch.cuda.current_stream()
for k in (1, 17):
    b = torch.randn((k, w.n), dtype=torch.float64, device="cuda")  # column-major n x k
    o = torch.empty_like(b)

    def step():
        _lib.call("kgp_engine_matmul", e.handle, k, b.data_ptr(), 1, w.n, o.data_ptr(), None, None, 1, w.n,
                  st.cuda_stream)

    for _ in range(5):
        step()
    a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(50):
        step()
    z.record(st)
    torch.cuda.synchronize()
    print(f"symm={os.environ.get('KGP_DENSE_SYMM', '0')} k={k}: {a.elapsed_time(z) / 50 * 1e3:.1f} us/product")
pre = precond.build(e, w.rank)
for _ in range(3):
    lg = gp.nlml_grad_iterative(e, w.y, pre, probes, tol=0.0, max_iter=50, probe_tol=0.0, probe_max_iter=20)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20):
    lg = gp.nlml_grad_iterative(e, w.y, pre, probes, tol=0.0, max_iter=50, probe_tol=0.0, probe_max_iter=20)
torch.cuda.synchronize()
print(f"eval {(time.perf_counter() - t0) / 20 * 1e3:.2f} ms  loss {lg.loss!r}")
