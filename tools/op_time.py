"""Time one fused-operator product and its error vs the fp64 operator (diagnostic):
python tools/op_time.py kernel d k nout [n]"""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2503_02259_b200 as kgp
from paper_2503_02259_b200 import workloads

kt, d, k, nout = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
n = int(sys.argv[5]) if len(sys.argv) > 5 else 65536
w = workloads.cfg3(n=n) if d == 4 else workloads.cfg2(n=n)
x = w.x[:, :d]
hp = kgp.Hyperparams(0.2 if d <= 4 else 1.0, 1.5, 1e-3)
e = kgp.KernelEngine(kgp.KernelType(kt), x, hp, precision="fast")
z = torch.randn(n, k, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(0))
outs = (torch.empty_like(z), torch.empty_like(z) if nout == 2 else None, None)
for _ in range(3):
    e.apply(z, outs=outs)
torch.cuda.synchronize()
s, t = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10):
    e.apply(z, outs=outs)
t.record()
t.synchronize()
ms = s.elapsed_time(t) / 10
rows = np.arange(0, n, max(1, n // 512))
ref = kgp.KernelEngine(kgp.KernelType(kt), x, hp, precision="fp64")
sub = np.ascontiguousarray(z.cpu().numpy())
rk = ref.matmul_with_grads(sub)
gk = outs[0].cpu().numpy()
err = np.abs(gk[rows] - rk[0][rows]).max() / np.abs(rk[0][rows]).max()
msg = f"{kt} d={d} k={k} nout={nout} n={n}: {ms:.3f} ms, K err {err:.2e}"
if nout == 2:
    gl = outs[1].cpu().numpy()
    msg += f", dL err {np.abs(gl[rows] - rk[1][rows]).max() / np.abs(rk[1][rows]).max():.2e}"
print(msg, flush=True)
