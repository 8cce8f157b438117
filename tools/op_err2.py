"""Max-relative error of the tensor-core precisions (both outputs) against the fp64 operator
on a row block (diagnostic): python tools/op_err2.py [n] [k] [precisions...]"""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2503_02259_b200 as kgp
from paper_2503_02259_b200 import _lib, workloads

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
k = int(sys.argv[2]) if len(sys.argv) > 2 else 32
precs = sys.argv[3:] or ["fast", "bf16x3", "tf32"]
w = workloads.cfg2(n=n, k=k)
hp = kgp.Hyperparams(1.0, 1.0, 1e-2)
ed = kgp.KernelEngine(kgp.KernelType.GAUSSIAN, w.x, hp, precision="fp64")
rows = 1024
_lib.call("kgp_engine_set_rows", ed.handle, n - rows, rows)
zd = torch.from_numpy(w.z).cuda()
dk, dl, _ = ed.apply(zd, True, True, False)
dk, dl = dk.cpu().numpy()[:rows], dl.cpu().numpy()[:rows]  # the engine's rows [n - rows, n)
for prec in precs:
    ef = kgp.KernelEngine(kgp.KernelType.GAUSSIAN, w.x, hp, precision=prec)
    fk, fl, _ = ef.apply(zd, True, True, False)
    fk, fl = fk.cpu().numpy()[n - rows:], fl.cpu().numpy()[n - rows:]
    ek = np.abs(fk - dk).max() / np.abs(dk).max()
    el = np.abs(fl - dl).max() / np.abs(dl).max()
    print(f"{prec:7s} n={n:6d} k={k:3d}  Khat.Z err {ek:.2e}  dKhat/dl.Z err {el:.2e}", flush=True)
    ef.close()
