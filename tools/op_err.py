"""Max-relative error of the fast operator (both outputs) against the fp64 operator (diagnostic)."""
import sys
sys.path.insert(0, ".")
import numpy as np
import paper_2503_02259_b200 as kgp
from paper_2503_02259_b200 import workloads

for n in (4096, 16384, 65536):
    for k in (16, 32, 48):
        w = workloads.cfg2(n=n, k=k)
        hp = kgp.Hyperparams(1.0, 1.0, 1e-2)
        ef = kgp.KernelEngine(kgp.KernelType.GAUSSIAN, w.x, hp, precision="fast")
        ed = kgp.KernelEngine(kgp.KernelType.GAUSSIAN, w.x, hp, precision="fp64")
        fk, fl, _ = ef.matmul_with_grads(w.z)
        dk, dl, _ = ed.matmul_with_grads(w.z)
        ek = np.abs(fk - dk).max() / np.abs(dk).max()
        el = np.abs(fl - dl).max() / np.abs(dl).max()
        print(f"n={n:6d} k={k:3d}  K err {ek:.2e}  dL err {el:.2e}", flush=True)
        ef.close(); ed.close()
