"""Max-relative error of the fast operator (both outputs) against the fp64 operator at one
cfg2-generator size (diagnostic for kernel variants: KGP_LIB=... python tools/variant_err.py [n] [k])."""
import sys
sys.path.insert(0, ".")
import numpy as np
import paper_2503_02259_b200 as kgp
from paper_2503_02259_b200 import workloads

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
k = int(sys.argv[2]) if len(sys.argv) > 2 else 32
w = workloads.cfg2(n=n, k=k)
hp = kgp.Hyperparams(1.0, 1.0, 1e-2)
ef = kgp.KernelEngine(kgp.KernelType.GAUSSIAN, w.x, hp, precision="fast")
ed = kgp.KernelEngine(kgp.KernelType.GAUSSIAN, w.x, hp, precision="fp64")
fk, fl, _ = ef.matmul_with_grads(w.z)
dk, dl, _ = ed.matmul_with_grads(w.z)
print(f"err n={n} k={k}: K {np.abs(fk - dk).max() / np.abs(dk).max():.2e}  dL {np.abs(fl - dl).max() / np.abs(dl).max():.2e}")
