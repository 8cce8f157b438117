"""Max-relative error of the fast operator (both outputs) against the fp64 operator (diagnostic for
kernel variants): KGP_LIB=... python tools/variant_err.py [n] [k] [kernel] [d]
(Gaussian d=8: the cfg2 generator; other kernels: X ~ U[0,1]^d with l = 0.2, s = 1e-3)."""
import sys
sys.path.insert(0, ".")
import numpy as np
import paper_2503_02259_b200 as kgp
from paper_2503_02259_b200 import workloads

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
k = int(sys.argv[2]) if len(sys.argv) > 2 else 32
kt = sys.argv[3] if len(sys.argv) > 3 else "gaussian"
d = int(sys.argv[4]) if len(sys.argv) > 4 else 8
if kt == "gaussian" and d == 8:
    w = workloads.cfg2(n=n, k=k)
    x, z, hp = w.x, w.z, kgp.Hyperparams(1.0, 1.0, 1e-2)
else:
    rng = np.random.default_rng(3)
    x, z, hp = rng.uniform(0, 1, (n, d)), rng.standard_normal((n, k)), kgp.Hyperparams(0.2, 1.5, 1e-3)
ef = kgp.KernelEngine(kgp.KernelType(kt), x, hp, precision="fast")
ed = kgp.KernelEngine(kgp.KernelType(kt), x, hp, precision="fp64")
fk, fl, _ = ef.matmul_with_grads(z)
dk, dl, _ = ed.matmul_with_grads(z)
print(f"err {kt} d={d} n={n} k={k}: K {np.abs(fk - dk).max() / np.abs(dk).max():.2e}  dL {np.abs(fl - dl).max() / np.abs(dl).max():.2e}")
