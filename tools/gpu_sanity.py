"""Quick device sanity check: fast (tcgen05) vs fp64 operator on small shapes, with timing."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2503_02259_b200 as kgp

rng = np.random.default_rng(0)
for (n, d, k, kt) in [(256, 8, 32, "gaussian"), (1000, 3, 17, "matern32"), (777, 2, 1, "matern52"), (4096, 8, 32, "gaussian")]:
    x = rng.standard_normal((n, d)); b = rng.standard_normal((n, k))
    hp = kgp.Hyperparams(1.0, 1.0, 1e-2)
    ref = kgp.KernelEngine(kgp.KernelType(kt), x, hp, precision="fp64").matmul_with_grads(b)
    for prec in ("fast", "tf32"):
        t0 = time.time()
        got = kgp.KernelEngine(kgp.KernelType(kt), x, hp, precision=prec).matmul_with_grads(b)
        torch.cuda.synchronize()
        errs = [float(np.abs(g - r).max() / np.abs(r).max()) for g, r in zip(got, ref)]
        print(n, d, k, kt, prec, "rel errs", ["%.2e" % e for e in errs], "%.3fs" % (time.time() - t0), flush=True)
