"""configs[0] tolerance-mode NLML+gradient in each operator precision vs the reference's
golden values (tests/golden/cfg1_full.npz): relative error per component."""
import sys
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import numpy as np
import paper_2503_02259_b200 as kgp
from paper_2503_02259_b200 import gp, precond, workloads
from conftest import golden

g = golden("cfg1_full.npz")
ref = g["iter_tight"][:4]
w = workloads.cfg1()
probes = gp.ProbeSet.generate(w.n, w.k_z, w.probe_seed)
for prec in (sys.argv[1:] or ["fp64", "fast", "tf32"]):
    e = kgp.KernelEngine(kgp.KernelType.GAUSSIAN, w.x, kgp.Hyperparams(w.l, w.f, w.s), precision=prec)
    try:
        lg = gp.nlml_grad_iterative(e, w.y, precond.build(e, w.rank), probes, tol=1e-10, max_iter=3000,
                                    probe_tol=1e-10)
        got = np.array([lg.loss, lg.grad_l, lg.grad_f, lg.grad_s])
        print(prec, "rel err (loss, l, f, s):", np.array2string(np.abs(got - ref) / np.abs(ref), precision=2),
              "converged", lg.converged, flush=True)
    except Exception as exc:
        print(prec, "failed:", exc, flush=True)
