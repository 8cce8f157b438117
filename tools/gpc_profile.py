"""Time one cfg4 GPC training step's parts: AFN builds (3 classes) and the grouped NLML solve."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2503_02259_b200 as kgp
from paper_2503_02259_b200 import gpc, workloads, solver

n = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
w = workloads.cfg4(n=n)
prob = gpc.setup(w.x, w.extra["labels"], 3)
e = kgp.KernelEngine(kgp.KernelType.GAUSSIAN, w.x, kgp.Hyperparams(1.0, 1.0, 0.1), precision="fast")
torch.linalg.cholesky(torch.eye(8, dtype=torch.float64, device="cuda"))
kinds = sys.argv[2:] or ["afn"]
for rep, kind in enumerate(kinds):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    pcs = gpc.build_preconditioners(e, prob, w.rank, kind)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    probes = gpc.generate_probes(n, 3, w.k_z, (0, rep))
    lg = gpc.nlml_grad_iterative(e, prob, pcs, probes, tol=1e-6, max_iter=1000, probe_tol=1e-2)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    lp = gpc.nlml_grad_iterative(e, prob, pcs, probes, tol=1e-6, max_iter=1000, probe_tol=1e-2,
                                 preconditioned_probes=True)
    torch.cuda.synchronize(); t3 = time.perf_counter()
    print(f"[{kind}] build {1e3 * (t1 - t0):.1f} ms, nlml {1e3 * (t2 - t1):.1f} ms (loss {lg.loss:.6g}, conv {lg.converged}); "
          f"preconditioned probes {1e3 * (t3 - t2):.1f} ms (loss {lp.loss:.6g}, conv {lp.converged})", flush=True)
    for p in pcs:
        p.close()

# w-solve iteration counts per preconditioner kind (the grouped NLML runs max over columns)
import ctypes
from paper_2503_02259_b200 import _device, _lib
dn = torch.from_numpy(np.ascontiguousarray(prob.noise)).cuda()
yt = torch.from_numpy(np.ascontiguousarray(prob.targets)).cuda()
for kind in ("none", "nystrom", "afn"):
    pcs = gpc.build_preconditioners(e, prob, w.rank, kind)
    arr = (ctypes.c_void_p * max(1, len(pcs)))(*[p.handle for p in pcs]) if pcs else None
    x = torch.empty((3, n), dtype=torch.float64, device="cuda")
    al = torch.empty((3, 2000), dtype=torch.float64, device="cuda"); be = torch.empty_like(al)
    it = torch.empty(3, dtype=torch.int32, device="cuda"); rel = torch.empty(3, dtype=torch.float64, device="cuda")
    cv = torch.empty(3, dtype=torch.int32, device="cuda")
    _lib.call("kgp_engine_set_diag", e.handle, 3, dn.data_ptr(), 3, (ctypes.c_int32 * 3)(0, 1, 2), None)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    _lib.call("kgp_pcg_grouped", e.handle, arr, len(pcs), 3, 3, yt.data_ptr(), 1e-6, 2000, 1e-6, 2000, x.data_ptr(),
              al.data_ptr(), be.data_ptr(), it.data_ptr(), rel.data_ptr(), cv.data_ptr(), None)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    _lib.call("kgp_engine_set_diag", e.handle, 0, None, 0, None, None)
    print(f"w-solve [{kind}]: iterations {it.tolist()} in {1e3 * (t1 - t0):.1f} ms", flush=True)
    for p in pcs:
        p.close()
