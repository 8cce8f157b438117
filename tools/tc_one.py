"""Run one fused-operator config repeatedly (for ncu): tc_one.py n k nout precision [kernel] [d]"""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2503_02259_b200 as kgp
from paper_2503_02259_b200 import _lib, workloads

n, k, nout, prec = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
kt = sys.argv[5] if len(sys.argv) > 5 else "gaussian"
d = int(sys.argv[6]) if len(sys.argv) > 6 else 8
w = workloads.cfg2(n=n, k=max(k, 1))
e = kgp.KernelEngine(kgp.KernelType(kt), w.x[:, :d], kgp.Hyperparams(1.0, 1.0, 1e-2), precision=prec)
z = torch.from_numpy(np.ascontiguousarray(w.z[:, :k])).cuda()
ok = torch.empty((n, k), dtype=torch.float64, device="cuda")
ol = torch.empty_like(ok)
for _ in range(4):
    _lib.call("kgp_engine_matmul", e.handle, k, z.data_ptr(), z.stride(0), z.stride(1), ok.data_ptr(),
              ol.data_ptr() if nout == 2 else None, None, ok.stride(0), ok.stride(1),
              torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
print("done")
