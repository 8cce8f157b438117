"""Timeline of the host-buffer product at cfg2 (diagnostic): KGP_HOST_TRACE=1 python tools/e2e_trace.py"""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2503_02259_b200 as kgp
from paper_2503_02259_b200 import _lib, workloads

w = workloads.cfg2()
e = kgp.KernelEngine(kgp.KernelType.GAUSSIAN, w.x, kgp.Hyperparams(1.0, 1.0, 1e-2), precision="fast")
zh = torch.from_numpy(w.z).pin_memory()
ok = torch.empty((w.n, w.z.shape[1]), dtype=torch.float64).pin_memory()
ol = torch.empty_like(ok).pin_memory()
st = torch.cuda.current_stream()
for _ in range(4):
    _lib.call("kgp_engine_matmul_host", e.handle, w.z.shape[1], zh.data_ptr(), ok.data_ptr(), ol.data_ptr(), None,
              st.cuda_stream)
