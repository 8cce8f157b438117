"""Time the fused operator across precisions / output counts / RHS widths (diagnostic)."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2503_02259_b200 as kgp
from paper_2503_02259_b200 import _lib, workloads

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
w = workloads.cfg2(n=n)
for prec in ("fast", "tf32"):
    e = kgp.KernelEngine(kgp.KernelType.GAUSSIAN, w.x, kgp.Hyperparams(1.0, 1.0, 1e-2), precision=prec)
    for k in (16, 32, 64):
        z = torch.from_numpy(np.ascontiguousarray(w.z[:, :1].repeat(k, 1))).cuda() if k > 32 else torch.from_numpy(np.ascontiguousarray(w.z[:, :k])).cuda()
        ok = torch.empty((n, k), dtype=torch.float64, device="cuda"); ol = torch.empty_like(ok)
        for nout in (1, 2):
            def run():
                _lib.call("kgp_engine_matmul", e.handle, k, z.data_ptr(), z.stride(0), z.stride(1), ok.data_ptr(),
                          ol.data_ptr() if nout == 2 else None, None, ok.stride(0), ok.stride(1),
                          torch.cuda.current_stream().cuda_stream)
            for _ in range(3): run()
            torch.cuda.synchronize()
            s, t = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(5): run()
            t.record(); t.synchronize()
            ms = s.elapsed_time(t) / 5
            ncta = (n + 127) // 128
            cyc_blk = ms * 1e-3 * 1.9e9 / (np.ceil(ncta / 148) * (n // 32))
            print(f"{prec:5s} k={k:3d} nout={nout} {ms:8.3f} ms  ~{cyc_blk:7.0f} cycles/block/CTA", flush=True)
