"""Time one fused-operator configuration (diagnostic for kernel variants; env knobs such as
KGP_TC_DEBUG / KGP_TC_FLUSH / KGP_TC_MAXSPLIT are read by libkgp at launch).

    python tools/tc_probe.py [n] [k] [nout] [precision] [kernel] [d] [reps]

Prints ms per product (CUDA events over `reps` back-to-back launches after warm-up) and the
implied cycles per 32-column block per CTA at the measured SM clock (NVML, if available)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2503_02259_b200 as kgp
from paper_2503_02259_b200 import _lib, workloads

a = sys.argv[1:]
n = int(a[0]) if len(a) > 0 else 65536
k = int(a[1]) if len(a) > 1 else 32
nout = int(a[2]) if len(a) > 2 else 2
prec = a[3] if len(a) > 3 else "fast"
kt = a[4] if len(a) > 4 else "gaussian"
d = int(a[5]) if len(a) > 5 else 8
reps = int(a[6]) if len(a) > 6 else 10
w = workloads.cfg2(n=n, k=max(k, 1))
x = w.x[:, :d] if d <= 8 else np.random.default_rng(0).standard_normal((n, d))
e = kgp.KernelEngine(kgp.KernelType(kt), x, kgp.Hyperparams(1.0 * np.sqrt(d / 8), 1.0, 1e-2), precision=prec)
z = torch.from_numpy(np.ascontiguousarray(np.random.default_rng(1).standard_normal((n, k)))).cuda()
ok = torch.empty((n, k), dtype=torch.float64, device="cuda")
ol = torch.empty_like(ok)
st = torch.cuda.current_stream()


def run():
    _lib.call("kgp_engine_matmul", e.handle, k, z.data_ptr(), z.stride(0), z.stride(1), ok.data_ptr(),
              ol.data_ptr() if nout == 2 else None, None, ok.stride(0), ok.stride(1), st.cuda_stream)


for _ in range(3):
    run()
torch.cuda.synchronize()
_lib.call("kgp_engine_set_timing", e.handle, 1)
s, t = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(reps):
    run()
t.record()
t.synchronize()
kern_ms, kern_n = _lib.kernel_time(e.handle)
_lib.call("kgp_engine_set_timing", e.handle, 0)
ms = s.elapsed_time(t) / reps
kms = kern_ms / max(kern_n, 1)
mhz = 1965.0
try:
    import pynvml

    pynvml.nvmlInit()
    mhz = float(pynvml.nvmlDeviceGetClockInfo(pynvml.nvmlDeviceGetHandleByIndex(0), pynvml.NVML_CLOCK_SM))
except Exception:
    pass
blocks = (n + 127) // 128 * ((n + 31) // 32) / 148.0
env = " ".join(f"{kk}={v}" for kk, v in sorted(os.environ.items()) if kk.startswith("KGP_TC"))
print(f"{env or 'default':28s} n={n} k={k} nout={nout} {prec} {kt} d={d}: step {ms:.3f} ms, kernel {kms:.3f} ms, "
      f"~{kms * 1e-3 * mhz * 1e6 / blocks:.0f} cycles/block (at {mhz:.0f} MHz)", flush=True)
