"""Accuracy (cfg2, 512-row oracle subsample) and time of the fast operator for the current
KGP_TC_FLUSH (run once per value: the flush is read at first use)."""
import os, sys
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import numpy as np
import torch
import paper_2503_02259_b200 as kgp
from paper_2503_02259_b200 import _lib, workloads
from oracle import kgp_oracle_c as oc
from conftest import rel_max

w = workloads.cfg2()
e = kgp.KernelEngine(kgp.KernelType.GAUSSIAN, w.x, kgp.Hyperparams(w.l, w.f, w.s), precision="fast")
zd = torch.from_numpy(w.z).cuda()
kk, dl, _ = e.apply(zd, True, True, False)
rows = np.sort(np.random.default_rng(7).choice(w.n, 256, replace=False))
kk, dl = kk.cpu().numpy()[rows], dl.cpu().numpy()[rows]
refk = np.empty((len(rows), w.z.shape[1])); refd = np.empty_like(refk)
for i, gi in enumerate(rows):
    a, bb = oc.matmul("gaussian", w.x, w.l, w.f, w.s, w.z, row0=int(gi), nrows=1, want_dl=True)
    refk[i], refd[i] = a[0], bb[0]
ok = torch.empty((w.n, 32), dtype=torch.float64, device="cuda"); ol = torch.empty_like(ok)
def run():
    _lib.call("kgp_engine_matmul", e.handle, 32, zd.data_ptr(), zd.stride(0), zd.stride(1), ok.data_ptr(),
              ol.data_ptr(), None, ok.stride(0), ok.stride(1), torch.cuda.current_stream().cuda_stream)
for _ in range(3): run()
torch.cuda.synchronize()
s, t = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10): run()
t.record(); t.synchronize()
print(f"flush={os.environ.get('KGP_TC_FLUSH', '8')}: {s.elapsed_time(t) / 10:.3f} ms  errK {rel_max(kk, refk):.2e}  "
      f"errG {rel_max(dl, refd):.2e}", flush=True)
