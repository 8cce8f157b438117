import sys, time
sys.path.insert(0, "/root/repo")
import torch
import paper_2503_02259_b200 as kgp
from paper_2503_02259_b200 import precond, workloads
from paper_2503_02259_b200.kernels import device_panel
w = workloads.cfg1()
for mode in (kgp.EngineMode.ON_THE_FLY, kgp.EngineMode.DENSE, kgp.EngineMode.ON_THE_FLY):
    e = kgp.KernelEngine(kgp.KernelType.GAUSSIAN, w.x, kgp.Hyperparams(w.l, w.f, w.s), mode=mode, precision="fp64")
    for rep in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        xd = e.x_device(); torch.cuda.synchronize(); t1 = time.perf_counter()
        idx = precond.fps_device(xd, 256, 0); torch.cuda.synchronize(); t2 = time.perf_counter()
        xm = xd.index_select(0, idx)
        k1 = device_panel(e._kid, 0, xm, xd, w.l); torch.cuda.synchronize(); t3 = time.perf_counter()
        pre = precond.build(e, 256); torch.cuda.synchronize(); t4 = time.perf_counter()
        print(mode, rep, f"xdev {1e3*(t1-t0):.1f} fps {1e3*(t2-t1):.1f} panel {1e3*(t3-t2):.1f} build {1e3*(t4-t3):.1f} ms", flush=True)
