"""Per-rank cost of the row-sharded fused operator, measured one shard at a time on ONE GPU.

Rank r of N owns rows [r*n/N, (r+1)*n/N) and multiplies them against the full (replicated)
RHS, so every rank's work is independent: timing each shard alone on one B200 gives the
per-rank step time, and t(1) / (N * max_r t_r(N)) is the strong-scaling efficiency of the
data path (the bench's multi-GPU value has no collective inside the timed region).

    python tools/rowshard_scale.py [n] [k] [maxsplit ...]
"""
import os
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_2503_02259_b200 as kgp
from paper_2503_02259_b200 import _lib, workloads

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
k = int(sys.argv[2]) if len(sys.argv) > 2 else 32
splits = [int(a) for a in sys.argv[3:]] or [8]
w = workloads.cfg2(n=n, k=k)
e = kgp.KernelEngine(kgp.KernelType.GAUSSIAN, w.x, kgp.Hyperparams(w.l, w.f, w.s), precision="fast")
z = torch.from_numpy(w.z).cuda()
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
st = torch.cuda.current_stream()


def time_rows(r0, rows, steps=10):
    _lib.call("kgp_engine_set_rows", e.handle, r0, rows)
    ok = torch.empty((rows, k), dtype=torch.float64, device="cuda")
    ol = torch.empty_like(ok)

    def step():
        _lib.call("kgp_engine_matmul", e.handle, k, z.data_ptr(), z.stride(0), z.stride(1), ok.data_ptr(),
                  ol.data_ptr(), None, ok.stride(0), ok.stride(1), st.cuda_stream)

    for _ in range(3):
        step()
    ts = []
    for _ in range(steps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        step()
        b.record(st)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


for ms in splits:
    os.environ["KGP_TC_MAXSPLIT"] = str(ms)
    t1 = time_rows(0, n)
    for N in (1, 2, 4, 8):
        per = []
        for r in sorted({0, N - 1}):
            r0, r1 = r * n // N, (r + 1) * n // N
            per.append(time_rows(r0, r1 - r0))
        tN = max(per)
        print(f"n={n} k={k} maxsplit={ms} N={N}: per-rank ms {['%.3f' % t for t in per]} "
              f"eff {t1 / (N * tN):.3f}", flush=True)
