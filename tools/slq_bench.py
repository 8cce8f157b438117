"""SLQ kernel timing and accuracy: CG coefficients of seeded SPD systems, k probes of m steps.
python tools/slq_bench.py   (KGP_SLQ_GLOBAL toggled in-process: shared vs global scratch)"""
import os
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch
from scipy.linalg import eigh_tridiagonal

from paper_2503_02259_b200 import solver


def cg_coeffs(a, z, m):
    x = np.zeros_like(z)
    r = z.copy()
    p = r.copy()
    rz = r @ r
    al, be = [], []
    for _ in range(m):
        ap = a @ p
        alpha = rz / (p @ ap)
        x += alpha * p
        r -= alpha * ap
        rzn = r @ r
        beta = rzn / rz
        al.append(alpha)
        be.append(beta)
        p = r + beta * p
        rz = rzn
    return np.array(al), np.array(be)


rng = np.random.default_rng(0)
n = 600
q, _ = np.linalg.qr(rng.standard_normal((n, n)))
ev = np.exp(rng.uniform(np.log(1e-2), np.log(1e3), n))
a = (q * ev) @ q.T
for k, m in ((16, 20), (32, 200), (16, 500)):
    al = np.zeros((k, m))
    be = np.zeros((k, m))
    nz = np.zeros(k)
    ref = 0.0
    for c in range(k):
        z = rng.standard_normal(n)
        nz[c] = z @ z
        al[c], be[c] = cg_coeffs(a, z, m)
        d = 1 / al[c] + np.r_[0, be[c][:-1] / al[c][:-1]]
        e = np.sqrt(be[c][:-1]) / al[c][:-1]
        w, v = eigh_tridiagonal(d, e, lapack_driver="stev")
        ref += nz[c] * np.sum(v[0] ** 2 * np.log(w))
    ref /= k
    A, B = torch.from_numpy(al).cuda(), torch.from_numpy(be).cuda()
    it = torch.full((k,), m, dtype=torch.int32, device="cuda")
    N = torch.from_numpy(nz).cuda()
    for mode in ("shared", "global"):
        if mode == "global":
            os.environ["KGP_SLQ_GLOBAL"] = "1"
        else:
            os.environ.pop("KGP_SLQ_GLOBAL", None)
        got = solver.slq_logdet_device(A, B, it, N)
        t0 = time.perf_counter()
        reps = 20
        for _ in range(reps):
            got = solver.slq_logdet_device(A, B, it, N)
        dt = (time.perf_counter() - t0) / reps
        print(f"k={k} m={m} {mode}: {dt * 1e6:8.1f} us  rel err vs stev {abs(got - ref) / abs(ref):.2e}", flush=True)
