import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2503_02259_b200 import precond
for n, d in ((65536, 4), (262144, 4), (131072, 8)):
    x = np.random.default_rng(0).uniform(0, 1, (n, d))
    nbr = precond.knn_prev_device(torch.from_numpy(x).cuda(), 32).cpu().numpy()
    lev = np.zeros(n, dtype=np.int64)
    for i in range(n):
        nb = nbr[i]; nb = nb[nb >= 0]
        if nb.size: lev[i] = lev[nb].max() + 1
    print(n, d, "levels", lev.max() + 1, "mean rows/level", n / (lev.max() + 1), flush=True)
