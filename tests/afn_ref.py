"""Numpy statement of the AFN (adaptive factorized Nystrom) preconditioner — TEST HELPER.

The reference has no AFN: its SPEC leaves the AFN internals out
and substitutes the Nystrom preconditioner. The north star asks for AFN on the device
(landmark Cholesky solve plus a sparse FSAI factor), so this module restates the
algorithm the CUDA path implements in plain numpy,
for checking the device factors and applications at small n. Parity with HiGP's own
AFN is unpinned.

Ordering: landmarks X1 (FPS, k points) first, the rest X2 in original order.
    Khat = [K11 K12; K21 K22],  K11 = L L^T,  W = K21 L^-T,  S = K22 - W W^T
    S^-1 ~ G^T G,  G lower triangular, row i supported on {i} and the npt nearest
    points j < i of X2 (FSAI: S_PP z = e_i scaled so (G S G^T)_ii = 1)
    M^-1 b = [L^-T (y1 - W^T u2); u2],  y1 = L^-1 b1,  u2 = G^T G (b2 - W y1)
"""

from __future__ import annotations

import numpy as np
from scipy.linalg import cholesky, solve_triangular

from oracle import kgp_oracle as orc


def knn_prev(x, npt):
    """For each i, the npt nearest j < i (squared distance, ties to the lower j), -1 padded."""
    n = x.shape[0]
    out = -np.ones((n, npt), dtype=np.int64)
    for i in range(1, n):
        r2 = orc.sqdist(x[i:i + 1], x[:i])[0]
        order = np.lexsort((np.arange(i), r2))[:npt]
        out[i, :len(order)] = order
    return out


def fsai(kt, x2, l, f, s, w, nbr):
    """Rows of G: (n2, npt+1) values and columns (neighbours by distance, then i); -1 padded."""
    n2, npt = nbr.shape
    gval = np.zeros((n2, npt + 1))
    gcol = -np.ones((n2, npt + 1), dtype=np.int64)
    for i in range(n2):
        p = [int(j) for j in nbr[i] if j >= 0] + [i]
        xp = x2[p]
        spp = f * f * orc.eval_kernel(kt, xp, xp, l) + s * np.eye(len(p)) - w[p] @ w[p].T
        low = cholesky(spp, lower=True)
        e = np.zeros(len(p))
        e[-1] = 1.0
        z = solve_triangular(low.T, e, lower=False)
        gval[i, :len(p)] = z
        gcol[i, :len(p)] = p
    return gval, gcol


class AFN:
    def __init__(self, kt, x, l, f, s, k, npt):
        n = x.shape[0]
        idx = orc.fps(x, k, 0)
        mask = np.ones(n, dtype=bool)
        mask[idx] = False
        rest = np.nonzero(mask)[0]
        self.perm = np.concatenate([idx, rest])
        x1, x2 = x[idx], x[rest]
        k11 = f * f * orc.eval_kernel(kt, x1, x1, l) + s * np.eye(k)
        self.low = cholesky(k11, lower=True)
        k12 = f * f * orc.eval_kernel(kt, x1, x2, l)
        self.w = solve_triangular(self.low, k12, lower=True).T.copy()
        self.nbr = knn_prev(x2, npt)
        self.gval, self.gcol = fsai(kt, x2, l, f, s, self.w, self.nbr)
        self.n, self.k = n, k

    def g_matvec(self, v):
        out = np.zeros_like(v)
        for t in range(self.gval.shape[1]):
            c = self.gcol[:, t]
            ok = c >= 0
            out[ok] += self.gval[ok, t][:, None] * v[c[ok]]
        return out

    def gt_matvec(self, v):
        out = np.zeros_like(v)
        for t in range(self.gval.shape[1]):
            c = self.gcol[:, t]
            ok = c >= 0
            np.add.at(out, c[ok], self.gval[ok, t][:, None] * v[ok])
        return out

    def apply_inverse(self, b):
        b = np.asarray(b, dtype=np.float64)
        squeeze = b.ndim == 1
        if squeeze:
            b = b[:, None]
        bp = b[self.perm]
        y1 = solve_triangular(self.low, bp[:self.k], lower=True)
        t2 = bp[self.k:] - self.w @ y1
        u2 = self.gt_matvec(self.g_matvec(t2))
        o1 = solve_triangular(self.low.T, y1 - self.w.T @ u2, lower=False)
        out = np.empty_like(b)
        out[self.perm] = np.concatenate([o1, u2])
        return out[:, 0] if squeeze else out
