"""Numpy statement of the Dirichlet GP classification loss (gpc.py) — TEST HELPER.

No reference counterpart exists; this restates Milios et al. (2018)'s
label transformation and the summed per-class GP regression NLML densely, plus the
same-probe stochastic estimator the iterative path computes (the check the reference
makes for GPR in test_gp.py:104-119: iterative terms vs dense terms with the same probes).
"""

import math

import numpy as np

from oracle import kgp_oracle as orc


def transform(labels, num_classes, alpha_eps=0.01):
    onehot = (labels[None, :] == np.arange(num_classes)[:, None]).astype(np.float64)
    alpha = alpha_eps + onehot
    noise = np.log(1.0 / alpha + 1.0)
    t = np.log(alpha) - 0.5 * noise
    return t - t.mean(axis=1, keepdims=True), noise


def _mats(kt, x, l, f, s):
    kap = orc.eval_kernel(kt, x, x, l)
    return f * f * kap + s * np.eye(len(x)), [f * f * orc.eval_kernel_grad_l(kt, x, x, l), 2.0 * f * kap,
                                              np.eye(len(x))]


def exact(kt, x, targets, noise, l, f, s):
    kb, dks = _mats(kt, x, l, f, s)
    n = len(x)
    loss, g = 0.0, np.zeros(3)
    for c in range(len(targets)):
        k = kb + np.diag(noise[c])
        kinv = np.linalg.inv(k)
        w = kinv @ targets[c]
        loss += 0.5 * (targets[c] @ w + np.linalg.slogdet(k)[1] + n * math.log(2 * math.pi))
        for i, dk in enumerate(dks):
            g[i] += 0.5 * (-w @ dk @ w + np.trace(kinv @ dk))
    return loss, g


def estimator(kt, x, targets, noise, l, f, s, probes):
    """Same probes (C*k_z, n): logdet ~ mean z^T log(K) z, trace ~ mean z^T K^-1 dK z."""
    kb, dks = _mats(kt, x, l, f, s)
    n, c = len(x), len(targets)
    kz = probes.shape[0] // c
    loss, g = 0.0, np.zeros(3)
    for k in range(c):
        kk = kb + np.diag(noise[k])
        ev, vec = np.linalg.eigh(kk)
        logk = (vec * np.log(ev)) @ vec.T
        kinv = (vec / ev) @ vec.T
        z = probes[k * kz:(k + 1) * kz].T
        w = kinv @ targets[k]
        loss += 0.5 * (targets[k] @ w + np.einsum("ij,ij->", z, logk @ z) / kz + n * math.log(2 * math.pi))
        for i, dk in enumerate(dks):
            g[i] += 0.5 * (-w @ dk @ w + np.einsum("ij,ij->", kinv @ z, dk @ z) / kz)
    return loss, g
