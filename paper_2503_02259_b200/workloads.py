"""Seeded synthetic inputs for the five BASELINE.json configurations.

The reference names no dataset; every input here is drawn
from ``numpy.random.default_rng(seed)`` with the shapes, value distributions
and hyperparameters BASELINE.json states. ``n`` (and ``m_test``) can be
reduced for parity runs that must finish on the CPU oracle in seconds; the
generator is otherwise identical, so a reduced instance is a prefix-free
redraw with the same recipe, not a row subsample.

Draw order is fixed and documented per function (X first, then noise), so the
golden fixtures in ``tests/golden`` can be regenerated bit-for-bit.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np


@dataclass
class Workload:
    name: str
    kernel: str            # "gaussian" | "matern32" | "matern52"
    x: np.ndarray          # (n, d) float64 (fp32-representable when the config says fp32)
    l: float
    f: float
    s: float
    y: np.ndarray | None = None          # (n,) regression targets
    z: np.ndarray | None = None          # (n, k) RHS block for the standalone MatMul
    k_z: int = 0                         # probe count for NLML configs
    probe_seed: int = 0
    rank: int = 0                        # preconditioner rank
    extra: dict = field(default_factory=dict)

    @property
    def n(self) -> int:
        return self.x.shape[0]

    @property
    def d(self) -> int:
        return self.x.shape[1]


def cfg1(n: int = 4096, seed: int = 0) -> Workload:
    """GPR NLML+gradient, Gaussian, d=3, X~U[0,1]^3 (fp64), l=0.3 f=1 s=1e-2,
    16 probes, rank 256, PCG 50 iterations + 20 Lanczos steps (BASELINE.json configs[0])."""
    rng = np.random.default_rng(seed)
    x = rng.uniform(0.0, 1.0, (n, 3))
    y = (np.sin(2 * math.pi * x[:, 0]) * np.cos(2 * math.pi * x[:, 1]) + x[:, 2]
         + 0.1 * rng.standard_normal(n))
    return Workload("cfg1", "gaussian", x, 0.3, 1.0, 1e-2, y=y, k_z=16, probe_seed=seed,
                    rank=min(256, n), extra={"pcg_iters": 50, "slq_steps": 20})


def cfg2(n: int = 65536, k: int = 32, seed: int = 0) -> Workload:
    """Standalone fused MatMul: Gaussian, d=8, X~N(0,I) fp32, Z (n,32) N(0,1) fp32,
    l=1 f=1 s=1e-2; outputs Khat.Z and dKhat/dl.Z (BASELINE.json configs[1])."""
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((n, 8)).astype(np.float32).astype(np.float64)
    z = rng.standard_normal((n, k)).astype(np.float32).astype(np.float64)
    return Workload("cfg2", "gaussian", x, 1.0, 1.0, 1e-2, z=z)


def cfg3(n: int = 262144, seed: int = 0, k_z: int = 32) -> Workload:
    """GPR NLML+gradient, Matern-3/2, d=4, X~U[0,1]^4 fp32, y=sum sin(3x_k)+N(0,0.05^2),
    l=0.2 f=1.5 s=1e-3, 32 probes, rank 1024, PCG tol 1e-6 (configs[2])."""
    rng = np.random.default_rng(seed)
    x = rng.uniform(0.0, 1.0, (n, 4)).astype(np.float32).astype(np.float64)
    y = np.sin(3.0 * x).sum(axis=1) + 0.05 * rng.standard_normal(n)
    return Workload("cfg3", "matern32", x, 0.2, 1.5, 1e-3, y=y, k_z=k_z, probe_seed=seed,
                    rank=min(1024, n), extra={"tol": 1e-6})


def cfg4(n: int = 131072, seed: int = 0) -> Workload:
    """GPC 3-class (BASELINE configs[3]): Gaussian, d=8, X~N(0,I) fp32, labels = argmax of
    3 latent GP draws (l=1) from the seed, 16 probes, AFN rank 512, 10 training steps.

    The reference has no GPC and no large-n GP sampler: the latent draws
    are random-Fourier-feature draws of the l=1 Gaussian GP (gpc.sample_latent_labels),
    labels in extra["labels"]."""
    from paper_2503_02259_b200.gpc import sample_latent_labels

    rng = np.random.default_rng(seed)
    x = rng.standard_normal((n, 8)).astype(np.float32).astype(np.float64)
    labels = sample_latent_labels(x, 3, l=1.0, seed=seed)
    return Workload("cfg4", "gaussian", x, 1.0, 1.0, 1e-2, k_z=16, probe_seed=seed,
                    rank=min(512, n), extra={"labels": labels, "classes": 3, "train_steps": 10})


def cfg5(n: int = 1048576, m_test: int = 262144, seed: int = 0) -> Workload:
    """Large-scale GPR train+predict: Matern-5/2, d=2, X~U[0,1]^2 fp32,
    y=sin(4 pi x1)+cos(4 pi x2)+N(0,0.1^2), 64 RHS (y + 63 probes), rank 2048."""
    rng = np.random.default_rng(seed)
    x = rng.uniform(0.0, 1.0, (n, 2)).astype(np.float32).astype(np.float64)
    y = (np.sin(4 * math.pi * x[:, 0]) + np.cos(4 * math.pi * x[:, 1])
         + 0.1 * rng.standard_normal(n))
    xs = rng.uniform(0.0, 1.0, (m_test, 2)).astype(np.float32).astype(np.float64)
    return Workload("cfg5", "matern52", x, 0.1, 1.0, 1e-2, y=y, k_z=63, probe_seed=seed,
                    rank=min(2048, n), extra={"xstar": xs})
