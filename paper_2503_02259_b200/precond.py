"""Landmark (Nystrom) preconditioner on the device (kernelgp precond.py:31-126).

Build (precond.py:95-126): farthest-point landmarks (``kgp_fps``), the ridged
landmark block K_mm and the cross block K_mn from the device panel kernel, then
the two Cholesky factorisations and triangular solves through cuSOLVER/cuBLAS
(torch.linalg on CUDA tensors):

    K_mm + ridge I = L L^T,   V^T = L^-1 K_mn,   C = I/f^2 + V^T V / s = L_C L_C^T,
    W^T = L_C^-1 V^T.

Apply (precond.py:74-92), every PCG iteration, in libkgp:
    M^-1 B = B/s - W (W^T B)/s^2          M B = s B + f^2 V (V^T B)
which equals the reference's cho_solve form in exact arithmetic.

``build_afn`` / ``build_adaptive``: the AFN preconditioner the north star names
(landmark Cholesky block + FSAI factor of the Schur complement, afn.cu). The
reference has no AFN (SPEC.md:17, 219-227 substitute Nystrom), so its factors are
checked against the numpy statement in tests/afn_ref.py; it plugs in wherever the
Nystrom object does (``.handle``, ``.apply_inverse``, ``.rank``, ``.landmark_indices``).
"""

from __future__ import annotations

import ctypes
import math

import numpy as np

from paper_2503_02259_b200 import _device
from paper_2503_02259_b200._lib import call
from paper_2503_02259_b200.errors import BreakdownError
from paper_2503_02259_b200.kernels import as_points, device_panel

RIDGE_SCALE = 1e-10
PP_TAIL_SEED = 0x5EED  # second stream of the Nystrom preconditioned-probe draws


def default_rank(n: int) -> int:
    """precond.py:34-36."""
    return min(int(math.ceil(math.sqrt(n))) * 4, 500, n)


def fps_device(xd, m: int, seed_index: int = 0):
    """Farthest-point sampling on a device point tensor; returns an int64 CUDA tensor."""
    torch = _device.torch()
    n, d = xd.shape
    idx = torch.empty(m, dtype=torch.int64, device=xd.device)
    call("kgp_fps", n, d, xd.data_ptr(), m, int(seed_index), idx.data_ptr(), _device.stream_ptr())
    return idx


def fps_select(x, m: int, seed_index: int = 0) -> np.ndarray:
    """Greedy farthest-point landmarks, lowest index on ties (precond.py:39-59)."""
    x = as_points(x, "X")
    n = x.shape[0]
    if not 1 <= m <= n:
        raise ValueError(f"need 1 <= m <= n, got m={m}, n={n}")
    if not 0 <= seed_index < n:
        raise ValueError(f"seed_index {seed_index} out of range for n={n}")
    return _device.to_host(fps_device(_device.to_device(x), m, seed_index)).astype(np.intp)


class _LowRank:
    """Owns one libkgp low-rank handle (U^T on the device)."""

    def __init__(self, ut, s):
        ut = ut.contiguous()  # torch.linalg returns column-major factors; libkgp wants (m, n) row-major
        self.h = ctypes.c_void_p()
        call("kgp_precond_create", ctypes.byref(self.h), ut.shape[1], ut.shape[0], ut.data_ptr(), float(s),
             _device.stream_ptr())

    def close(self):
        if self.h:
            call("kgp_precond_destroy", self.h)
            self.h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class NystromPreconditioner:
    """M = s I + f^2 V V^T with Woodbury inverse, factors resident in HBM."""

    def __init__(self, landmark_indices, shift, inv, fwd, f2, n, logdet=None):
        self.landmark_indices = landmark_indices
        self.shift = float(shift)
        self._inv = inv
        self._fwd = fwd
        self._f2 = float(f2)
        self.n = int(n)
        self.logdet = logdet  # log|M| = n log s + m log f^2 + log|C|, C = I/f^2 + V^T V / s

    def draw_probes(self, probes):
        """Preconditioned-probe draws: w1 = the probe set's vectors, w2 from a second seeded
        stream default_rng([seed..., PP_TAIL_SEED]) (gp.nlml_grad_iterative)."""
        seed = probes.rng_seed if probes.rng_seed is not None else 0
        seed = list(seed) if isinstance(seed, (tuple, list)) else [seed]
        w2 = np.random.default_rng([*seed, PP_TAIL_SEED]).standard_normal((self.rank, probes.k_z))
        return self.sample(probes.vectors, w2)

    def sample(self, w1, w2):
        """Draws z = sqrt(s) w1 + f V w2 ~ N(0, M) from standard normals w1 (n, k), w2 (m, k)
        (host or device); returns a (k, n) CUDA tensor (probe c contiguous)."""
        torch = _device.torch()
        w1 = w1 if _device.is_tensor(w1) else _device.to_device(np.asarray(w1, dtype=np.float64))
        w2 = w2 if _device.is_tensor(w2) else _device.to_device(np.asarray(w2, dtype=np.float64))
        n, k = w1.shape
        if n != self.n or w2.shape != (self.rank, k):
            raise ValueError(f"need w1 ({self.n}, k) and w2 ({self.rank}, k)")
        t = w2.contiguous()
        out = torch.empty((k, n), dtype=torch.float64, device=w1.device)
        call("kgp_lowrank_expand", self._fwd.h, math.sqrt(self.shift), math.sqrt(self._f2), k, w1.data_ptr(),
             w1.stride(0), w1.stride(1), t.data_ptr(), out.data_ptr(), 1, n, _device.stream_ptr())
        return out

    @property
    def rank(self) -> int:
        return len(self.landmark_indices)

    @property
    def handle(self):
        return self._inv.h

    def close(self):
        """Free the device factors now (otherwise at garbage collection)."""
        self._inv.close()
        self._fwd.close()

    def _run(self, which, b, beta, alpha):
        torch = _device.torch()
        host = not _device.is_tensor(b)
        if host:
            b = np.asarray(b, dtype=np.float64)
        squeeze = b.ndim == 1
        bd = _device.to_device(b) if host else b
        if squeeze:
            bd = bd[:, None]
        out = torch.empty((bd.shape[0], bd.shape[1]), dtype=torch.float64, device=bd.device)
        call("kgp_lowrank_apply", which.h, beta, alpha, bd.shape[1], bd.data_ptr(), bd.stride(0), bd.stride(1),
             out.data_ptr(), out.stride(0), out.stride(1), _device.stream_ptr())
        if squeeze:
            out = out[:, 0]
        return _device.to_host(out) if host else out

    def apply_inverse(self, b):
        """inv(M) @ B via Woodbury (precond.py:74-83)."""
        s = self.shift
        return self._run(self._inv, b, 1.0 / s, -1.0 / (s * s))

    def apply(self, b):
        """M @ B (precond.py:85-92)."""
        return self._run(self._fwd, b, self.shift, self._f2)


def build(engine, m: int | None = None, shift: float | None = None) -> NystromPreconditioner:
    """Landmark preconditioner for an engine's Khat (precond.py:95-126). ``shift`` (extension)
    replaces the noise s of M = shift I + f^2 V V^T, e.g. s + the mean heteroscedastic noise
    of a GPC class."""
    torch = _device.torch()
    n = engine.n
    if m is None:
        m = default_rank(n)
    if not 1 <= m <= n:
        raise ValueError(f"need 1 <= m <= n, got m={m}, n={n}")
    p = engine.params
    sh = float(p.s if shift is None else shift)
    if not sh > 0:
        raise ValueError("shift must be positive")
    xd = engine.x_device()
    idx = fps_device(xd, m, 0)
    xm = xd.index_select(0, idx)
    kid = engine._kid
    kmm = device_panel(kid, 0, xm, xm, p.l)
    ridge = RIDGE_SCALE * float(torch.trace(kmm)) / m
    kmm.diagonal().add_(ridge)
    f2 = p.f * p.f

    def fail():
        return BreakdownError(f"landmark factorization failed even after ridge {ridge:.3e}; "
                              "increase the noise term s or reduce the rank m")

    low, info = torch.linalg.cholesky_ex(kmm)
    if int(info) != 0:
        raise fail()
    vt = torch.linalg.solve_triangular(low, device_panel(kid, 0, xm, xd, p.l), upper=False)
    cap = (vt @ vt.T) / sh
    cap.diagonal().add_(1.0 / f2)
    lc, info = torch.linalg.cholesky_ex(cap)
    if int(info) != 0 or not bool(torch.isfinite(vt).all()):
        raise fail()
    wt = torch.linalg.solve_triangular(lc, vt, upper=False)
    inv = _LowRank(wt, sh)
    del wt
    fwd = _LowRank(vt, sh)
    logdet = n * math.log(sh) + m * math.log(f2) + 2.0 * float(torch.log(torch.diagonal(lc)).sum())
    return NystromPreconditioner(_device.to_host(idx).astype(np.intp), sh, inv, fwd, f2, n, logdet)


# ----------------------------------------------------------------------------- AFN
AFN_DEFAULT_NPT = 32     # FSAI neighbours per row
AFN_MAX_NPT = 64


def knn_prev_device(xd, npt: int):
    """(n, npt) int64: for each point its npt nearest earlier points (-1 padded)."""
    torch = _device.torch()
    n, d = xd.shape
    out = torch.empty((n, npt), dtype=torch.int64, device=xd.device)
    call("kgp_knn_prev", n, d, xd.data_ptr(), npt, out.data_ptr(), _device.stream_ptr())
    return out


class AFNPreconditioner:
    """M = L diag(K11, (G^T G)^-1) L^T in the landmark-first ordering; factors in HBM."""

    kind = "afn"

    def __init__(self, handle, landmark_indices, shift, n, npt, logdet=None):
        self._h = handle
        self.landmark_indices = landmark_indices
        self.shift = float(shift)
        self.n = int(n)
        self.fsai_npt = int(npt)
        self.logdet = logdet  # log|M| = log|K11| - 2 sum log G_ii

    def sample(self, w):
        """z ~ N(0, M) from standard normals w (n, k) (host or device): (k, n) CUDA tensor."""
        torch = _device.torch()
        w = w if _device.is_tensor(w) else _device.to_device(np.asarray(w, dtype=np.float64))
        if w.dim() != 2 or w.shape[0] != self.n:
            raise ValueError(f"w must be ({self.n}, k)")
        out = torch.empty((w.shape[1], self.n), dtype=torch.float64, device=w.device)
        call("kgp_afn_sample", self._h, w.shape[1], w.data_ptr(), w.stride(0), w.stride(1), out.data_ptr(),
             _device.stream_ptr())
        return out

    def draw_probes(self, probes):
        """Preconditioned-probe draws for gp.nlml_grad_iterative(preconditioned_probes=...)."""
        return self.sample(probes.vectors)

    @property
    def rank(self) -> int:
        return len(self.landmark_indices)

    @property
    def handle(self):
        return self._h

    def apply_inverse(self, b):
        """inv(M) @ B: landmark solve + FSAI products (afn.cu)."""
        torch = _device.torch()
        host = not _device.is_tensor(b)
        if host:
            b = np.asarray(b, dtype=np.float64)
        squeeze = b.ndim == 1
        bd = _device.to_device(b) if host else b
        if squeeze:
            bd = bd[:, None]
        if bd.shape[0] != self.n:
            raise ValueError(f"B has {bd.shape[0]} rows, preconditioner has {self.n}")
        out = torch.empty((bd.shape[0], bd.shape[1]), dtype=torch.float64, device=bd.device)
        call("kgp_precond_apply_inverse", self._h, bd.shape[1], bd.data_ptr(), bd.stride(0), bd.stride(1),
             out.data_ptr(), out.stride(0), out.stride(1), _device.stream_ptr())
        if squeeze:
            out = out[:, 0]
        return _device.to_host(out) if host else out

    def close(self):
        if self._h:
            call("kgp_precond_destroy", self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def build_afn(engine, m: int | None = None, fsai_npt: int = AFN_DEFAULT_NPT, diag=None) -> AFNPreconditioner:
    """AFN for an engine's Khat: m FPS landmarks (exact block) + FSAI of the Schur complement.
    ``diag`` (n,) adds a per-point shift: the preconditioner then targets Khat + diag(diag)
    (one class of the Dirichlet GPC, gpc.py)."""
    torch = _device.torch()
    n = engine.n
    if m is None:
        m = default_rank(n)
    if not 1 <= m < n:
        raise ValueError(f"AFN needs 1 <= m < n, got m={m}, n={n}")
    if not 1 <= fsai_npt <= AFN_MAX_NPT:
        raise ValueError(f"fsai_npt must be in [1, {AFN_MAX_NPT}], got {fsai_npt}")
    p = engine.params
    f2 = p.f * p.f
    xd = engine.x_device()
    kid = engine._kid
    dev = xd.device
    idx = fps_device(xd, m, 0)
    mask = torch.ones(n, dtype=torch.bool, device=dev)
    mask[idx] = False
    rest = torch.nonzero(mask).squeeze(1)
    perm = torch.cat([idx, rest]).contiguous()
    n2 = n - m
    x1 = xd.index_select(0, idx).contiguous()
    x2 = xd.index_select(0, rest).contiguous()
    dd = None
    if diag is not None:
        dd = diag if _device.is_tensor(diag) else torch.from_numpy(np.asarray(diag, dtype=np.float64))
        dd = dd.to(device=dev, dtype=torch.float64).reshape(-1)
        if dd.shape[0] != n:
            raise ValueError(f"diag must have length {n}, got {dd.shape[0]}")
    k11 = device_panel(kid, 0, x1, x1, p.l).mul_(f2)
    k11.diagonal().add_(p.s)
    if dd is not None:
        k11.diagonal().add_(dd.index_select(0, idx))
    low, info = torch.linalg.cholesky_ex(k11)
    if int(info) != 0:
        raise BreakdownError("AFN landmark block is not positive definite; increase s or reduce m")
    wt = torch.linalg.solve_triangular(low, device_panel(kid, 0, x1, x2, p.l).mul_(f2), upper=False)
    w = wt.T.contiguous()
    del wt
    linv = torch.linalg.solve_triangular(low, torch.eye(m, dtype=torch.float64, device=dev), upper=False)
    linv = linv.contiguous()
    npt = int(fsai_npt)
    nbr = knn_prev_device(x2, npt)
    gval = torch.empty((npt + 1, n2), dtype=torch.float64, device=dev)
    gcol = torch.empty((npt + 1, n2), dtype=torch.int32, device=dev)
    d2 = None if dd is None else dd.index_select(0, rest).contiguous()
    call("kgp_afn_fsai", kid, n2, x2.shape[1], x2.data_ptr(), float(p.l), float(p.f), float(p.s),
         None if d2 is None else d2.data_ptr(), m, w.data_ptr(), npt, nbr.data_ptr(), gval.data_ptr(),
         gcol.data_ptr(), _device.stream_ptr())
    # G^T as CSR: entries sorted by (column, row)
    rows = torch.arange(n2, dtype=torch.int64, device=dev).expand(npt + 1, n2).reshape(-1)
    cols = gcol.reshape(-1).to(torch.int64)
    ok = cols >= 0
    rows, cols, vals = rows[ok], cols[ok], gval.reshape(-1)[ok]
    order = torch.argsort(cols * n2 + rows)
    gtrow = rows[order].to(torch.int32).contiguous()
    gtval = vals[order].contiguous()
    gtptr = torch.zeros(n2 + 1, dtype=torch.int64, device=dev)
    gtptr[1:] = torch.cumsum(torch.bincount(cols, minlength=n2), 0)
    gtptr = gtptr.to(torch.int32).contiguous()
    low = low.contiguous()
    h = ctypes.c_void_p()
    call("kgp_afn_create", ctypes.byref(h), n, m, perm.data_ptr(), linv.data_ptr(), low.data_ptr(), w.data_ptr(),
         npt + 1, gval.data_ptr(), gcol.data_ptr(), int(gtrow.numel()), gtptr.data_ptr(), gtrow.data_ptr(),
         gtval.data_ptr(), float(p.s), _device.stream_ptr())
    diag_g = gval[gcol == torch.arange(n2, dtype=torch.int32, device=dev)[None, :]]  # G_ii (one per row)
    logdet = 2.0 * float(torch.log(torch.diagonal(low)).sum()) - 2.0 * float(torch.log(diag_g).sum())
    return AFNPreconditioner(h, _device.to_host(idx).astype(np.intp), p.s, n, npt, logdet)


def estimate_rank(engine, sample: int = 1000, seed: int = 0) -> int:
    """Numerical rank of f^2 kappa(X, X) at the noise level s, from a seeded row sample:
    eigenvalues of the sample kernel scaled by n/sample that exceed s."""
    torch = _device.torch()
    n = engine.n
    ns = min(n, sample)
    p = engine.params
    rng = np.random.default_rng(seed)
    pick = np.sort(rng.choice(n, ns, replace=False)) if ns < n else np.arange(n)
    xs = engine.x_device().index_select(0, torch.as_tensor(pick, device=engine.x_device().device))
    ks = device_panel(engine._kid, 0, xs, xs, p.l).mul_(p.f * p.f * n / ns)
    ev = torch.linalg.eigvalsh(ks)
    return int((ev > p.s).sum())


def build_adaptive(engine, m: int | None = None, fsai_npt: int = AFN_DEFAULT_NPT):
    """AFN's adaptive choice: Nystrom(m) when the kernel's numerical rank fits in m
    landmarks, the factorized AFN otherwise."""
    n = engine.n
    if m is None:
        m = default_rank(n)
    if m >= n or estimate_rank(engine) <= m:
        return build(engine, m)
    return build_afn(engine, m, fsai_npt)
