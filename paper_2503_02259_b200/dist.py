"""Row-partitioned multi-GPU PCG / NLML+gradient.

A preconditioner whose application does not shard by rows (AFN: its FSAI factor couples
each row to its nearest earlier points anywhere in X) is REPLICATED instead: every rank
holds the full factor, the residual is all-gathered (one more n x k exchange per
iteration, the same volume as the operator's) and each rank keeps its rows of M^-1 r
(``ops.replicated_minv``).

One process per GPU. X is replicated (n*d*8 bytes); every n-vector -- the PCG
state, y, the probes -- is split into contiguous row blocks, rank g owning rows
I_g. One operator application is

    P_full = all_gather(P_g)                (NCCL over NVLink; k x n fp64)
    (K^ P)_g = K^[I_g, :] . P_full          (libkgp fused kernel, rows I_g only)

and the per-column PCG scalars (p.Ap, r.r, r.z) are all-reduced (2k doubles per
iteration), so alpha/beta -- and therefore every freeze decision and the Lanczos
coefficients that feed SLQ -- are bitwise identical on all ranks. The Woodbury
preconditioner keeps W row-sharded too: W_g^T R_g is all-reduced (m x k) before
the local expansion. SLQ is replicated (scalars only). Gradient: local partial
dots, one all-reduce of 3(1+k_z) values.

The recurrences are the reference's (solver.py:143-192, gp.py:133-179). They run
over a small "local ops" interface so the host-side logic is exercised on the
CPU with gloo (tests/test_dist.py injects an oracle-backed implementation);
``CudaRowOps`` is the GPU implementation (libkgp).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from paper_2503_02259_b200.errors import BreakdownError, NumericalError

LOG_2PI = math.log(2.0 * math.pi)


def row_range(n: int, world: int, rank: int, align: int = 1):
    """Balanced contiguous row block of `rank`; inner boundaries rounded down to multiples of
    `align` (32 for the fused all-gather operator: its column blocks)."""
    def edge(q):
        return n if q >= world else (q * n // world) // align * align
    return edge(rank), edge(rank + 1)


class Comm:
    """The two collectives the solver needs, over torch.distributed (nccl or gloo)."""

    def __init__(self, n: int, group=None, align: int = 1):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.n = n
        self.ranges = [row_range(n, self.world, r, align) for r in range(self.world)]
        self.maxloc = max(r1 - r0 for r0, r1 in self.ranges)
        self.nccl = dist.get_backend(group) == "nccl"

    def allgather_rows(self, x_loc, ranges=None):
        """(k, n_loc) on every rank -> (k, n) full, rows in rank order (``ranges``: another
        balanced split than the training rows', e.g. of the test points)."""
        torch = __import__("torch")
        k, nloc = x_loc.shape
        if self.world == 1:
            return x_loc
        ranges = self.ranges if ranges is None else ranges
        maxloc = max(r1 - r0 for r0, r1 in ranges)
        pad = torch.zeros((k, maxloc), dtype=x_loc.dtype, device=x_loc.device)
        pad[:, :nloc] = x_loc
        if self.nccl:
            buf = torch.empty((self.world, k, maxloc), dtype=x_loc.dtype, device=x_loc.device)
            self.dist.all_gather_into_tensor(buf, pad, group=self.group)
            parts = [buf[r] for r in range(self.world)]
        else:
            parts = [torch.empty_like(pad) for _ in range(self.world)]
            self.dist.all_gather(parts, pad, group=self.group)
        return torch.cat([parts[r][:, :r1 - r0] for r, (r0, r1) in enumerate(ranges)], dim=1)

    def allreduce(self, t):
        if self.world > 1:
            self.dist.all_reduce(t, group=self.group)
        return t


@dataclass
class DistSolve:
    x: object          # (k, n_loc) local rows of the solution
    alphas: object     # (k, max_iter), identical on all ranks
    betas: object
    iters: np.ndarray  # (k,)
    rel: np.ndarray
    converged: np.ndarray


def dist_pcg(ops, comm: Comm, y_loc, tol, max_iter: int, precondition, shift: float = 1.0, diag_loc=None,
             minv_fn=None, check_every: int = 8):
    """Batched PCG over row-sharded state (solver.py:122-192). y_loc: (k, n_loc).

    Column groups as the device driver's (pcg.cu pcg_grouped_impl): ``tol`` and the
    per-column iteration cap may be scalars or length-k arrays, and ``precondition`` a bool
    or the number of LEADING columns to precondition -- so the NLML's w-solve and probe solves
    share one operator application (one all-gather) per iteration.

    ``diag_loc`` (k, n_loc): a per-column diagonal added to the operator on the local rows
    (column j solves (Khat + diag(d_j)) x = y_j -- the Dirichlet GPC classes, the device
    path's kgp_engine_set_diag). ``minv_fn(head_loc) -> z_loc`` replaces the built-in
    preconditioner on the leading columns (e.g. one replicated handle per GPC class).

    Device-resident: every per-column scalar (alpha, beta, rz, rel, the active mask, the
    iteration counts, the breakdown flags) lives in device tensors, the dot products are
    all-reduced in-stream (NCCL on GPUs: two all-reduces of k or 2k values per iteration, no
    host synchronisation), and the host reads the active count only every ``check_every``
    iterations -- iterations issued past a column's stop are masked no-ops (alpha = 0,
    p unchanged), the pcg.cu driver's look-ahead. Per column the recurrence is the
    reference's, so results equal a per-iteration host loop's."""
    torch = __import__("torch")
    k = y_loc.shape[0]
    tol_h = np.broadcast_to(np.asarray(tol, dtype=np.float64), (k,)).copy()
    cap_h = np.broadcast_to(np.asarray(max_iter, dtype=np.int64), (k,)).copy()
    if np.any(tol_h < 0) or np.any(cap_h < 1):
        raise ValueError("need tol >= 0 and max_iter >= 1")
    kp = k if precondition is True else (0 if precondition is False else int(precondition))
    stride = int(cap_h.max())
    dev, f64 = y_loc.device, torch.float64
    tol_d = torch.from_numpy(tol_h).to(dev)
    cap_d = torch.from_numpy(cap_h).to(dev)

    def rowdots(*pairs):
        """all-reduced per-column dots of each (a, b) pair, one collective: (len(pairs), k)."""
        part = torch.stack([(a * b).sum(dim=1) for a, b in pairs])
        return comm.allreduce(part)

    full_minv = getattr(ops, "replicated_minv", None)
    r0, r1 = comm.ranges[comm.rank]

    def minv(r):
        if kp == 0:
            return r
        head = r[:kp]
        if minv_fn is not None:
            zh = minv_fn(head)
        elif full_minv is not None:  # replicated preconditioner (AFN): gather, apply, keep own rows
            zh = full_minv(comm.allgather_rows(head))[:, r0:r1].contiguous()
        else:
            t = comm.allreduce(ops.project(head))
            zh = ops.expand(head, t, 1.0 / shift, -1.0 / (shift * shift))
        return zh if kp == k else torch.cat([zh, r[kp:]], dim=0)

    x = torch.zeros_like(y_loc)
    r = y_loc.clone()
    ynorm = torch.sqrt(rowdots((r, r))[0])
    rel = torch.where(ynorm > 0, torch.ones_like(ynorm), torch.zeros_like(ynorm))
    active = rel > tol_d
    alphas = torch.zeros((k, stride), dtype=f64, device=dev)
    betas = torch.zeros((k, stride), dtype=f64, device=dev)
    iters = torch.zeros(k, dtype=torch.int64, device=dev)
    colbase = torch.arange(k, device=dev) * stride
    brk_col = torch.full((), -1, dtype=torch.int64, device=dev)     # first column that broke down
    brk_val = torch.zeros((), dtype=f64, device=dev)
    nonfinite = torch.zeros((), dtype=torch.bool, device=dev)
    safe_ynorm = torch.where(ynorm > 0, ynorm, torch.ones_like(ynorm))

    def check():
        c = int(brk_col.item())
        if c >= 0:
            raise BreakdownError(f"p^T A p = {float(brk_val.item())} in column {c}; operator is not SPD")
        if bool(nonfinite.item()):
            raise NumericalError("residual became non-finite during PCG")

    if bool(active.any().item()):
        z = minv(r)
        p = z.clone()
        rz = rowdots((r, z))[0]
        peer = getattr(ops, "matmul_local", None)  # fused all-gather operator (PeerTiles)
        for it in range(stride):
            ap = peer(p) if peer is not None else ops.matmul_rows(comm.allgather_rows(p))
            if diag_loc is not None:
                ap = ap + diag_loc * p
            pap = rowdots((p, ap))[0]
            bad = active & (~torch.isfinite(pap) | (pap <= 0.0))
            first = torch.where(bad, torch.arange(k, device=dev), torch.full_like(iters, k)).min()
            newbrk = (brk_col < 0) & (first < k)
            brk_val = torch.where(newbrk, pap[first.clamp(max=k - 1)], brk_val)
            brk_col = torch.where(newbrk, first, brk_col)
            alpha = torch.where(active, rz / torch.where(active, pap, torch.ones_like(pap)), torch.zeros_like(pap))
            x += alpha[:, None] * p
            r -= alpha[:, None] * ap
            slot = colbase + iters.clamp(max=stride - 1)
            flat_a = alphas.view(-1)
            flat_a[slot] = torch.where(active, alpha, flat_a[slot])
            z = minv(r)
            if kp > 0:  # unpreconditioned columns have z = r, so r.z is their r.r bit for bit
                d = rowdots((r, r), (r, z))
                rr, rzn = d[0], d[1]
            else:
                rr = rowdots((r, r))[0]
                rzn = rr
            nonfinite = nonfinite | (active & ~torch.isfinite(rr)).any()
            beta = torch.where(active, rzn / torch.where(active, rz, torch.ones_like(rz)), torch.zeros_like(rz))
            flat_b = betas.view(-1)
            flat_b[slot] = torch.where(active, beta, flat_b[slot])
            iters = iters + active.to(torch.int64)
            rz = torch.where(active, rzn, rz)
            rel = torch.where(active, torch.sqrt(rr) / safe_ynorm, rel)
            active = active & (rel > tol_d) & (iters < cap_d)
            p = torch.where(active[:, None], z + beta[:, None] * p, p)
            if (it + 1) % check_every == 0 or it + 1 == stride:
                check()
                if not bool(active.any().item()):
                    break
        check()
    rel_h = rel.cpu().numpy()
    return DistSolve(x, alphas, betas, iters.cpu().numpy(), rel_h, rel_h <= tol_h)


def _grads(ops, comm, v_loc):
    """This rank's rows of dKhat/dl V and dKhat/df V: through the fused all-gather operator
    when ``ops`` has one (``grads_local``), else all_gather + row-block product."""
    local = getattr(ops, "grads_local", None)
    if local is not None:
        return local(v_loc)
    return ops.grads_rows(comm.allgather_rows(v_loc))


def dist_nlml_grad(ops, comm: Comm, y_loc, probes_loc, norms_sq, tol, max_iter, probe_tol=None,
                   precondition=True, shift=1.0, probe_max_iter=None):
    """nlml_grad_iterative (gp.py:133-179) over row-sharded vectors.

    y_loc: (n_loc,), probes_loc: (k_z, n_loc) local rows; norms_sq: (k_z,) full |z|^2.
    Returns (loss, grad_l, grad_f, grad_s, converged), identical on every rank."""
    torch = __import__("torch")
    probe_tol = tol if probe_tol is None else probe_tol
    probe_max_iter = max_iter if probe_max_iter is None else probe_max_iter
    kz = probes_loc.shape[0]
    # the w-solve (preconditioned) and the probe solves (not) as ONE grouped PCG: every
    # iteration is one all-gather + one fused Khat [p_w, P_Z] on the local rows
    torch_ = __import__("torch")
    v0 = torch_.cat([y_loc[None, :], probes_loc], dim=0)
    tols = np.array([tol] + [probe_tol] * kz)
    caps = np.array([max_iter] + [probe_max_iter] * kz)
    sol = dist_pcg(ops, comm, v0, tols, caps, 1 if precondition else False, shift)
    us = DistSolve(sol.x[1:], sol.alphas[1:], sol.betas[1:], sol.iters[1:], sol.rel[1:], sol.converged[1:])
    ws = DistSolve(sol.x[:1], sol.alphas[:1], sol.betas[:1], sol.iters[:1], sol.rel[:1], sol.converged[:1])
    logdet = ops.slq(us.alphas, us.betas, us.iters, norms_sq)
    w = ws.x[0]
    yw = float(comm.allreduce((y_loc * w).sum()[None])[0])
    loss = 0.5 * (yw + logdet + comm.n * LOG_2PI)
    v_loc = torch.cat([w[None, :], probes_loc], dim=0)
    u_loc = torch.cat([w[None, :], us.x], dim=0)
    dl, df = _grads(ops, comm, v_loc)
    part = torch.stack([(u_loc * dl).sum(dim=1), (u_loc * df).sum(dim=1), (u_loc * v_loc).sum(dim=1)])
    part = comm.allreduce(part).cpu().numpy()
    grads = [0.5 * (-part[t, 0] + part[t, 1:].sum() / kz) for t in range(3)]
    ok = bool(ws.converged.all() and us.converged.all())
    return loss, grads[0], grads[1], grads[2], ok


def dist_gpc_nlml_grad(ops, comm: Comm, targets_loc, noise_loc, probes_loc, norms_sq, tol, max_iter,
                       probe_tol=None, probe_max_iter=None, minv_classes=None):
    """Dirichlet GPC loss and (l, f, s) gradient (gpc.nlml_grad_iterative, the device path's
    kgp_gpc_nlml_grad) over row-sharded vectors: class c solves (Khat + diag(noise_c)).

    targets_loc, noise_loc: (C, n_loc); probes_loc: (C * k_z, n_loc), block c for class c;
    norms_sq: (C * k_z,) full |z|^2. The C target solves (preconditioned by
    ``minv_classes(r_head) -> z_head`` when given) and the C * k_z probe solves run as ONE
    grouped PCG: one all-gather and one fused Khat [P] on the local rows per iteration.
    Returns (loss, grad_l, grad_f, grad_s, converged), summed over classes, identical on every
    rank."""
    torch = __import__("torch")
    probe_tol = tol if probe_tol is None else probe_tol
    probe_max_iter = max_iter if probe_max_iter is None else probe_max_iter
    c = targets_loc.shape[0]
    kz = probes_loc.shape[0] // c
    if probes_loc.shape[0] != c * kz or kz < 1:
        raise ValueError(f"probes must hold k_z >= 1 rows per class ({c} classes), got {probes_loc.shape[0]}")
    v0 = torch.cat([targets_loc, probes_loc], dim=0)
    cls = np.concatenate([np.arange(c), np.repeat(np.arange(c), kz)])
    diag = noise_loc[torch.from_numpy(cls).to(noise_loc.device)]
    tols = np.array([tol] * c + [probe_tol] * (c * kz))
    caps = np.array([max_iter] * c + [probe_max_iter] * (c * kz))
    sol = dist_pcg(ops, comm, v0, tols, caps, c if minv_classes is not None else False, diag_loc=diag,
                   minv_fn=minv_classes)
    loss, grads = 0.0, np.zeros(3)
    w = sol.x[:c]
    yw = comm.allreduce((targets_loc * w).sum(dim=1)).cpu().numpy()
    v_loc = torch.cat([w, probes_loc], dim=0)
    u_loc = torch.cat([w, sol.x[c:]], dim=0)
    dl, df = _grads(ops, comm, v_loc)
    part = torch.stack([(u_loc * dl).sum(dim=1), (u_loc * df).sum(dim=1), (u_loc * v_loc).sum(dim=1)])
    part = comm.allreduce(part).cpu().numpy()
    for k in range(c):
        rows = slice(c + k * kz, c + (k + 1) * kz)
        logdet = ops.slq(sol.alphas[rows], sol.betas[rows], sol.iters[rows], norms_sq[k * kz:(k + 1) * kz])
        loss += 0.5 * (yw[k] + logdet + comm.n * LOG_2PI)
        for t in range(3):
            grads[t] += 0.5 * (-part[t, k] + part[t, rows].sum() / kz)
    return loss, grads[0], grads[1], grads[2], bool(sol.converged.all())


def dist_predict_mean(ops, comm: Comm, xs, alpha_loc):
    """Predictive mean K(X*, X) alpha (gp.py:223-236) with alpha row-sharded like the training
    points: each rank contracts the cross kernel against its own training columns
    (``ops.cross_rows``, never materialised on the device) and one all-reduce of the m-vector
    sums the shards. xs: (m, d) test points (replicated); alpha_loc: (k, n_loc)."""
    return comm.allreduce(ops.cross_rows(xs, alpha_loc))


def dist_fit(comm: Comm, y_loc, config, initial, make_ops):
    """Hyperparameter training (train.fit, train.py:176-240) over row-sharded vectors: Adam in
    softplus space on the distributed NLML gradient. Every rank evaluates the same loss and
    gradient (all-reduced scalars), so the parameter trajectory is identical on all ranks.

    y_loc: (n_loc,) this rank's targets; ``initial``: Hyperparams (train.initial_hyperparams
    on the full data, computed identically everywhere); ``make_ops(hp) -> (ops, shift)``
    builds this rank's local operator rows (and sharded preconditioner) at hp --
    ``CudaRowOps`` on the GPU. Probes are the reference's per-step seeds
    ``ProbeSet.generate(n, k_z, (rng_seed, step))``, cut to the local rows."""
    from paper_2503_02259_b200 import gp
    from paper_2503_02259_b200.train import Adam, RawParams, TrainResult, TrainStatus, chain_grads

    torch = __import__("torch")
    if config.mode != "iterative":
        raise ValueError("the distributed trainer runs the iterative estimator (mode='iterative')")
    r0, r1 = comm.ranges[comm.rank]
    raw = RawParams.from_hyperparams(initial)
    opt = Adam(config.learning_rate)
    result = TrainResult(params=raw.to_hyperparams(), raw=raw)
    warned = False
    for step in range(config.max_steps):
        hp = raw.to_hyperparams()
        ops, shift = make_ops(hp)
        probes = gp.ProbeSet.generate(comm.n, config.k_z, (config.rng_seed, step)).vectors
        z_loc = torch.from_numpy(np.ascontiguousarray(probes.T[:, r0:r1])).to(y_loc.device)
        loss, gl, gf, gs, ok = dist_nlml_grad(ops, comm, y_loc, z_loc, np.einsum("ij,ij->j", probes, probes),
                                              config.tol, config.max_iter, config.probe_tol, precondition=True,
                                              shift=shift)
        warned |= not ok
        g_rho = chain_grads(raw, [gl, gf, gs])
        gnorm = float(np.linalg.norm(g_rho))
        result.loss_history.append(loss)
        result.grad_norm_history.append(gnorm)
        if gnorm < config.grad_norm_tol:
            result.status = TrainStatus.GRAD_TOL
            break
        raw = RawParams.from_array(opt.step(raw.as_array(), g_rho))
    if warned:
        result.status = TrainStatus.SOLVER_WARNING
    result.raw = raw
    result.params = raw.to_hyperparams()
    return result


def cuda_ops_factory(kt, x, comm: Comm, precond_rank: int, precision=None):
    """make_ops for dist_fit on the GPU: a row-block engine + the replicated-build, row-sharded
    Nystrom/Woodbury factor at each step's hyperparameters."""
    from paper_2503_02259_b200.kmat import KernelEngine

    r0, r1 = comm.ranges[comm.rank]

    def make(hp):
        engine = KernelEngine(kt, x, hp, precision=precision)
        return CudaRowOps(engine, r0, r1, build_precond_factor(engine, precond_rank)), hp.s

    return make


def dist_local_variance(comm: Comm, xs, local_var_fn):
    """Local predictive variance (gp.predict_local) with the TEST points split over the ranks:
    the training points are replicated, so each rank runs the cross kNN + per-point kriging
    (``local_var_fn(xs_slice) -> (m_loc,)``; ``CudaRowOps.local_variance`` on the GPU) on its
    balanced slice of xs and one all-gather assembles the (m,) variance."""
    m = len(xs)
    ranges = [row_range(m, comm.world, r) for r in range(comm.world)]
    q0, q1 = ranges[comm.rank]
    return comm.allgather_rows(local_var_fn(np.asarray(xs)[q0:q1])[None, :], ranges)[0]


class CudaRowOps:
    """GPU local ops: this rank's rows of the fused operator and of the Woodbury factor."""

    def __init__(self, engine, r0: int, r1: int, precond_wt=None, replicated=None):
        from paper_2503_02259_b200 import _device
        from paper_2503_02259_b200._lib import call
        from paper_2503_02259_b200.kmat import KernelEngine

        self._device, self._call = _device, call
        self.r0, self.r1 = r0, r1
        # a private engine handle restricted to rows [r0, r1)
        self.engine = KernelEngine(engine.kt, engine.x, engine.params, precision=engine.precision)
        call("kgp_engine_set_rows", self.engine.handle, r0, r1 - r0)
        self.pre = None
        if replicated is not None:  # e.g. an AFNPreconditioner built on every rank
            self._rep = replicated
            self.replicated_minv = self._replicated_minv
        if precond_wt is not None:
            from paper_2503_02259_b200.precond import _LowRank

            self.pre = _LowRank(precond_wt[:, r0:r1], engine.params.s)
            self.m = precond_wt.shape[0]

    def _replicated_minv(self, r_full):
        torch = self._device.torch()
        k, n = r_full.shape
        out = torch.empty_like(r_full)
        self._call("kgp_precond_apply_inverse", self._rep.handle, k, r_full.data_ptr(), 1, n, out.data_ptr(), 1, n,
                   self._device.stream_ptr())
        return out

    def _out(self, k):
        torch = self._device.torch()
        return torch.empty((k, self.r1 - self.r0), dtype=torch.float64, device=self._device.device())

    def _matmul_peer(self, p_loc):
        """This rank's rows of Khat P from the local rows of P alone (kgp_engine_peer_publish +
        kgp_engine_peer_matmul): the other ranks' rows are read from their published tiles
        inside the operator kernel."""
        k, nloc = p_loc.shape
        p_loc = p_loc.contiguous()
        out = self._out(k)
        self._epoch = getattr(self, "_epoch", 0) + 1
        st = self._device.stream_ptr()
        self._call("kgp_engine_peer_publish", self.engine.handle, k, p_loc.data_ptr(), 1, nloc, self._epoch, st)
        self._call("kgp_engine_peer_matmul", self.engine.handle, k, self._epoch, out.data_ptr(), None, None, 1, nloc,
                   st)
        return out

    def _grads_peer(self, v_loc):
        """dKhat/dl and dKhat/df on this rank's rows from the local rows of V (fused all-gather)."""
        k, nloc = v_loc.shape
        v_loc = v_loc.contiguous()
        dl, df = self._out(k), self._out(k)
        self._epoch = getattr(self, "_epoch", 0) + 1
        st = self._device.stream_ptr()
        self._call("kgp_engine_peer_publish", self.engine.handle, k, v_loc.data_ptr(), 1, nloc, self._epoch, st)
        self._call("kgp_engine_peer_matmul", self.engine.handle, k, self._epoch, None, dl.data_ptr(), df.data_ptr(), 1,
                   nloc, st)
        return dl, df

    def matmul_rows(self, p_full):
        k, n = p_full.shape
        out = self._out(k)
        self._call("kgp_engine_matmul", self.engine.handle, k, p_full.data_ptr(), 1, n, out.data_ptr(), None, None,
                   1, out.shape[1], self._device.stream_ptr())
        return out

    def grads_rows(self, v_full):
        k, n = v_full.shape
        dl, df = self._out(k), self._out(k)
        self._call("kgp_engine_matmul", self.engine.handle, k, v_full.data_ptr(), 1, n, None, dl.data_ptr(),
                   df.data_ptr(), 1, dl.shape[1], self._device.stream_ptr())
        return dl, df

    def project(self, r_loc):
        torch = self._device.torch()
        k, nloc = r_loc.shape
        t = torch.empty((self.m, k), dtype=torch.float64, device=r_loc.device)
        self._call("kgp_lowrank_project", self.pre.h, k, r_loc.data_ptr(), 1, nloc, t.data_ptr(),
                   self._device.stream_ptr())
        return t

    def expand(self, r_loc, t, beta, alpha):
        k, nloc = r_loc.shape
        out = self._out(k)
        self._call("kgp_lowrank_expand", self.pre.h, beta, alpha, k, r_loc.data_ptr(), 1, nloc, t.contiguous().data_ptr(),
                   out.data_ptr(), 1, nloc, self._device.stream_ptr())
        return out

    def cross_rows(self, xs, alpha_loc):
        """K(xs, X[r0:r1]) alpha_loc: the cross kernel against this rank's training points, on
        an engine built over those points only (kgp_engine_cross_matmul)."""
        from paper_2503_02259_b200.kmat import KernelEngine

        torch = self._device.torch()
        if getattr(self, "_local", None) is None:
            self._local = KernelEngine(self.engine.kt, self.engine.x[self.r0:self.r1], self.engine.params,
                                       precision=self.engine.precision)
        xs_d = torch.as_tensor(np.asarray(xs, dtype=np.float64)).to(self._device.device()).contiguous()
        return self._local.cross_matmul(xs_d, alpha_loc.T.contiguous()).T.contiguous()

    def local_variance(self, xs, k_nn: int = 64):
        """f^2 - c^T Khat_NN^-1 c over the k_nn nearest training points of each test point in xs
        (kgp_knn_cross + kgp_local_variance against the replicated X)."""
        from paper_2503_02259_b200.kernels import kernel_id

        torch = self._device.torch()
        xd = self.engine.x_device()
        n, d = xd.shape
        xs_d = torch.as_tensor(np.asarray(xs, dtype=np.float64)).to(xd.device).contiguous()
        m = xs_d.shape[0]
        k_nn = int(min(k_nn, n))
        nbr = torch.empty((m, k_nn), dtype=torch.int64, device=xd.device)
        var = torch.empty(m, dtype=torch.float64, device=xd.device)
        if m:
            p = self.engine.params
            self._call("kgp_knn_cross", m, xs_d.data_ptr(), n, xd.data_ptr(), d, k_nn, nbr.data_ptr(),
                       self._device.stream_ptr())
            self._call("kgp_local_variance", kernel_id(self.engine.kt), m, d, xs_d.data_ptr(), xd.data_ptr(),
                       float(p.l), float(p.f), float(p.s), k_nn, nbr.data_ptr(), var.data_ptr(),
                       self._device.stream_ptr())
        return var

    def slq(self, alphas, betas, iters, norms_sq):
        from paper_2503_02259_b200 import solver

        torch = self._device.torch()
        dev = alphas.device
        return solver.slq_logdet_device(alphas.contiguous(), betas.contiguous(),
                                        torch.from_numpy(np.asarray(iters, dtype=np.int32)).to(dev),
                                        torch.from_numpy(np.asarray(norms_sq, dtype=np.float64)).to(dev))


class PeerTiles:
    """The fused all-gather operator's buffers for one rank (kgp_engine_set_peers): this rank's
    published tile buffer plus every peer's, mapped through CUDA IPC (the 64-byte handles are
    exchanged with all_gather_object, so any torch.distributed backend carries them).

    ``bases`` (single-process use, e.g. ranks simulated on one device): the buffers of all
    ranks, already allocated with kgp_peer_alloc; no IPC."""

    def __init__(self, engine_handle, world: int, rank: int, row_start, k: int, comm=None, bases=None):
        import ctypes

        from paper_2503_02259_b200._lib import call

        self._call = call
        self.comm = comm
        self.world, self.rank, self.k = world, rank, int(k)
        self.row_start = np.asarray(row_start, dtype=np.int64)
        self._opened, self._own = [], None
        if bases is None:
            nbytes = ctypes.c_int64()
            own_rows = int(self.row_start[rank + 1] - self.row_start[rank])
            call("kgp_engine_peer_buffer_bytes", engine_handle, self.k, own_rows, ctypes.byref(nbytes))
            ptr, handle = ctypes.c_void_p(), ctypes.create_string_buffer(64)
            call("kgp_peer_alloc", nbytes.value, ctypes.byref(ptr), handle)
            self._own = ptr.value
            handles = [None] * world
            comm.dist.all_gather_object(handles, handle.raw, group=comm.group)
            bases = []
            for q in range(world):
                if q == rank:
                    bases.append(self._own)
                    continue
                mapped = ctypes.c_void_p()
                call("kgp_peer_open", ctypes.create_string_buffer(handles[q], 64), ctypes.byref(mapped))
                self._opened.append(mapped.value)
                bases.append(mapped.value)
        self.bases = list(bases)
        arr = (ctypes.c_void_p * world)(*self.bases)
        call("kgp_engine_set_peers", engine_handle, world, rank, self.row_start.ctypes.data, arr, self.k)
        self._arr = arr
        # every rank is configured before any rank publishes: the only waits the device ever
        # does on a peer flag are then for device progress, never for a peer's host setup
        if comm is not None:
            comm.dist.barrier(group=comm.group)

    def close(self):
        """Tear down safely: this rank's kernels finish (sync), then every rank's (barrier),
        before any mapping is closed or the exported buffer freed -- a peer's operator may
        still be reading this rank's tiles over NVLink until it has passed the barrier."""
        if self._opened or self._own is not None:
            import torch

            if torch.cuda.is_available():
                torch.cuda.synchronize()
            if self.comm is not None:
                self.comm.dist.barrier(group=self.comm.group)
        for p in self._opened:
            self._call("kgp_peer_close", p)
        self._opened = []
        if self._own is not None:
            self._call("kgp_peer_free", self._own)
            self._own = None
        if self.comm is not None:  # nobody frees its buffer while a peer still maps it
            self.comm.dist.barrier(group=self.comm.group)


def enable_peer_exchange(ops, comm, k: int):
    """Switch ``ops`` (CudaRowOps) to the fused all-gather operator for RHS blocks of k
    columns: dist_pcg then calls ``ops.matmul_local(p_loc)`` instead of all_gather + product.
    ``comm`` must split rows on multiples of 32 (``Comm(n, align=32)``)."""
    starts = [r0 for r0, _ in comm.ranges] + [comm.n]
    ops.peer = PeerTiles(ops.engine.handle, comm.world, comm.rank, starts, k, comm=comm)
    ops.matmul_local = ops._matmul_peer
    ops.grads_local = ops._grads_peer
    return ops


def build_precond_factor(engine, m):
    """Replicated device build (every rank runs the same deterministic FPS + factorisation);
    returns W^T (m, n) so each rank can keep its own columns of it."""
    from paper_2503_02259_b200 import precond

    torch = __import__("torch")
    xd = engine.x_device()
    p = engine.params
    idx = precond.fps_device(xd, m, 0)
    xm = xd.index_select(0, idx)
    from paper_2503_02259_b200.kernels import device_panel

    kmm = device_panel(engine._kid, 0, xm, xm, p.l)
    kmm.diagonal().add_(precond.RIDGE_SCALE * float(torch.trace(kmm)) / m)
    low, info = torch.linalg.cholesky_ex(kmm)
    if int(info):
        raise BreakdownError("landmark factorization failed; increase the noise term s or reduce the rank m")
    vt = torch.linalg.solve_triangular(low, device_panel(engine._kid, 0, xm, xd, p.l), upper=False)
    cap = (vt @ vt.T) / p.s
    cap.diagonal().add_(1.0 / (p.f * p.f))
    lc, info = torch.linalg.cholesky_ex(cap)
    if int(info):
        raise BreakdownError("landmark factorization failed; increase the noise term s or reduce the rank m")
    return torch.linalg.solve_triangular(lc, vt, upper=False).contiguous()
