"""World-size-2 gloo test of the row-partitioned solver logic on the CPU.

Each rank owns a contiguous row block; the local operator rows, Woodbury halves and SLQ
come from the CPU oracle (the GPU implementation is dist.CudaRowOps). The distributed
PCG and NLML+gradient must reproduce the single-process oracle on the same inputs.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp
from scipy.linalg import cho_solve

from oracle import kgp_oracle as orc
from paper_2503_02259_b200 import dist as kdist

KT, L, F, S = "matern52", 0.7, 1.2, 0.05


def _problem(n=240, seed=8):
    rng = np.random.default_rng(seed)
    x = rng.uniform(-1, 1, (n, 2))
    y = np.sin(3 * x[:, 0]) + 0.1 * rng.standard_normal(n)
    z = rng.standard_normal((n, 5))
    return x, y, z


class OracleRowOps:
    def __init__(self, x, r0, r1, ny, hp=(L, F, S)):
        self.x, self.r0, self.r1, self.ny = x, r0, r1, ny
        self.rows = np.arange(r0, r1)
        self.l, self.f, self.s = hp

    def matmul_rows(self, p_full):
        out = orc.khat_matmul(KT, self.x, self.l, self.f, self.s, p_full.numpy().T, rows=self.rows)
        return torch.from_numpy(np.ascontiguousarray(out.T))

    def grads_rows(self, v_full):
        b = v_full.numpy().T
        dl = orc.khat_matmul(KT, self.x, self.l, self.f, self.s, b, theta="l", rows=self.rows)
        df = orc.khat_matmul(KT, self.x, self.l, self.f, self.s, b, theta="f", rows=self.rows)
        return torch.from_numpy(np.ascontiguousarray(dl.T)), torch.from_numpy(np.ascontiguousarray(df.T))

    def project(self, r_loc):
        return torch.from_numpy(self.ny.v[self.r0:self.r1].T @ r_loc.numpy().T)

    def expand(self, r_loc, t, beta, alpha):
        y = cho_solve(self.ny.cap, t.numpy())
        out = beta * r_loc.numpy().T + alpha * (self.ny.v[self.r0:self.r1] @ y)
        return torch.from_numpy(np.ascontiguousarray(out.T))

    def cross_rows(self, xs, alpha_loc):
        kx = self.f * self.f * orc.eval_kernel(KT, np.asarray(xs), self.x[self.r0:self.r1], self.l)
        return torch.from_numpy(np.ascontiguousarray((kx @ alpha_loc.numpy().T).T))

    def slq(self, alphas, betas, iters, norms_sq):
        a = [alphas[j, :it].numpy() for j, it in enumerate(iters)]
        b = [betas[j, :it].numpy() for j, it in enumerate(iters)]
        return orc.slq_logdet(a, b, norms_sq)


def _worker(rank, world, port, errfile):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        x, y, z = _problem()
        n = len(y)
        ny = orc.Nystrom(KT, x, L, F, S, 30)
        comm = kdist.Comm(n)
        r0, r1 = kdist.row_range(n, world, rank)
        ops = OracleRowOps(x, r0, r1, ny)

        def op(b):
            return orc.khat_matmul(KT, x, L, F, S, b)

        # batched PCG, preconditioned and not, against the single-process oracle
        for pre, tol in ((True, 1e-10), (False, 1e-8)):
            res = kdist.dist_pcg(ops, comm, torch.from_numpy(np.ascontiguousarray(z.T[:, r0:r1])), tol, 500,
                                 pre, shift=S)
            sol, al, be, rel, conv = orc.pcg(op, ny.apply_inverse if pre else None, z, tol, 500)
            full = comm.allgather_rows(res.x).numpy().T
            assert np.max(np.abs(full - sol)) <= 1e-6 * np.max(np.abs(sol)), "solution"
            assert np.all(np.abs(res.iters - np.array([len(a) for a in al])) <= 3), (res.iters, [len(a) for a in al])
            for j in range(z.shape[1]):
                m = min(6, len(al[j]))
                np.testing.assert_allclose(res.alphas[j, :m].numpy(), al[j][:m], rtol=1e-9)
            assert list(res.converged) == list(conv)
        # NLML + gradient in tolerance mode
        got = kdist.dist_nlml_grad(ops, comm, torch.from_numpy(y[r0:r1].copy()),
                                   torch.from_numpy(np.ascontiguousarray(z.T[:, r0:r1])),
                                   np.einsum("ij,ij->j", z, z), 1e-10, 3000, precondition=True, shift=S)
        ref = orc.nlml_grad(KT, x, y, L, F, S, z, ny, tol=1e-10, max_iter=3000)
        assert np.all(np.abs(np.array(got[:4]) - np.array(ref[:4])) <= 1e-8 * np.abs(np.array(ref[:4]))), (got, ref)
        dist.barrier()
        dist.destroy_process_group()
    except Exception as exc:  # surface the failure to the parent
        with open(errfile, "a") as fh:
            fh.write(f"rank {rank}: {type(exc).__name__}: {exc}\n")
        raise


class ReplicatedAfnOps(OracleRowOps):
    """Local operator rows from the oracle, M^-1 replicated: the numpy AFN on full vectors."""

    def __init__(self, x, r0, r1, afn):
        super().__init__(x, r0, r1, None)
        self.afn = afn

    def replicated_minv(self, r_full):
        return torch.from_numpy(np.ascontiguousarray(self.afn.apply_inverse(r_full.numpy().T).T))


def _afn_worker(rank, world, port, errfile):
    try:
        import afn_ref

        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        x, y, z = _problem()
        n = len(y)
        afn = afn_ref.AFN(KT, x, L, F, S, 24, 6)
        comm = kdist.Comm(n)
        r0, r1 = kdist.row_range(n, world, rank)
        ops = ReplicatedAfnOps(x, r0, r1, afn)
        res = kdist.dist_pcg(ops, comm, torch.from_numpy(np.ascontiguousarray(z.T[:, r0:r1])), 1e-10, 500, True)
        sol, al, be, rel, conv = orc.pcg(lambda b: orc.khat_matmul(KT, x, L, F, S, b), afn.apply_inverse, z, 1e-10,
                                         500)
        full = comm.allgather_rows(res.x).numpy().T
        assert np.max(np.abs(full - sol)) <= 1e-6 * np.max(np.abs(sol)), "solution"
        assert np.all(np.abs(res.iters - np.array([len(a) for a in al])) <= 2), (res.iters, [len(a) for a in al])
        assert all(res.converged)
        dist.barrier()
        dist.destroy_process_group()
    except Exception as exc:
        with open(errfile, "a") as fh:
            fh.write(f"rank {rank}: {type(exc).__name__}: {exc}\n")
        raise


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2])
def test_row_partitioned_pcg_and_nlml_gloo(tmp_path, world):
    errfile = str(tmp_path / "err.txt")
    mp.spawn(_worker, args=(world, _free_port(), errfile), nprocs=world, join=True)
    assert not os.path.exists(errfile), open(errfile).read()


def test_row_ranges_cover_and_balance():
    for n, w in ((10, 3), (65536, 8), (7, 8)):
        rs = [kdist.row_range(n, w, r) for r in range(w)]
        assert rs[0][0] == 0 and rs[-1][1] == n
        assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
        sizes = [b - a for a, b in rs]
        assert max(sizes) - min(sizes) <= 1


def test_row_partitioned_pcg_replicated_afn_gloo(tmp_path):
    """AFN (not row-shardable) replicated on every rank: gather r, apply, keep own rows."""
    errfile = str(tmp_path / "err.txt")
    mp.spawn(_afn_worker, args=(2, _free_port(), errfile), nprocs=2, join=True)
    assert not os.path.exists(errfile), open(errfile).read()


def _gpc_worker(rank, world, port, errfile):
    """Dirichlet GPC loss/gradient and the predictive mean over row-sharded vectors."""
    try:
        import gpc_ref

        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        x, y, z = _problem()
        n, c, kz = len(y), 3, 4
        labels = np.argmax(np.stack([np.sin(2 * x[:, 0]), np.cos(3 * x[:, 1]), x[:, 0] * x[:, 1]]), axis=0)
        targets, noise = gpc_ref.transform(labels, c)
        probes = np.random.default_rng(3).standard_normal((c * kz, n))
        comm = kdist.Comm(n)
        r0, r1 = kdist.row_range(n, world, rank)
        ops = OracleRowOps(x, r0, r1, None)
        t_loc = torch.from_numpy(np.ascontiguousarray(targets[:, r0:r1]))
        d_loc = torch.from_numpy(np.ascontiguousarray(noise[:, r0:r1]))
        z_loc = torch.from_numpy(np.ascontiguousarray(probes[:, r0:r1]))
        loss, g = gpc_ref.estimator(KT, x, targets, noise, L, F, S, probes)
        ref = np.array([loss, *g])
        # a row-local (Jacobi) preconditioner per class exercises the minv_fn path
        kdiag = F * F + S
        jac = lambda head: head / (kdiag + d_loc)  # noqa: E731
        for minv in (None, jac):
            got = kdist.dist_gpc_nlml_grad(ops, comm, t_loc, d_loc, z_loc, np.einsum("ij,ij->i", probes, probes),
                                           1e-11, 3000, minv_classes=minv)
            assert got[4], "converged"
            assert np.all(np.abs(np.array(got[:4]) - ref) <= 1e-6 * np.abs(ref)), (got, ref)
        # predictive mean: alpha sharded like the training rows
        xs = np.random.default_rng(4).uniform(-1, 1, (17, 2))
        alpha = np.random.default_rng(5).standard_normal((2, n))
        mean = kdist.dist_predict_mean(ops, comm, xs, torch.from_numpy(np.ascontiguousarray(alpha[:, r0:r1])))
        want = F * F * orc.eval_kernel(KT, xs, x, L) @ alpha.T
        assert np.max(np.abs(mean.numpy().T - want)) <= 1e-12 * np.max(np.abs(want))
        # local variance with the test points split over the ranks (k_nn = n: the exact variance)
        kh = orc.khat_dense(KT, x, L, F, S)

        def exact_var(xq):
            cq = F * F * orc.eval_kernel(KT, xq, x, L)
            return torch.from_numpy(F * F - np.einsum("ij,ji->i", cq, np.linalg.solve(kh, cq.T)))

        var = kdist.dist_local_variance(comm, xs, exact_var)
        np.testing.assert_allclose(var.numpy(), exact_var(xs).numpy(), rtol=1e-12)
        dist.barrier()
        dist.destroy_process_group()
    except Exception as exc:
        with open(errfile, "a") as fh:
            fh.write(f"rank {rank}: {type(exc).__name__}: {exc}\n")
        raise


@pytest.mark.parametrize("world", [2, 3])
def test_row_partitioned_gpc_and_predict_gloo(tmp_path, world):
    errfile = str(tmp_path / "err.txt")
    mp.spawn(_gpc_worker, args=(world, _free_port(), errfile), nprocs=world, join=True)
    assert not os.path.exists(errfile), open(errfile).read()


def _fit_worker(rank, world, port, errfile):
    """dist_fit: the distributed Adam trajectory equals a single-process loop over the oracle."""
    try:
        from paper_2503_02259_b200 import gp
        from paper_2503_02259_b200.kmat import Hyperparams
        from paper_2503_02259_b200.train import Adam, RawParams, TrainConfig, chain_grads

        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        x, y, _ = _problem(n=160)
        n, m = len(y), 20
        cfg = TrainConfig(learning_rate=0.05, max_steps=3, mode="iterative", k_z=4, tol=1e-10, probe_tol=1e-10,
                          max_iter=2000, rng_seed=2)
        hp0 = Hyperparams(0.6, 1.0, 0.05)
        comm = kdist.Comm(n)
        r0, r1 = kdist.row_range(n, world, rank)

        def make_ops(hp):
            ny = orc.Nystrom(KT, x, hp.l, hp.f, hp.s, m)
            return OracleRowOps(x, r0, r1, ny, (hp.l, hp.f, hp.s)), hp.s

        res = kdist.dist_fit(comm, torch.from_numpy(y[r0:r1].copy()), cfg, hp0, make_ops)
        raw, opt, hist = RawParams.from_hyperparams(hp0), Adam(cfg.learning_rate), []
        for step in range(cfg.max_steps):
            hp = raw.to_hyperparams()
            z = gp.ProbeSet.generate(n, cfg.k_z, (cfg.rng_seed, step)).vectors
            ref = orc.nlml_grad(KT, x, y, hp.l, hp.f, hp.s, z, orc.Nystrom(KT, x, hp.l, hp.f, hp.s, m), tol=1e-10,
                                max_iter=2000)
            hist.append(ref[0])
            raw = RawParams.from_array(opt.step(raw.as_array(), chain_grads(raw, ref[1:4])))
        np.testing.assert_allclose(res.loss_history, hist, rtol=1e-8)
        np.testing.assert_allclose(res.raw.as_array(), raw.as_array(), rtol=1e-6)
        dist.barrier()
        dist.destroy_process_group()
    except Exception as exc:
        with open(errfile, "a") as fh:
            fh.write(f"rank {rank}: {type(exc).__name__}: {exc}\n")
        raise


def test_row_partitioned_fit_gloo(tmp_path):
    errfile = str(tmp_path / "err.txt")
    mp.spawn(_fit_worker, args=(2, _free_port(), errfile), nprocs=2, join=True)
    assert not os.path.exists(errfile), open(errfile).read()


class PeerExchangeOps(OracleRowOps):
    """dist_pcg's fused all-gather branch (``matmul_local``): the operator gets only the local
    rows of P. The device path reads the peers' published tiles inside its kernel
    (kgp_engine_peer_matmul); here the peers' rows arrive through a gloo all_gather."""

    def __init__(self, x, r0, r1, ny, comm):
        super().__init__(x, r0, r1, ny)
        self.comm = comm
        self.local_calls = 0

    def matmul_local(self, p_loc):
        self.local_calls += 1
        # stand-in for the peers' published tiles (the base-class gather is not counted)
        return self.matmul_rows(kdist.Comm.allgather_rows(self.comm, p_loc))

    def grads_local(self, v_loc):
        self.local_calls += 1
        return self.grads_rows(kdist.Comm.allgather_rows(self.comm, v_loc))


class CountingComm(kdist.Comm):
    def __init__(self, *a, **kw):
        super().__init__(*a, **kw)
        self.gathers = 0

    def allgather_rows(self, x_loc, ranges=None):
        self.gathers += 1
        return super().allgather_rows(x_loc, ranges)


def _peer_worker(rank, world, port, errfile):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        x, y, z = _problem()
        n = len(y)
        ny = orc.Nystrom(KT, x, L, F, S, 30)
        comm = CountingComm(n, align=32)  # the fused operator's row blocks: 32-row boundaries
        r0, r1 = comm.ranges[rank]
        assert r0 % 32 == 0
        ops = PeerExchangeOps(x, r0, r1, ny, comm)
        res = kdist.dist_pcg(ops, comm, torch.from_numpy(np.ascontiguousarray(z.T[:, r0:r1])), 1e-10, 500, True,
                             shift=S)
        sol, al, be, rel, conv = orc.pcg(lambda b: orc.khat_matmul(KT, x, L, F, S, b), ny.apply_inverse, z, 1e-10,
                                         500)
        # no separate operator all-gather; one operator call per iteration, plus at most the
        # look-ahead of dist_pcg's device-resident loop (host checks every 8 iterations)
        assert comm.gathers == 0 and int(res.iters.max()) <= ops.local_calls <= int(res.iters.max()) + 8
        full = comm.allgather_rows(res.x).numpy().T
        assert np.max(np.abs(full - sol)) <= 1e-6 * np.max(np.abs(sol)), "solution"
        assert list(res.converged) == list(conv)
        # NLML + gradient: the solves and the derivative products all go through the fused path
        g0 = comm.gathers
        got = kdist.dist_nlml_grad(ops, comm, torch.from_numpy(y[r0:r1].copy()),
                                   torch.from_numpy(np.ascontiguousarray(z.T[:, r0:r1])),
                                   np.einsum("ij,ij->j", z, z), 1e-10, 3000, precondition=True, shift=S)
        ref = orc.nlml_grad(KT, x, y, L, F, S, z, ny, tol=1e-10, max_iter=3000)
        assert np.all(np.abs(np.array(got[:4]) - np.array(ref[:4])) <= 1e-8 * np.abs(np.array(ref[:4]))), (got, ref)
        assert comm.gathers == g0  # no operator all-gather anywhere in the evaluation
        dist.barrier()
        dist.destroy_process_group()
    except Exception as exc:
        with open(errfile, "a") as fh:
            fh.write(f"rank {rank}: {type(exc).__name__}: {exc}\n")
        raise


@pytest.mark.parametrize("world", [2, 3])
def test_row_partitioned_pcg_fused_exchange_gloo(tmp_path, world):
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    errfile = str(tmp_path / "err.txt")
    mp.spawn(_peer_worker, args=(world, port, errfile), nprocs=world, join=True)
    assert not os.path.exists(errfile), open(errfile).read()
