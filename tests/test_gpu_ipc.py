"""The fused all-gather operator across two real processes (kgp_peer_open had never
run between processes). Two ranks, one process each, both on cuda:0 (the box has one GPU):
each allocates its tile buffer, the 64-byte CUDA IPC handles travel by all_gather_object over
gloo, each maps the other's buffer with kgp_peer_open (dist.PeerTiles), and per epoch each
rank publishes its rows of B (kgp_engine_peer_publish) and multiplies with
kgp_engine_peer_matmul, whose producer warp bulk-copies the other rank's tiles out of the
mapped buffer. Every epoch is bracketed by synchronize + barrier, so no kernel ever waits on
a launch that has not run (the ready / done flags are already set when a kernel reads them).
Checked bitwise against each rank's ordinary row-block product of the same B."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _worker(rank, world, port, errfile, n, k):
    try:
        import torch
        import torch.distributed as dist

        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        import paper_2503_02259_b200 as kgp
        from paper_2503_02259_b200 import _lib
        from paper_2503_02259_b200 import dist as kdist

        x = np.random.default_rng(3).standard_normal((n, 8))
        e = kgp.KernelEngine(kgp.KernelType.GAUSSIAN, x, kgp.Hyperparams(1.2, 1.1, 0.05), precision="fast")
        comm = kdist.Comm(n, align=32)
        r0, r1 = comm.ranges[rank]
        nl = r1 - r0
        _lib.call("kgp_engine_set_rows", e.handle, r0, nl)
        starts = [a for a, _ in comm.ranges] + [n]
        tiles = kdist.PeerTiles(e.handle, world, rank, starts, k, comm=comm)  # IPC handles + kgp_peer_open
        assert len(tiles._opened) == world - 1
        st = torch.cuda.current_stream().cuda_stream
        for epoch in (1, 2, 3):
            b = torch.from_numpy(np.random.default_rng(100 + epoch).standard_normal((k, n))).cuda()  # same B on all ranks
            loc = b[:, r0:r1].contiguous()
            _lib.call("kgp_engine_peer_publish", e.handle, k, loc.data_ptr(), 1, nl, epoch, st)
            torch.cuda.synchronize()
            dist.barrier()  # every rank's tiles of this epoch are written
            got = torch.empty((k, nl), dtype=torch.float64, device="cuda")
            gl = torch.empty_like(got)
            _lib.call("kgp_engine_peer_matmul", e.handle, k, epoch, got.data_ptr(), gl.data_ptr(), None, 1, nl, st)
            ref = torch.empty_like(got)
            rl = torch.empty_like(got)
            _lib.call("kgp_engine_matmul", e.handle, k, b.data_ptr(), 1, n, ref.data_ptr(), rl.data_ptr(), None, 1,
                      nl, st)
            torch.cuda.synchronize()
            assert torch.equal(got, ref), (rank, epoch, float((got - ref).abs().max()))
            assert torch.equal(gl, rl), (rank, epoch)
            dist.barrier()  # every rank has read this epoch's tiles before anyone republishes
        tiles.close()
        e.close()
        dist.destroy_process_group()
    except Exception as exc:
        with open(errfile, "a") as fh:
            fh.write(f"rank {rank}: {type(exc).__name__}: {exc}\n")
        raise


@pytest.mark.parametrize("n,k", [(4096, 16), (3000, 32)])
def test_fused_allgather_two_processes(tmp_path, n, k):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    errfile = str(tmp_path / "err.txt")
    mp.spawn(_worker, args=(2, port, errfile, n, k), nprocs=2, join=True)
    assert not os.path.exists(errfile), open(errfile).read()
