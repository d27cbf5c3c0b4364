"""GPU tier, sharded mode with PEER MEMORY: two / three processes on one device (CUDA IPC works
between processes on the same GPU exactly as across NVLink), gloo only for the one-time exchange
of the IPC handles.  The gradient step must be ONE launch and NO collective, and every rank's rows
bit-identical to the whole-problem C oracle; the objective bit-identical on every rank.  Also: the
NCCL backend's code path with a group of one rank (all that one GPU allows: NCCL refuses two ranks
on a device)."""

import os

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from conftest import assert_bits, free_port

pytestmark = pytest.mark.gpu


def _collect(procs, out, timeout=300):
    """first item of the queue, failing early when a worker dies"""
    import queue
    import time

    t0 = time.time()
    while True:
        try:
            return out.get(timeout=2)
        except queue.Empty:
            if any(p.exitcode not in (None, 0) for p in procs):
                raise AssertionError("a worker process failed (see its traceback above)")
            if time.time() - t0 > timeout:
                raise


def _whole(n):
    from oracle import cport

    rng = np.random.default_rng(n)
    x, b = rng.normal(size=n), rng.normal(size=n)
    dx0, db0 = rng.normal(size=n), rng.normal(size=n)
    xo, dxo, dbo = x.copy(), dx0.copy(), db0.copy()
    f = cport.laplacian_primal(x.copy(), b.copy())
    cport.laplacian_grad(xo, b.copy(), dxo, dbo, 1.0)
    return x, b, dx0, db0, xo, dxo, dbo, f


def _peer_worker(rank, world, port, n, own_stream, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    import paper_2507_13204_b200 as krn
    from paper_2507_13204_b200.sharded import ShardedLaplacian

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        if own_stream:
            dev = krn.Device(0)  # the library's private stream: the class must order it against torch's
        else:
            s = torch.cuda.Stream()
            torch.cuda.set_stream(s)
            dev = krn.Device(0, s.cuda_stream)
        x, b, dx0, db0, *_ = _whole(n)
        sh = ShardedLaplacian(n, dev)
        o, l = sh.offset, sh.n_local
        xt, bt = torch.from_numpy(x[o:o + l].copy()).cuda(), torch.from_numpy(b[o:o + l].copy()).cuda()
        dxt, dbt = torch.from_numpy(dx0[o:o + l].copy()).cuda(), torch.from_numpy(db0[o:o + l].copy()).cuda()
        xo, f = torch.empty_like(xt), torch.zeros(1, dtype=torch.float64, device="cuda")
        sh.attach(xt, bt)
        calls = {"n": 0}
        for name in ("all_gather_into_tensor", "all_reduce", "all_gather", "broadcast", "barrier"):
            real = getattr(dist, name)

            def counted(*a, _real=real, **k):
                calls["n"] += 1
                return _real(*a, **k)

            setattr(dist, name, counted)
        l0 = dev.launches()
        sh.grad(xt, xo, bt, dxt, dbt)
        grad_launches, grad_collectives = dev.launches() - l0, calls["n"]
        sh.primal(xt, xo, bt, f)
        primal_collectives = calls["n"] - grad_collectives
        torch.cuda.synchronize()
        dev.sync()
        piece = (xo.cpu().numpy(), dxt.cpu().numpy(), dbt.cpu().numpy(), float(f.item()), grad_launches,
                 grad_collectives, primal_collectives)
        # second step on the same attachment after the inputs changed everywhere: fence, then step
        xt.mul_(0.5)
        sh.fence()
        dx2 = torch.zeros_like(xt)
        db2 = torch.zeros_like(xt)
        sh.grad(xt, xo, bt, dx2, db2, dx_zero=True, db_zero=True)
        torch.cuda.synchronize()
        dev.sync()
        piece += (dx2.cpu().numpy(), db2.cpu().numpy())
        sh.fence()
        sh.detach()
        pieces = [None] * world
        dist.all_gather_object(pieces, piece)
        if rank == 0:
            out.put(pieces)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,own_stream", [(2, 2500, False), (2, 100_003, True), (3, 3 * 8192 + 77, False)])
def test_peer_halo_two_processes_one_device(world, n, own_stream):
    from oracle import cport

    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_peer_worker, args=(r, world, port, n, own_stream, out)) for r in range(world)]
    for p in procs:
        p.start()
    pieces = _collect(procs, out)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    x, b, dx0, db0, xo, dxo, dbo, f = _whole(n)
    assert_bits(np.concatenate([p[0] for p in pieces]), xo, "3x")
    assert_bits(np.concatenate([p[1] for p in pieces]), dxo, "_d_x")
    assert_bits(np.concatenate([p[2] for p in pieces]), dbo, "_d_b")
    for r, p in enumerate(pieces):
        assert_bits(p[3], f, f"objective on rank {r}")  # tree-aligned partials: the reference's bits on every rank
        assert p[4] == 1, f"gradient step on rank {r}: {p[4]} launches"
        assert p[5] == 0, f"gradient step on rank {r}: {p[5]} collectives"
        assert p[6] == 1, f"primal step on rank {r}: {p[6]} collectives (the partials' all_gather)"
    x2 = 0.5 * x
    dx2, db2 = np.zeros(n), np.zeros(n)
    cport.laplacian_grad(x2, b.copy(), dx2, db2, 1.0)
    assert_bits(np.concatenate([p[7] for p in pieces]), dx2, "_d_x after the inputs changed")
    assert_bits(np.concatenate([p[8] for p in pieces]), db2, "_d_b after the inputs changed")


def _fallback_worker(rank, world, port, n, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import ctypes as C

    import torch.distributed as dist

    import paper_2507_13204_b200 as krn
    from paper_2507_13204_b200 import _cabi
    from paper_2507_13204_b200.sharded import ShardedLaplacian

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        s = torch.cuda.Stream()
        torch.cuda.set_stream(s)
        dev = krn.Device(0, s.cuda_stream)
        x, b, dx0, db0, *_ = _whole(n)
        sh = ShardedLaplacian(n, dev)
        o, l = sh.offset, sh.n_local
        xt, bt = torch.from_numpy(x[o:o + l].copy()).cuda(), torch.from_numpy(b[o:o + l].copy()).cuda()
        dxt, dbt = torch.from_numpy(dx0[o:o + l].copy()).cuda(), torch.from_numpy(db0[o:o + l].copy()).cuda()
        xo = torch.empty_like(xt)
        if rank == 1:  # this rank cannot import its neighbours' handles (no peer access, say)
            garbage = (C.c_ubyte * 64)()
            real = dev.lib.krn_ipc_open

            def refuse(h, handle, flags, base, ptr):
                return real(h, garbage, flags, base, ptr)

            class Lib:  # the library with one entry point replaced
                def __getattr__(self, name, _lib=dev.lib):
                    return refuse if name == "krn_ipc_open" else getattr(_lib, name)

            dev.lib = Lib()
        sh.attach(xt, bt)
        failure = sh.attach_failure
        assert failure is not None and not sh._attached(xt, bt)
        sh.grad(xt, xo, bt, dxt, dbt)
        torch.cuda.synchronize()
        dev.sync()
        pieces = [None] * world
        dist.all_gather_object(pieces, (xo.cpu().numpy(), dxt.cpu().numpy(), dbt.cpu().numpy(), failure))
        if rank == 0:
            out.put(pieces)
    finally:
        dist.destroy_process_group()


def test_a_rank_that_cannot_map_its_neighbours_takes_everybody_to_the_collective_path():
    world, n = 2, 40_001
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_fallback_worker, args=(r, world, port, n, out)) for r in range(world)]
    for p in procs:
        p.start()
    pieces = _collect(procs, out)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    x, b, dx0, db0, xo, dxo, dbo, f = _whole(n)
    assert_bits(np.concatenate([p[0] for p in pieces]), xo, "3x")
    assert_bits(np.concatenate([p[1] for p in pieces]), dxo, "_d_x")
    assert_bits(np.concatenate([p[2] for p in pieces]), dbo, "_d_b")
    assert "neighbour" in pieces[0][3] and pieces[1][3]  # rank 0 mapped fine but follows rank 1


def _nccl_worker(port, n, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    import paper_2507_13204_b200 as krn
    from paper_2507_13204_b200.sharded import ShardedLaplacian

    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        s = torch.cuda.Stream()
        torch.cuda.set_stream(s)
        dev = krn.Device(0, s.cuda_stream)
        x, b, dx0, db0, *_ = _whole(n)
        sh = ShardedLaplacian(n, dev, shortcut_single=False)  # keep the collectives in: NCCL all_gather x 2
        xt, bt = torch.from_numpy(x).cuda(), torch.from_numpy(b).cuda()
        dxt, dbt = torch.from_numpy(dx0.copy()).cuda(), torch.from_numpy(db0.copy()).cuda()
        xo, f = torch.empty_like(xt), torch.zeros(1, dtype=torch.float64, device="cuda")
        sh.primal(xt, xo, bt, f)
        sh.grad(xt, xo, bt, dxt, dbt)
        sh.attach(xt, bt)  # a group of one has no neighbour to map
        torch.cuda.synchronize()
        out.put((xo.cpu().numpy(), dxt.cpu().numpy(), dbt.cpu().numpy(), float(f.item())))
    finally:
        dist.destroy_process_group()


def test_nccl_backend_with_a_group_of_one():
    n = 300_001
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    p = ctx.Process(target=_nccl_worker, args=(free_port(), n, out))
    p.start()
    xo_g, dx_g, db_g, f_g = _collect([p], out)
    p.join(timeout=120)
    assert p.exitcode == 0
    x, b, dx0, db0, xo, dxo, dbo, f = _whole(n)
    assert_bits(xo_g, xo, "3x")
    assert_bits(dx_g, dxo, "_d_x")
    assert_bits(db_g, dbo, "_d_b")
    assert_bits(f_g, f, "objective")


def test_short_shards_are_refused_before_any_collective():
    import paper_2507_13204_b200 as krn
    from paper_2507_13204_b200.sharded import ShardedLaplacian, partition

    class FakeDist:  # a group of 4 without a process group: only rank / size are asked for
        @staticmethod
        def is_initialized():
            return True

        @staticmethod
        def get_rank(group=None):
            return 0

        @staticmethod
        def get_world_size(group=None):
            return 4

    import torch.distributed as dist

    dev = krn.Device.get()
    real = (dist.is_initialized, dist.get_rank, dist.get_world_size)
    dist.is_initialized, dist.get_rank, dist.get_world_size = FakeDist.is_initialized, FakeDist.get_rank, FakeDist.get_world_size
    try:
        assert any(l < 2 for _, l in partition(1500, 4, 1024))
        with pytest.raises(ValueError, match="fewer than 2 rows"):
            ShardedLaplacian(1500, dev)
    finally:
        dist.is_initialized, dist.get_rank, dist.get_world_size = real
