"""CPU tier: the multi-GPU host logic (partition, halo protocol, collectives) with
world_size 2 and 3 over gloo.  The per-shard arithmetic is played by the numpy
shard oracle (oracle/shard.py); what is under test is that the rows a rank
receives in its halo are the right ones, and that shard outputs concatenate to
the whole-problem oracle bit for bit."""

import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2507_13204_b200.sharded import assemble_halo, pack_boundary, partition
from conftest import assert_bits, free_port


def test_partition_covers_and_aligns():
    for n, world, align in [(10, 3, 1), (1000, 8, 1), (1 << 20, 8, 1024), (10_000_019, 4, 8192), (5, 8, 1)]:
        parts = partition(n, world, align)
        assert len(parts) == world and parts[0][0] == 0
        assert sum(length for _, length in parts) == n
        for (o0, l0), (o1, _) in zip(parts, parts[1:]):
            assert o0 + l0 == o1 and o1 % align == 0


def _whole(n, seed=1.0):
    from oracle import cport

    rng = np.random.default_rng(n)
    x, b = rng.normal(size=n), rng.normal(size=n)
    dx0, db0 = rng.normal(size=n), rng.normal(size=n)
    xo, dxo, dbo = x.copy(), dx0.copy(), db0.copy()
    cport.laplacian_grad(xo, b.copy(), dxo, dbo, seed)
    return x, b, dx0, db0, xo, dxo, dbo


@pytest.mark.parametrize("world", [1, 2, 3, 5])
def test_halo_protocol_single_process(world):
    """all ranks simulated in one process: pack -> (all_gather) -> assemble -> shard kernel"""
    from oracle import shard as shard_oracle

    n = 101
    x, b, dx0, db0, xo, dxo, dbo = _whole(n)
    parts = partition(n, world)
    packed = torch.stack([pack_boundary(torch.from_numpy(x[o:o + l]), torch.from_numpy(b[o:o + l])) for o, l in parts])
    got_x, got_dx, got_db = [], [], []
    for r, (o, l) in enumerate(parts):
        halo = assemble_halo(packed, r, world).numpy()
        dx, db = dx0[o:o + l].copy(), db0[o:o + l].copy()
        xs, _ = shard_oracle.laplacian_shard(x[o:o + l], b[o:o + l], dx, db, halo, o, n)
        got_x.append(xs), got_dx.append(dx), got_db.append(db)
    assert_bits(np.concatenate(got_x), xo, "3x")
    assert_bits(np.concatenate(got_dx), dxo, "_d_x")
    assert_bits(np.concatenate(got_db), dbo, "_d_b")


def _worker(rank, world, port, n, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import shard as shard_oracle

        x, b, dx0, db0, *_ = _whole(n)
        o, l = partition(n, world)[rank]
        xt, bt = torch.from_numpy(x[o:o + l].copy()), torch.from_numpy(b[o:o + l].copy())
        mine = pack_boundary(xt, bt)
        gathered = torch.empty(world * 6, dtype=torch.float64)
        dist.all_gather_into_tensor(gathered, mine)
        halo = assemble_halo(gathered.view(world, 6), rank, world).numpy()
        dx, db = dx0[o:o + l].copy(), db0[o:o + l].copy()
        xs, y2 = shard_oracle.laplacian_shard(x[o:o + l], b[o:o + l], dx, db, halo, o, n)
        f = torch.tensor([float(np.sum(y2))], dtype=torch.float64)
        dist.all_reduce(f)  # the scalar objective: the only data-path collective besides the halo
        pieces = [None] * world
        dist.all_gather_object(pieces, (xs, dx, db))
        if rank == 0:
            out.put((float(f.item()), pieces))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_halo_exchange_over_gloo(world):
    from oracle import cport

    n = 257
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, out)) for r in range(world)]
    for p in procs:
        p.start()
    f, pieces = out.get(timeout=60)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    x, b, dx0, db0, xo, dxo, dbo = _whole(n)
    assert_bits(np.concatenate([p[0] for p in pieces]), xo, "3x")
    assert_bits(np.concatenate([p[1] for p in pieces]), dxo, "_d_x")
    assert_bits(np.concatenate([p[2] for p in pieces]), dbo, "_d_b")
    fo = cport.laplacian_primal(x.copy(), b.copy())
    assert abs(f - fo) <= 1e-14 * abs(fo)  # allreduce order differs from the tree: reassociation only


def _exact_worker(rank, world, port, n, span, out):
    """the exact-objective protocol of ShardedLaplacian.primal over gloo: pad the block partials to
    the widest rank, all_gather, cut the padding off, fold with the reference's tree"""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import interp, shard as shard_oracle
        from paper_2507_13204_b200.sharded import combine_partials, partial_count

        x, b, dx0, db0, *_ = _whole(n)
        parts = partition(n, world, span)
        o, l = parts[rank]
        xt, bt = torch.from_numpy(x[o:o + l].copy()), torch.from_numpy(b[o:o + l].copy())
        gathered = torch.empty(world * 6, dtype=torch.float64)
        dist.all_gather_into_tensor(gathered, pack_boundary(xt, bt))
        halo = assemble_halo(gathered.view(world, 6), rank, world).numpy()
        _, y2 = shard_oracle.laplacian_shard(x[o:o + l], b[o:o + l], dx0[o:o + l].copy(), db0[o:o + l].copy(), halo, o, n)
        counts = [partial_count(length, span) for _, length in parts]
        width = max(counts)
        mine = torch.zeros(width, dtype=torch.float64)
        mine[:counts[rank]] = torch.from_numpy(shard_oracle.block_partials(y2, o, n, span))
        allp = torch.empty(world * width, dtype=torch.float64)
        dist.all_gather_into_tensor(allp, mine)
        nodes = combine_partials(allp.view(world, width), counts).numpy()
        out.put((rank, float(interp.pairwise_sum(nodes))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,span", [(2, 257, 16), (3, 1000, 64), (3, 96, 16)])
def test_exact_objective_over_gloo(world, n, span):
    """every rank ends up with the SAME bits, equal to the whole-problem oracle"""
    from oracle import cport

    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_exact_worker, args=(r, world, port, n, span, out)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(out.get(timeout=60) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    x, b, *_ = _whole(n)
    fo = cport.laplacian_primal(x.copy(), b.copy())
    for r in range(world):
        assert_bits(got[r], fo, f"rank {r} of {world}")


def test_block_partials_fold_to_the_reference_tree():
    from oracle import interp, shard as shard_oracle

    rng = np.random.default_rng(0)
    for n, span, world in [(1, 4, 1), (100, 8, 3), (257, 16, 2), (1000, 64, 5), (64, 16, 4)]:
        v = rng.normal(size=n)
        parts = partition(n, world, span)
        nodes = np.concatenate([shard_oracle.block_partials(v[o:o + l], o, n, span) for o, l in parts if l])
        assert_bits(interp.pairwise_sum(nodes), interp.pairwise_sum(v), f"n={n} span={span} world={world}")
