"""GPU tier, sharded mode on ONE device: the shard interface of the fused kernels
(offset / n_global / halo rows) driven through sharded.partition, pack_boundary and
assemble_halo exactly as the ranks of a multi-GPU run would, one shard after the
other, against the whole-problem C oracle.  (NCCL refuses two ranks on one GPU, so
the collectives themselves are covered over gloo in tests/test_sharded_cpu.py.)"""

import ctypes as C

import numpy as np
import pytest
import torch

import paper_2507_13204_b200 as krn
from paper_2507_13204_b200 import _cabi
from paper_2507_13204_b200.sharded import ShardedLaplacian, assemble_halo, pack_boundary, partition
from conftest import assert_bits

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    return krn.Device(0, s.cuda_stream)


@pytest.mark.parametrize("world,n,align", [(2, 257, 1), (3, 5000, 1), (4, 100_003, 1024), (8, (1 << 21) + 12345, 8192),
                                           (5, 10, 1)])
def test_shards_reproduce_the_whole_problem(dev, world, n, align):
    from oracle import cport

    rng = np.random.default_rng(world * 1000 + n)
    x, b = rng.normal(size=n), rng.normal(size=n)
    dx0, db0 = rng.normal(size=n), rng.normal(size=n)
    xo, dxo, dbo = x.copy(), dx0.copy(), db0.copy()
    fo = cport.laplacian_primal(x.copy(), b.copy())
    cport.laplacian_grad(xo, b.copy(), dxo, dbo, 1.0)
    parts = partition(n, world, align)
    xt = [torch.from_numpy(x[o:o + l].copy()).cuda() for o, l in parts]
    bt = [torch.from_numpy(b[o:o + l].copy()).cuda() for o, l in parts]
    if any(l < 2 for _, l in parts):
        with pytest.raises(ValueError):
            [pack_boundary(xi, bi) for xi, bi in zip(xt, bt)]
        return
    gathered = torch.stack([pack_boundary(xi, bi) for xi, bi in zip(xt, bt)])
    f_total = 0.0
    got_x, got_dx, got_db = [], [], []
    for r, (o, l) in enumerate(parts):
        halo = assemble_halo(gathered, r, world)
        dxs, dbs = torch.from_numpy(dx0[o:o + l].copy()).cuda(), torch.from_numpy(db0[o:o + l].copy()).cuda()
        xout = torch.empty_like(xt[r])
        f = torch.zeros(1, dtype=torch.float64, device="cuda")
        P = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
        _cabi.check(dev.lib.krn_laplacian_primal(dev.h, P(xt[r]), P(xout), P(bt[r]), l, o, n, P(halo), P(f), 0))
        _cabi.check(dev.lib.krn_laplacian_grad(dev.h, P(xt[r]), P(xout), P(bt[r]), P(dxs), P(dbs), 0, 0,
                                               l, o, n, P(halo), 1.0))
        torch.cuda.synchronize()
        f_total += float(f.item())
        got_x.append(xout.cpu().numpy()), got_dx.append(dxs.cpu().numpy()), got_db.append(dbs.cpu().numpy())
    assert_bits(np.concatenate(got_x), xo, "3x")
    assert_bits(np.concatenate(got_dx), dxo, "_d_x")
    assert_bits(np.concatenate(got_db), dbo, "_d_b")
    assert abs(f_total - fo) <= 1e-13 * abs(fo)


def test_single_rank_object(dev):
    """ShardedLaplacian without a process group = the whole problem"""
    from oracle import cport

    n = 70_001
    rng = np.random.default_rng(1)
    x, b = rng.normal(size=n), rng.normal(size=n)
    sh = ShardedLaplacian(n, dev)
    assert (sh.rank, sh.world, sh.offset, sh.n_local) == (0, 1, 0, n)
    xt, bt = torch.from_numpy(x).cuda(), torch.from_numpy(b).cuda()
    xo_t, f = torch.empty_like(xt), torch.zeros(1, dtype=torch.float64, device="cuda")
    dx, db = torch.zeros_like(xt), torch.zeros_like(xt)
    sh.primal(xt, xo_t, bt, f)
    sh.grad(xt, xo_t, bt, dx, db, dx_zero=True, db_zero=True)
    torch.cuda.synchronize()
    xo, dxo, dbo = x.copy(), np.zeros(n), np.zeros(n)
    fo = cport.laplacian_primal(x.copy(), b.copy())
    cport.laplacian_grad(xo, b.copy(), dxo, dbo, 1.0)
    assert_bits(float(f.item()), fo, "f")
    assert_bits(dx.cpu().numpy(), dxo, "_d_x")
    assert_bits(db.cpu().numpy(), dbo, "_d_b")
    assert_bits(xo_t.cpu().numpy(), xo, "3x")


@pytest.mark.parametrize("world,n", [(2, 5000), (3, 100_003), (8, (1 << 21) + 12345), (4, (1 << 20) + 1), (7, 3 * 8192 * 7)])
def test_sharded_objective_is_bit_identical(dev, world, n):
    """per-block tree partials of every shard, concatenated in rank order and folded with the
    reference's tree (what ShardedLaplacian.primal does after its all_gather), equal the
    single-device objective - and the oracle's - bit for bit, for any number of shards"""
    from oracle import cport
    from paper_2507_13204_b200.sharded import combine_partials, partial_count

    rng = np.random.default_rng(world + n)
    x, b = rng.normal(size=n), rng.normal(size=n)
    fo = cport.laplacian_primal(x.copy(), b.copy())
    span = int(dev.lib.krn_laplacian_partial_span(n))
    parts = partition(n, world, span)
    xt = [torch.from_numpy(x[o:o + l].copy()).cuda() for o, l in parts]
    bt = [torch.from_numpy(b[o:o + l].copy()).cuda() for o, l in parts]
    gathered = torch.stack([pack_boundary(xi, bi) for xi, bi in zip(xt, bt)])
    counts = [partial_count(l, span) for _, l in parts]
    width = max(counts)
    rows = torch.zeros(world, width, dtype=torch.float64, device="cuda")
    P = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    plain = 0.0
    for r, (o, l) in enumerate(parts):
        halo = assemble_halo(gathered, r, world)
        xout, f = torch.empty_like(xt[r]), torch.zeros(1, dtype=torch.float64, device="cuda")
        _cabi.check(dev.lib.krn_laplacian_primal(dev.h, P(xt[r]), P(xout), P(bt[r]), l, o, n, P(halo), P(f), 0))
        _cabi.check(dev.lib.krn_laplacian_partials(dev.h, P(rows[r]), counts[r]))
        torch.cuda.synchronize()
        plain += float(f.item())
    nodes = combine_partials(rows, counts)
    f = torch.zeros(1, dtype=torch.float64, device="cuda")
    _cabi.check(dev.lib.krn_reduce_pairwise(dev.h, P(nodes), nodes.numel(), P(f), 0))
    torch.cuda.synchronize()
    assert_bits(float(f.item()), fo, f"exact objective, {world} shards")
    assert abs(plain - fo) <= 1e-13 * abs(fo)  # what a plain all_reduce(SUM) would give
