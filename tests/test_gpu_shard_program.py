"""GPU tier: sharded execution of row-wise functions (shard_program.py) with the real `execute`:
the ranks of a multi-GPU run are played by threads on ONE device (segments serialised by a lock,
the all-reduce a barrier), and once by two processes over gloo sharing the device - NCCL refuses
two ranks on one GPU.  Compared with the single-device run of the whole problem."""

import os
import threading

import numpy as np
import pytest

import paper_2507_13204_b200 as krn
from paper_2507_13204_b200 import ExecutionConfig, ViewStorage, shard_program
from conftest import assert_bits, free_port
from test_shard_program_cpu import INDEXED, ROWWISE, _data, run_sharded

pytestmark = pytest.mark.gpu
_lock = threading.Lock()


def locked_execute(program, fn_name, inputs, cfg=None):
    with _lock:  # one context, one stream: a rank's launch sequence must not interleave with another's
        return krn.execute(program, fn_name, inputs, cfg)


def _whole(program, fn_name, data, policy):
    call = {k: (ViewStorage.from_values(k, v) if isinstance(v, np.ndarray) else v) for k, v in data.items()}
    value = krn.execute(program, fn_name, call, ExecutionConfig(policy=policy)).value
    return value, {k: v.buffer for k, v in call.items() if isinstance(v, ViewStorage)}


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("n", [97, 5000, 300_001])
@pytest.mark.parametrize("stem", ROWWISE)
def test_rowwise_corpus_sharded_on_one_device(stem, n, world):
    prog = krn.load_program(stem)
    fn = prog.functions[0]
    rng = np.random.default_rng(n + world)
    data = _data(fn, n, rng)
    wrt = tuple(p.name for p in fn.params if p.is_view)
    gp = krn.differentiate(prog, fn.name, wrt)
    gfn = gp.functions[-1]
    gdata = dict(data)
    for sp, w in zip(gfn.params[len(fn.params):], wrt):
        gdata[sp.name] = rng.normal(size=np.shape(data[w]))
    exact = stem != "mean_shift"  # there a gathered scalar is written back into the Views
    for program, name, d in ((prog, fn.name, data), (gp, gfn.name, gdata)):
        wv, want = _whole(program, name, d, "compiled")
        values, whole = run_sharded(program, name, d, world, locked_execute)
        for v in values:
            if wv is None:
                assert v is None
            else:
                assert v == values[0] and abs(v - wv) <= 1e-12 * abs(wv), (stem, v, wv)
        for k, arr in whole.items():
            if exact:
                assert_bits(arr, want[k], f"{name} n={n} world={world} {k}")
            else:
                assert np.all(np.abs(arr - want[k]) <= 1e-12 * np.abs(want[k])), (name, k)


@pytest.mark.parametrize("world", [2, 5])
def test_localised_guards_on_the_device(world):
    prog = krn.parse(INDEXED)
    rng = np.random.default_rng(world)
    n = 10_007
    data = {"a": rng.normal(size=n), "b": rng.normal(size=n), "c": 0.75}
    wv, want = _whole(prog, "f", data, "compiled")
    values, whole = run_sharded(prog, "f", data, world, locked_execute)
    assert all(v == values[0] for v in values) and abs(values[0] - wv) <= 1e-12 * abs(wv)
    assert_bits(whole["a"], want["a"], "a (independent of the gathered scalars)")
    assert np.all(np.abs(whole["b"] - want["b"]) <= 1e-12 * np.abs(want["b"]))


def _gloo_worker(rank, world, port, n, out):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2507_13204_b200.sharded import partition

        prog = krn.load_program("mean_shift")
        v = np.random.default_rng(11).uniform(0.5, 1.5, size=n)
        lo, ln = partition(n, world)[rank]
        sp = shard_program.ShardedProgram(prog, "shiftedEnergy", n, lo)  # default comm: torch.distributed
        local = {"v": v[lo:lo + ln].copy()}
        value = sp.run(local)
        out.put((rank, value, local["v"].buffer.copy()))
    finally:
        dist.destroy_process_group()


def test_two_processes_over_gloo():
    import torch.multiprocessing as mp

    n, world = 20_001, 2
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, world, port, n, out)) for r in range(world)]
    for p in procs:
        p.start()
    got = sorted(out.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    prog = krn.load_program("mean_shift")
    v = np.random.default_rng(11).uniform(0.5, 1.5, size=n)
    wv, want = _whole(prog, "shiftedEnergy", {"v": v}, "compiled")
    assert got[0][1] == got[1][1] and abs(got[0][1] - wv) <= 1e-12 * abs(wv)
    assert_bits(np.concatenate([got[0][2], got[1][2]]), want["v"], "v")


def _ghost_worker(rank, world, port, n, out):
    """the headline gradient (ghost rows: 2 either side) through ShardedProgram with the default
    torch.distributed comm: the edge rows are sliced, all-gathered and copied INSIDE device memory"""
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2507_13204_b200.sharded import partition

        torch.cuda.set_device(0)
        prog = krn.load_program("laplacian")
        gp = krn.differentiate(prog, "normRes1DLaplacianSQ", ("x", "b"))
        rng = np.random.default_rng(12)
        x, b, dx, db = (rng.normal(size=n) for _ in range(4))
        lo, ln = partition(n, world)[rank]
        sp = shard_program.ShardedProgram(gp, "normRes1DLaplacianSQ_grad", n, lo)
        assert sp.ghost == 2 and hasattr(sp.comm, "exchange_rows_device")
        seen = {"host": 0}
        real = sp.comm.exchange_rows
        sp.comm.exchange_rows = lambda *a: seen.__setitem__("host", seen["host"] + 1) or real(*a)
        local = {k: ViewStorage.from_values(k, v[lo:lo + ln].copy()) for k, v in
                 (("x", x), ("b", b), ("_d_x", dx), ("_d_b", db))}
        for v in local.values():
            v.device_ptr(krn.Device.get())  # resident before the call, as in a real run
        sp.run(local)
        assert seen["host"] == 0, "ghost rows travelled through the host"
        out.put((rank, {k: v.buffer.copy() for k, v in local.items()}))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_ghost_rows_stay_on_the_device(world):
    import torch.multiprocessing as mp

    n = 30_011
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_ghost_worker, args=(r, world, port, n, out)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(out.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    prog = krn.load_program("laplacian")
    gp = krn.differentiate(prog, "normRes1DLaplacianSQ", ("x", "b"))
    rng = np.random.default_rng(12)
    x, b, dx, db = (rng.normal(size=n) for _ in range(4))
    _, want = _whole(gp, "normRes1DLaplacianSQ_grad", {"x": x, "b": b, "_d_x": dx, "_d_b": db}, "compiled")
    for k in ("x", "_d_x", "_d_b"):
        assert_bits(np.concatenate([got[r][k] for r in range(world)]), want[k], f"world={world} {k}")


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("stem", ["gather_indirect", "gather_rows_rank2"])
def test_replicated_views_and_their_scattered_shadows(stem, world):
    """indirectly indexed Views are replicated; the generated adjoint scatters into a replicated
    shadow on every rank (hardware atomics) and the copies are all-reduced at the end"""
    prog = krn.load_program(stem)
    fn = prog.functions[0]
    n, rows = 40_003, 6_001
    rng = np.random.default_rng(world)
    data = {}
    for p in fn.params:
        if p.name == "idx":
            data[p.name] = rng.integers(0, rows, size=n).astype(np.float64)
        elif p.name in ("x", "q"):
            data[p.name] = rng.normal(size=(rows, 3) if p.type.rank == 2 else rows)
        else:
            data[p.name] = rng.normal(size=n)
    wv, want = _whole(prog, fn.name, data, "compiled")
    values, whole = run_sharded(prog, fn.name, data, world, locked_execute)
    assert all(v == values[0] for v in values) and abs(values[0] - wv) <= 1e-12 * abs(wv)
    wrt = tuple(p.name for p in fn.params if p.is_view and p.name != "idx")
    gp = krn.differentiate(prog, fn.name, wrt)
    gfn = gp.functions[-1]
    gdata = dict(data)
    for sp, w in zip(gfn.params[len(fn.params):], wrt):
        gdata[sp.name] = rng.normal(size=np.shape(data[w]))
    _, want = _whole(gp, gfn.name, gdata, "statements")
    _, whole = run_sharded(gp, gfn.name, gdata, world, locked_execute)
    for k, arr in whole.items():
        assert np.all(np.abs(arr - want[k]) <= 1e-12 * np.maximum(np.abs(want[k]), 1.0)), (stem, k)


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("n", [64, 5000, 200_003])
@pytest.mark.parametrize("stem", ["laplacian", "stencil_smooth", "window_wide", "window_scatter"])
def test_neighbour_reads_through_ghost_rows_on_the_device(stem, n, world):
    """every rank keeps `ghost` rows of its neighbours and re-runs their edge iterations: own rows
    bit-identical to the single-device run (generated window kernels on both sides)"""
    prog = krn.load_program(stem)
    fn = prog.functions[0]
    rng = np.random.default_rng(n + world + len(stem))
    data = _data(fn, n, rng)
    wrt = tuple(p.name for p in fn.params if p.is_view)
    cases = [(prog, fn.name, data)]
    try:
        gp = krn.differentiate(prog, fn.name, wrt)
        gfn = gp.functions[-1]
        gdata = dict(data)
        for sp, w in zip(gfn.params[len(fn.params):], wrt):
            gdata[sp.name] = rng.normal(size=np.shape(data[w]))
        cases.append((gp, gfn.name, gdata))
    except (krn.NotFeasible, ValueError):
        pass
    for program, name, d in cases:
        wv, want = _whole(program, name, d, "compiled")
        values, whole = run_sharded(program, name, d, world, locked_execute)
        for v in values:
            if wv is None:
                assert v is None
            else:
                assert v == values[0] and abs(v - wv) <= 1e-12 * abs(wv), (stem, v, wv)
        for k, arr in whole.items():
            assert_bits(arr, want[k], f"{name} n={n} world={world} {k}")


def _gloo_worker_all(rank, world, port, n, out):
    """the torch.distributed communicator on every collective it offers: scalar all-reduce
    (laplacian primal), ghost-row exchange (laplacian gradient), array all-reduce (indirect gather)"""
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2507_13204_b200.sharded import partition

        rng = np.random.default_rng(21)
        x, b, dx, db = (rng.normal(size=n) for _ in range(4))
        idx = rng.integers(0, 500, size=n).astype(np.float64)
        xs, dxs = rng.normal(size=500), rng.normal(size=500)
        lo, ln = partition(n, world)[rank]
        sl = slice(lo, lo + ln)
        lap = krn.load_program("laplacian")
        gp = krn.differentiate(lap, "normRes1DLaplacianSQ", ("x", "b"))
        local = {"x": x[sl].copy(), "b": b[sl].copy()}
        f = shard_program.ShardedProgram(lap, "normRes1DLaplacianSQ", n, lo).run(local)
        g = {"x": x[sl].copy(), "b": b[sl].copy(), "_d_x": dx[sl].copy(), "_d_b": db[sl].copy()}
        shard_program.ShardedProgram(gp, "normRes1DLaplacianSQ_grad", n, lo).run(g)
        gi = krn.load_program("gather_indirect")
        ggi = krn.differentiate(gi, "gatherSquares", ("x",))
        h = {"x": xs.copy(), "idx": idx[sl].copy(), "_d_x": dxs.copy()}
        shard_program.ShardedProgram(ggi, "gatherSquares_grad", n, lo).run(h)
        out.put((rank, f, g["_d_x"].buffer.copy(), g["_d_b"].buffer.copy(), g["x"].buffer.copy(), h["_d_x"].buffer.copy()))
    finally:
        dist.destroy_process_group()


def test_every_collective_over_gloo():
    import torch.multiprocessing as mp

    n, world = 30_011, 2
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_gloo_worker_all, args=(r, world, port, n, out)) for r in range(world)]
    for p in procs:
        p.start()
    got = sorted(out.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(21)
    x, b, dx, db = (rng.normal(size=n) for _ in range(4))
    idx = rng.integers(0, 500, size=n).astype(np.float64)
    xs, dxs = rng.normal(size=500), rng.normal(size=500)
    lap = krn.load_program("laplacian")
    gp = krn.differentiate(lap, "normRes1DLaplacianSQ", ("x", "b"))
    wf, _ = _whole(lap, "normRes1DLaplacianSQ", {"x": x, "b": b}, "fused")
    _, want = _whole(gp, "normRes1DLaplacianSQ_grad", {"x": x, "b": b, "_d_x": dx, "_d_b": db}, "fused")
    assert got[0][1] == got[1][1] and abs(got[0][1] - wf) <= 1e-12 * abs(wf)
    assert_bits(np.concatenate([got[0][2], got[1][2]]), want["_d_x"], "_d_x")
    assert_bits(np.concatenate([got[0][3], got[1][3]]), want["_d_b"], "_d_b")
    assert_bits(np.concatenate([got[0][4], got[1][4]]), want["x"], "x")
    gi = krn.load_program("gather_indirect")
    ggi = krn.differentiate(gi, "gatherSquares", ("x",))
    _, wi = _whole(ggi, "gatherSquares_grad", {"x": xs, "idx": idx, "_d_x": dxs}, "statements")
    for r in range(world):  # the replicated shadow is the same, complete, on every rank
        assert np.all(np.abs(got[r][5] - wi["_d_x"]) <= 1e-12 * np.maximum(np.abs(wi["_d_x"]), 1.0))
    assert np.array_equal(got[0][5], got[1][5])


def test_device_tensor_aliases_the_view():
    """the NCCL path all-reduces a replicated shadow in place: the torch tensor handed to NCCL must
    alias the View's HBM buffer, not copy it"""
    import torch

    dev = krn.Device.get()
    v = ViewStorage.from_values("v", np.arange(12.0).reshape(4, 3))
    t = shard_program.device_tensor(v, dev)
    assert t.shape == (4, 3) and t.dtype == torch.float64 and t.is_cuda
    assert t.data_ptr() == v.device_ptr(dev, write=False)
    dev.sync()
    t.mul_(2.0)
    torch.cuda.synchronize()
    assert np.array_equal(v.buffer, 2.0 * np.arange(12.0).reshape(4, 3))
