"""CPU tier: sharded execution of row-wise functions (shard_program.py).  The transform under
test - segmentation at the gathers, localisation of guards / float(i) / extents, host scalars,
the all-reduce protocol - runs here with the oracle interpreter standing in for the GPU
`execute` and one thread per rank (a barrier-based all-reduce), against the whole-problem oracle."""

import threading

import numpy as np
import pytest

import paper_2507_13204_b200 as krn
from paper_2507_13204_b200 import shard_program
from paper_2507_13204_b200.sharded import partition
from conftest import assert_bits

ROWWISE = ["affine_weighted", "copy_chain", "fill_scale", "inplace_axpy", "mean_shift", "rowscale_rank2",
           "safe_divide", "sum_squares"]
INDEXED = """fn f(a: view<f64, 1>, b: view<f64, 1>, c: f64) -> f64 {
    let t: view<f64, 1> = view("t", extent(a, 0));
    let w: f64 = c * 2.0 + extent(a, 0);
    parallel_for i in 0..extent(a, 0) {
        t(i) = a(i) * i + w;
        if (i != 0) { t(i) += b(i); }
        if (i >= 5) { a(i) = a(i) - c; }
        if (i != extent(a, 0) - 1) { b(i) = b(i) * 0.5 + extent(a, 0); }
    }
    s = parallel_sum(t);
    deep_copy(t, s);
    parallel_for i in 0..extent(a, 0) { b(i) += t(i) * 1.0e-3; }
    s2 = parallel_sum(b);
    return s * 0.5 + s2 - extent(a, 0);
}"""


class ThreadComm:
    """all-reduce among `world` threads: every rank deposits its value, all sum in rank order."""

    def __init__(self, world):
        self.world, self.slots, self.barrier = world, [0.0] * world, threading.Barrier(world)

    def view(self, rank):
        comm = self

        class _C:
            def allreduce_sum(self, value):
                comm.slots[rank] = value
                comm.barrier.wait()
                total = 0.0
                for v in comm.slots:
                    total = total + v
                comm.barrier.wait()
                return total

            def exchange_rows(self, first, last):
                comm.slots[rank] = (first, last)
                comm.barrier.wait()
                below = comm.slots[rank - 1][1].copy() if rank > 0 else None
                above = comm.slots[rank + 1][0].copy() if rank < comm.world - 1 else None
                comm.barrier.wait()
                return below, above

            def allreduce_array(self, arr):
                comm.slots[rank] = arr.copy()
                comm.barrier.wait()
                total = comm.slots[0].copy()
                for v in comm.slots[1:]:
                    total = total + v
                comm.barrier.wait()
                arr[...] = total

        return _C()


def oracle_execute(program, fn_name, inputs, cfg=None):
    """stand-in for runtime.execute on the CPU: the oracle interpreter on the Views' host arrays"""
    from oracle import interp

    arrays = {k: (v.buffer if isinstance(v, krn.ViewStorage) else v) for k, v in inputs.items()}
    return krn.ExecResult(interp.run(program, fn_name, arrays))


def run_sharded(program, fn_name, data, world, execute):
    """data: whole-problem arrays/scalars.  Returns (values per rank, whole arrays reassembled)."""
    fn = program.function(fn_name)
    rep, _ = shard_program.classify(fn)
    n = next(np.shape(data[p.name])[0] for p in fn.params if p.is_view and p.name not in rep)
    parts = partition(n, world)
    comm = ThreadComm(world)
    results, pieces, errors = [None] * world, [None] * world, []

    def work(r):
        try:
            lo, ln = parts[r]
            replicated, _ = shard_program.classify(fn)
            local = {k: ((np.array(v) if k in replicated else np.array(v[lo:lo + ln])) if isinstance(v, np.ndarray)
                         else v) for k, v in data.items()}
            sp = shard_program.ShardedProgram(program, fn_name, n, lo, comm.view(r))
            results[r] = sp.run(local)
            pieces[r] = {k: (v.buffer if isinstance(v, krn.ViewStorage) else v) for k, v in local.items()}
        except Exception as e:  # noqa: BLE001
            errors.append(e)
            comm.barrier.abort()

    old = shard_program.__dict__.get("_execute_override")
    shard_program._execute_override = execute
    try:
        threads = [threading.Thread(target=work, args=(r,)) for r in range(world)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
    finally:
        shard_program._execute_override = old
    if errors:
        raise errors[0]
    replicated, _ = shard_program.classify(fn)
    whole = {}
    for k, v in data.items():
        if isinstance(v, np.ndarray):
            if k in replicated:
                for p in pieces[1:]:
                    assert np.array_equal(p[k], pieces[0][k]), f"replicated view {k} differs between ranks"
                whole[k] = pieces[0][k]
            else:
                whole[k] = np.concatenate([p[k] for p in pieces])
    return results, whole


def _data(fn, n, rng):
    out = {}
    for p in fn.params:
        if not p.is_view:
            out[p.name] = 0.75
        elif p.type.rank == 2:
            out[p.name] = rng.uniform(0.5, 1.5, size=(n, 3))
        else:
            out[p.name] = rng.uniform(0.5, 1.5, size=n)
    return out


def _check(program, fn_name, data, world, exact_views):
    from oracle import interp

    want = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in data.items()}
    wv = interp.run(program, fn_name, want)
    values, whole = run_sharded(program, fn_name, data, world, oracle_execute)
    for v in values:
        if wv is None:
            assert v is None
        else:
            assert v == values[0] and abs(v - wv) <= 1e-12 * abs(wv), (v, wv)
    for k, arr in whole.items():
        if exact_views:
            assert_bits(arr, want[k], f"{fn_name} world={world} {k}")
        else:
            assert np.all(np.abs(arr - want[k]) <= 1e-12 * np.abs(want[k])), (fn_name, k)


@pytest.mark.parametrize("world", [1, 2, 3])
@pytest.mark.parametrize("stem", ROWWISE)
def test_rowwise_corpus_programs_and_gradients(stem, world):
    prog = krn.load_program(stem)
    fn = prog.functions[0]
    rng = np.random.default_rng(len(stem) + world)
    n = 41
    data = _data(fn, n, rng)
    feeds_views = stem == "mean_shift"  # a gathered scalar is written back into Views there
    _check(prog, fn.name, data, world, exact_views=not feeds_views)
    wrt = tuple(p.name for p in fn.params if p.is_view)
    gp = krn.differentiate(prog, fn.name, wrt)
    gfn = gp.functions[-1]
    gdata = dict(data)
    for sp, w in zip(gfn.params[len(fn.params):], wrt):
        gdata[sp.name] = rng.normal(size=np.shape(data[w]))
    _check(gp, gfn.name, gdata, world, exact_views=not feeds_views)


@pytest.mark.parametrize("world", [1, 2, 4])
def test_guards_float_i_and_extents_are_localised(world):
    prog = krn.parse(INDEXED)
    rng = np.random.default_rng(world)
    data = {"a": rng.normal(size=23), "b": rng.normal(size=23), "c": 0.75}
    _check(prog, "f", data, world, exact_views=False)
    # the first kernel's Views do not depend on a gathered scalar: compare those exactly
    from oracle import interp

    want = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in data.items()}
    interp.run(prog, "f", want)
    _, whole = run_sharded(prog, "f", data, world, oracle_execute)
    assert_bits(whole["a"], want["a"], "a")


@pytest.mark.parametrize("world", [2, 3])
def test_row_number_in_an_atomic_contribution_is_localised(world):
    """float(i) inside the VALUE of an atomic_add (the generated adjoint of `t(i) = i * m(i, c)`): found
    by the random-program test below - the contribution was computed with the rank-local row"""
    prog = krn.parse("""fn f(a: view<f64, 1>, m: view<f64, 2>) -> f64 {
        let t0: view<f64, 1> = view("t0", extent(a, 0));
        parallel_for i in 0..extent(a, 0) { t0(i) = (i * (m(i, 0) + m(i, 1))) + a(i); }
        r = parallel_sum(t0);
        return r;
    }""")
    rng = np.random.default_rng(7)
    n = 37
    gp = krn.differentiate(prog, "f", ("a", "m"))
    gfn = gp.functions[-1]
    assert any(type(s).__name__ == "AtomicAdd" for s in krn.lang.nodes.walk_statements(gfn.body))
    data = {"a": rng.normal(size=n), "m": rng.normal(size=(n, 3)),
            "_d_a": rng.normal(size=n), "_d_m": rng.normal(size=(n, 3))}
    _check(gp, gfn.name, data, world, exact_views=True)


def test_segments_are_plain_functions_of_the_language():
    prog = krn.load_program("mean_shift")
    sp = shard_program.ShardedProgram(prog, "shiftedEnergy", 100, 25, comm=ThreadComm(1).view(0))
    kinds = [s.what for s in sp.steps]
    assert kinds == ["host", "decl", "segment", "segment", "return"]
    seg = [s for s in sp.steps if s.what == "segment"]
    assert seg[0].gather == ("total", True) and seg[1].scalars == ("total",)
    from paper_2507_13204_b200.lang.nodes import Program

    for s in seg:
        assert krn.validate(Program((s.fn,))) == []
        krn.parse(krn.emit(Program((s.fn,))).replace("__part", "part_"))  # prints and parses back


@pytest.mark.parametrize("world", [1, 2, 3])
@pytest.mark.parametrize("stem", ["gather_indirect", "gather_rows_rank2"])
def test_indirectly_indexed_views_are_replicated(stem, world):
    """x(idx(i)) / q(idx(i), c): the indexed View is replicated, its shadow accumulates per rank and
    is all-reduced at the end"""
    from oracle import interp

    prog = krn.load_program(stem)
    fn = prog.functions[0]
    n, rows = 53, 17
    rng = np.random.default_rng(world)
    data = {}
    for p in fn.params:
        if p.name == "idx":
            data[p.name] = rng.integers(0, rows, size=n).astype(np.float64)
        elif p.name in ("x", "q"):
            data[p.name] = rng.normal(size=(rows, 3) if p.type.rank == 2 else rows)
        else:
            data[p.name] = rng.normal(size=n)
    assert shard_program.classify(fn)[0] == {"x"} or shard_program.classify(fn)[0] == {"q"}
    _check(prog, fn.name, data, world, exact_views=True)
    wrt = tuple(p.name for p in fn.params if p.is_view and p.name != "idx")
    gp = krn.differentiate(prog, fn.name, wrt)
    gfn = gp.functions[-1]
    gdata = dict(data)
    for sp, w in zip(gfn.params[len(fn.params):], wrt):
        gdata[sp.name] = rng.normal(size=np.shape(data[w]))
    rep, scat = shard_program.classify(gfn)
    assert scat == {"_d_" + next(iter(shard_program.classify(fn)[0]))}
    want = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in gdata.items()}
    interp.run(gp, gfn.name, want)
    _, whole = run_sharded(gp, gfn.name, gdata, world, oracle_execute)
    for k, arr in whole.items():
        assert np.all(np.abs(arr - want[k]) <= 1e-12 * np.maximum(np.abs(want[k]), 1.0)), (stem, k)


@pytest.mark.parametrize("world", [1, 2, 3, 5])
@pytest.mark.parametrize("stem", ["laplacian", "stencil_smooth", "window_wide", "window_partial", "window_war",
                                  "window_scatter"])
def test_neighbour_reads_are_served_by_ghost_rows(stem, world):
    """stencils, scatters to neighbouring rows, in-place updates read by neighbours: every rank keeps
    `ghost` rows of its neighbours and recomputes their edge iterations; own rows must equal the
    single-device result bit for bit (gathered scalars within 1e-12)"""
    from oracle import interp

    prog = krn.load_program(stem)
    fn = prog.functions[0]
    rng = np.random.default_rng(world + len(stem))
    n = 61
    data = _data(fn, n, rng)
    assert shard_program.classify(fn).ghost >= 1
    _check(prog, fn.name, data, world, exact_views=True)
    wrt = tuple(p.name for p in fn.params if p.is_view)
    try:
        gp = krn.differentiate(prog, fn.name, wrt)
    except (krn.NotFeasible, ValueError):
        return
    gfn = gp.functions[-1]
    gdata = dict(data)
    for sp, w in zip(gfn.params[len(fn.params):], wrt):
        gdata[sp.name] = rng.normal(size=np.shape(data[w]))
    _check(gp, gfn.name, gdata, world, exact_views=True)


def test_shards_smaller_than_the_ghost_band_are_refused():
    prog = krn.load_program("laplacian")
    gp = krn.differentiate(prog, "normRes1DLaplacianSQ", ("x", "b"))
    data = {k: np.ones(3) for k in ("x", "b", "_d_x", "_d_b")}
    with pytest.raises(shard_program.NotShardable, match="at least 2 rows"):
        run_sharded(gp, "normRes1DLaplacianSQ_grad", data, 3, oracle_execute)


def test_strided_accesses_are_refused():
    prog = krn.parse("""fn f(a: view<f64, 1>, b: view<f64, 1>) { parallel_for i in 0..extent(b, 0) {
                        b(i) = a(2 * i); } }""")
    with pytest.raises(shard_program.NotShardable):
        shard_program.ShardedProgram(prog, "f", 100, 0, comm=ThreadComm(1).view(0))


def test_random_programs_sharded_against_the_whole_problem():
    """random programs (pointwise statements, stencils on inputs and on temporaries, in-place
    updates, fills, copies, gathers feeding later statements, rank-2 rows, indirect reads) and their
    gradients: sharded over 2 and 3 ranks with the oracle as executor, against the oracle on the
    whole problem"""
    import warnings

    from hypothesis import HealthCheck, assume, given, settings, strategies as st

    from oracle import interp
    from test_gpu_random_programs import _inputs as fuzz_inputs, programs

    ran = [0]

    # the default run draws the same 150 programs every time; KRN_FUZZ=<n> explores n fresh ones
    import os

    @settings(max_examples=int(os.environ.get("KRN_FUZZ", "150")), deadline=None, suppress_health_check=list(HealthCheck),
              derandomize="KRN_FUZZ" not in os.environ, database=None)
    @given(programs(), st.sampled_from([2, 3]), st.integers(0, 10**6))
    def run(prog, world, seed):
        text, use_idx, use_c, use_m = prog
        program = krn.parse(text)
        n = 37
        base = fuzz_inputs(n, use_idx, use_c, seed, use_m)
        cases = [(program, "f", base)]
        wrt = ("a", "b") + (("m",) if use_m else ())
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            try:
                gp = krn.differentiate(program, "f", wrt, tape=True)
                gfn = gp.functions[-1]
                gdata = dict(base)
                rng = np.random.default_rng(seed)
                for sp in gfn.params[len(program.functions[0].params):]:
                    gdata[sp.name] = rng.normal(size=np.shape(base[sp.name[3:]]))
                cases.append((gp, gfn.name, gdata))
            except krn.NotFeasible:
                pass
        for pr, name, data in cases:
            try:
                cls = shard_program.classify(pr.function(name))
            except shard_program.NotShardable:
                continue
            if cls.ghost and n // world < cls.ghost:
                continue
            want = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in data.items()}
            with np.errstate(all="ignore"):
                wv = interp.run(pr, name, want)
                values, whole = run_sharded(pr, name, data, world, oracle_execute)
            if wv is not None:
                assume(np.isfinite(wv))
                assert all(v == values[0] for v in values)
                assert abs(values[0] - wv) <= 1e-9 * max(1.0, abs(wv)), (text, values[0], wv)
            for k, arr in whole.items():
                scale = max(1.0, float(np.max(np.abs(want[k])))) if want[k].size else 1.0
                assert np.all(np.abs(arr - want[k]) <= 1e-9 * scale) or not np.all(np.isfinite(want[k])), (text, name, k)
            ran[0] += 1

    run()
    assert ran[0] >= 60


def test_order_dependent_kernels_are_refused():
    """A kernel whose iterations may meet at a plainly written location has a result defined by one
    in-order sweep over the whole range (runtime._Run.do_kernel): it cannot be cut across ranks."""
    import paper_2507_13204_b200 as krn
    from paper_2507_13204_b200 import shard_program as sp

    scan = krn.parse("fn f(v: view<f64,1>) -> f64 { parallel_for i in 0..extent(v,0) { if (i != 0) { "
                     "v(i) = v(i - 1) + i; } } return v(extent(v,0) - 1); }")
    with pytest.raises(sp.NotShardable, match="depends on their order"):
        sp.check_shardable(scan.functions[0])
    sp.check_shardable(krn.load_program("stencil_smooth").functions[0])   # neighbours of a read-only View: fine
