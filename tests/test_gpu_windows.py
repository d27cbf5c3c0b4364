"""GPU parity, halo-recompute fusion (tilegen.window_kernel): statements that exchange
values between neighbouring iterations run in one kernel, each warp re-running the few
iterations either side of its own 128 whose results it reads.  Checked bit for bit
against the CPU oracle at sizes around the warp-step (128), block (1024) and multi-step
(2^20) boundaries, and against the statement path at bandwidth-bound sizes."""

import numpy as np
import pytest

import paper_2507_13204_b200 as krn
from paper_2507_13204_b200 import ExecutionConfig, ViewStorage, compiled, parse
from conftest import assert_bits

pytestmark = pytest.mark.gpu
WIN = ExecutionConfig(policy="compiled")
STMT = ExecutionConfig(policy="statements")

WIDE = """fn f(a: view<f64, 1>, b: view<f64, 1>, c: view<f64, 1>) -> f64 {
    let t: view<f64, 1> = view("t", extent(a, 0));
    let u: view<f64, 1> = view("u", extent(a, 0));
    parallel_for i in 0..extent(a, 0) { a(i) = 0.5 * a(i) + b(i); }
    parallel_for i in 0..extent(a, 0) {
        t(i) = a(i);
        if (i >= 3) { t(i) += 0.25 * a(i - 3); }
        if (i < extent(a, 0) - 2) { t(i) -= 1.5 * a(i + 2); }
    }
    parallel_for i in 0..extent(a, 0) {
        u(i) = t(i) * t(i);
        if (i != 0) { u(i) += t(i - 1) * b(i); }
        if (i != extent(a, 0) - 1) { u(i) -= t(i + 1); }
    }
    parallel_for i in 0..extent(a, 0) { c(i) = u(i) - b(i); }
    return parallel_sum(u);
}"""

# a window View that is only partly rewritten (guarded), read at an offset, rewritten again
PARTIAL = """fn f(a: view<f64, 1>, b: view<f64, 1>) -> f64 {
    let t: view<f64, 1> = view("t", extent(a, 0));
    parallel_for i in 0..extent(a, 0) { if (i >= 2) { a(i) = a(i) * 3.0; } }
    parallel_for i in 0..extent(a, 0) { t(i) = b(i); if (i != 0) { t(i) += a(i - 1); } }
    parallel_for i in 0..extent(a, 0) { a(i) = a(i) - t(i); }
    parallel_for i in 0..extent(a, 0) { b(i) = t(i); if (i != extent(a, 0) - 1) { b(i) += a(i + 1); } }
    return parallel_sum(t);
}"""

# write-after-read across iterations: the stencil must see the OLD neighbours
WAR = """fn f(a: view<f64, 1>, b: view<f64, 1>) {
    parallel_for i in 0..extent(a, 0) { b(i) = a(i); if (i != 0) { b(i) += a(i - 1); } }
    parallel_for i in 0..extent(a, 0) { a(i) = 2.0 * b(i); }
    parallel_for i in 0..extent(a, 0) { if (i != extent(a, 0) - 1) { b(i) -= a(i + 1); } }
}"""

# scatter with offsets on both sides, applied to a View the next statement rescales
SCATTER = """fn f(a: view<f64, 1>, acc: view<f64, 1>) {
    parallel_for i in 0..extent(a, 0) {
        if (i >= 2) { atomic_add(acc(i - 2), a(i) * 0.5); }
        atomic_add(acc(i), a(i));
        if (i != extent(a, 0) - 1) { atomic_add(acc(i + 1), -a(i)); }
        atomic_add(acc(i), 0.125);
    }
    parallel_for i in 0..extent(a, 0) { acc(i) = acc(i) * a(i); }
}"""

CASES = {"wide": WIDE, "partial": PARTIAL, "war": WAR, "scatter": SCATTER}
SIZES = [1, 2, 3, 4, 5, 6, 31, 32, 33, 127, 128, 129, 130, 131, 132, 255, 256, 257, 1023, 1024, 1025, 1027, 2500]


def _views(fn, n, rng):
    return {p.name: rng.normal(size=n) for p in fn.params if p.is_view}


@pytest.mark.parametrize("name", sorted(CASES))
def test_plan_uses_one_window_kernel(name):
    fn = parse(CASES[name]).functions[0]
    plan = compiled.plan_for(fn, True)
    assert plan.windowed
    assert sum(1 for s in plan.steps if s[0] in ("group", "kernel")) == 1


@pytest.mark.parametrize("n", SIZES)
@pytest.mark.parametrize("name", sorted(CASES))
def test_window_kernels_against_oracle(name, n):
    from oracle import interp

    prog = parse(CASES[name])
    fn = prog.functions[0]
    data = _views(fn, n, np.random.default_rng(7 * n + len(name)))
    want = {k: v.copy() for k, v in data.items()}
    wv = interp.run(prog, "f", want)
    got = {k: ViewStorage.from_values(k, v) for k, v in data.items()}
    assert_bits(krn.execute(prog, "f", got, WIN).value, wv, f"{name} n={n} value")
    for k in data:
        assert_bits(got[k].buffer, want[k], f"{name} n={n} {k}")


@pytest.mark.parametrize("n", [5, 129, 1030])
@pytest.mark.parametrize("name", ["wide", "partial"])
def test_gradients_of_window_programs(name, n):
    from oracle import interp

    prog = parse(CASES[name])
    gp = krn.differentiate(prog, "f", ("a", "b"))
    gfn = gp.functions[-1]
    data = _views(prog.functions[0], n, np.random.default_rng(n))
    want = {k: v.copy() for k, v in data.items()}
    got = {k: ViewStorage.from_values(k, v) for k, v in data.items()}
    for p in gfn.params[len(prog.functions[0].params):]:
        want[p.name] = np.zeros(n)
        got[p.name] = ViewStorage.zeros(p.name, (n,))
    interp.run(gp, gfn.name, want)
    krn.execute(gp, gfn.name, got, WIN)
    for k in want:
        assert_bits(got[k].buffer, want[k], f"{name} grad n={n} {k}")


@pytest.mark.parametrize("n", [(1 << 20) - 1, 1 << 20, (1 << 20) + 1, (1 << 20) + 1024 * 8 + 5, 3_000_017])
@pytest.mark.parametrize("name", sorted(CASES))
def test_window_kernels_large_against_statement_path(name, n):
    """multi-step warps (8 steps of 128 rows above 2^20 iterations): the statement path, itself
    checked against the oracle, is the yardstick"""
    prog = parse(CASES[name])
    data = _views(prog.functions[0], n, np.random.default_rng(n % 1000))
    ref = {k: ViewStorage.from_values(k, v) for k, v in data.items()}
    got = {k: ViewStorage.from_values(k, v) for k, v in data.items()}
    rv = krn.execute(prog, "f", ref, STMT).value
    gv = krn.execute(prog, "f", got, WIN).value
    assert_bits(gv, rv, f"{name} n={n} value")
    for k in data:
        assert_bits(got[k].buffer, ref[k].buffer, f"{name} n={n} {k}")


def test_prefilled_and_longer_views_take_the_safe_route():
    """a View longer than the range cannot be swapped out of place: the call must still be right
    (the dry check hands it to the pointwise plan)"""
    from oracle import interp

    prog = parse(WAR)
    n = 300
    rng = np.random.default_rng(3)
    a, b = rng.normal(size=n), rng.normal(size=n + 7)
    want = {"a": a.copy(), "b": b.copy()}
    interp.run(prog, "f", want)
    got = {"a": ViewStorage.from_values("a", a), "b": ViewStorage.from_values("b", b)}
    krn.execute(prog, "f", got, WIN)
    assert_bits(got["a"].buffer, want["a"], "a")
    assert_bits(got["b"].buffer, want["b"], "b")


def test_aliased_arguments_keep_reference_semantics():
    """one storage object bound to two parameters: registers and windows would hide the aliasing
    (a = 3a instead of 4a here), so the call runs on the statement path"""
    from oracle import interp

    src = """fn f(a: view<f64, 1>, b: view<f64, 1>) {
        parallel_for i in 0..extent(a, 0) { b(i) = a(i) * 2.0; }
        parallel_for i in 0..extent(a, 0) { a(i) = a(i) + b(i); } }"""
    prog = parse(src)
    v = np.random.default_rng(5).normal(size=200)
    shared = v.copy()
    interp.run(prog, "f", {"a": shared, "b": shared})
    assert_bits(shared, 4.0 * v, "oracle aliases")
    s = ViewStorage.from_values("a", v)
    krn.execute(prog, "f", {"a": s, "b": s}, WIN)
    assert_bits(s.buffer, shared, "aliased")


def test_repeated_calls_accumulate_like_the_reference():
    """out-of-place outputs are adopted by the View: a second call must see the first call's result"""
    from oracle import interp

    lap = krn.load_program("laplacian")
    gp = krn.differentiate(lap, "normRes1DLaplacianSQ", ("x", "b"))
    n = 777
    rng = np.random.default_rng(9)
    x, b = rng.normal(size=n), rng.normal(size=n)
    want = {"x": x.copy(), "b": b.copy(), "_d_x": np.zeros(n), "_d_b": np.zeros(n)}
    got = {"x": ViewStorage.from_values("x", x), "b": ViewStorage.from_values("b", b),
           "_d_x": ViewStorage.zeros("_d_x", (n,)), "_d_b": ViewStorage.zeros("_d_b", (n,))}
    for _ in range(2):
        interp.run(gp, "normRes1DLaplacianSQ_grad", want)
        krn.execute(gp, "normRes1DLaplacianSQ_grad", got, WIN)
    for k in want:
        assert_bits(got[k].buffer, want[k], k)


# ---- rank-2 Views: rows at the running index, literal columns -> register columns --------------------

RANK2 = """fn f(m: view<f64, 2>, r: view<f64, 1>, out: view<f64, 2>) -> f64 {
    let q: view<f64, 2> = view("q", extent(m, 0), extent(m, 1));
    deep_copy(q, 0.5);
    parallel_for i in 0..extent(m, 0) {
        q(i, 0) += r(i) * m(i, 0);
        q(i, 2) = q(i, 0) - m(i, 1);
        if (i != 0) { q(i, 1) = m(i, 2) * r(i - 1); }
    }
    parallel_sum(out, q);
    parallel_for i in 0..extent(m, 0) { out(i, 1) -= r(i); m(i, 0) = q(i, 2); }
    return parallel_sum(out);
}"""


@pytest.mark.parametrize("n", [1, 2, 5, 127, 128, 129, 1025, 4100])
def test_rank2_register_columns_against_oracle(n):
    from oracle import interp

    prog = parse(RANK2)
    plan = compiled.plan_for(prog.functions[0], True)
    # every rank-2 statement (bulk ones included) runs in a generated window kernel, none through the library
    assert plan.windowed and not any(s[0] in ("kernel", "deepcopy", "suminto") for s in plan.steps)
    rng = np.random.default_rng(n)
    data = {"m": rng.normal(size=(n, 3)), "r": rng.normal(size=n), "out": rng.normal(size=(n, 3))}
    want = {k: v.copy() for k, v in data.items()}
    wv = interp.run(prog, "f", want)
    got = {k: ViewStorage.from_values(k, v) for k, v in data.items()}
    assert_bits(krn.execute(prog, "f", got, WIN).value, wv, f"n={n} value")
    for k in data:
        assert_bits(got[k].buffer, want[k], f"n={n} {k}")


def test_rank2_with_more_columns_than_the_program_names():
    """deep_copy / parallel_sum over a rank-2 View are unrolled over the columns the function names;
    a View with MORE columns must take the general route and still be right"""
    from oracle import interp

    prog = parse(RANK2)
    n = 300
    rng = np.random.default_rng(1)
    data = {"m": rng.normal(size=(n, 5)), "r": rng.normal(size=n), "out": rng.normal(size=(n, 5))}
    want = {k: v.copy() for k, v in data.items()}
    wv = interp.run(prog, "f", want)
    got = {k: ViewStorage.from_values(k, v) for k, v in data.items()}
    assert_bits(krn.execute(prog, "f", got, WIN).value, wv, "value")
    for k in data:
        assert_bits(got[k].buffer, want[k], k)


def test_rank2_column_out_of_bounds_is_reported_like_the_reference():
    prog = parse(RANK2)
    n = 10
    rng = np.random.default_rng(2)
    data = {"m": rng.normal(size=(n, 2)), "r": rng.normal(size=n), "out": rng.normal(size=(n, 2))}
    with pytest.raises(krn.OutOfBounds, match=r"outside extents 10x2"):
        krn.execute(prog, "f", {k: ViewStorage.from_values(k, v) for k, v in data.items()}, WIN)


@pytest.mark.parametrize("n", [3, 1000, 1 << 21])
def test_rowscale_gradient_prefilled_shadows(n):
    """the shipped 2-D case with accumulating shadows, against the statement path (itself checked
    against the oracle in test_gpu_corpus)"""
    prog = krn.load_program("rowscale_rank2")
    gp = krn.differentiate(prog, "rowScaleEnergy", ("m", "r"))
    rng = np.random.default_rng(n)
    data = {"m": rng.normal(size=(n, 3)), "r": rng.normal(size=n), "_d_m": rng.normal(size=(n, 3)),
            "_d_r": rng.normal(size=n)}
    ref = {k: ViewStorage.from_values(k, v) for k, v in data.items()}
    got = {k: ViewStorage.from_values(k, v) for k, v in data.items()}
    krn.execute(gp, "rowScaleEnergy_grad", ref, STMT)
    krn.execute(gp, "rowScaleEnergy_grad", got, WIN)
    for k in data:
        assert_bits(got[k].buffer, ref[k].buffer, f"n={n} {k}")


def test_untouched_local_read_at_neighbours_reads_as_zero():
    """found by the random-program test: a fresh local (all +0.0) read at i - 1 / i + 1 lives in a
    window that nothing loads - the window itself must be zero filled"""
    from oracle import interp

    src = """fn f(a: view<f64, 1>, b: view<f64, 1>) -> f64 {
        let t0: view<f64, 1> = view("t0", extent(a, 0));
        let t1: view<f64, 1> = view("t1", extent(a, 0));
        parallel_for i in 0..extent(a, 0) { t0(i) = t1(i) + a(i); if (i != 0) { t0(i) += 0.5 * t1(i - 1); }
                                            if (i != extent(a, 0) - 1) { t0(i) -= 0.5 * t1(i + 1); } }
        parallel_for i in 0..extent(a, 0) { a(i) = 0.5 * a(i) + b(i); }
        r = parallel_sum(t0);
        return r; }"""
    prog = parse(src)
    for n in (2, 130, 1030):
        rng = np.random.default_rng(n)
        data = {"a": rng.normal(size=n), "b": rng.normal(size=n)}
        want = {k: v.copy() for k, v in data.items()}
        wv = interp.run(prog, "f", want)
        got = {k: ViewStorage.from_values(k, v) for k, v in data.items()}
        assert_bits(krn.execute(prog, "f", got, WIN).value, wv, f"n={n} value")
        assert_bits(got["a"].buffer, want["a"], f"n={n} a")


def test_rank2_partial_column_store_keeps_the_other_columns():
    """found by the taped-gradient test: a zero-provenance rank-2 View of which a kernel writes
    only some columns must still read as zero in the others afterwards"""
    from oracle import interp

    src = """fn f(m: view<f64, 2>, out: view<f64, 2>) -> f64 {
        parallel_for i in 0..extent(m, 0) { out(i, 1) = m(i, 0) * 2.0; }
        return parallel_sum(out); }"""
    prog = parse(src)
    for n in (1, 130, 5000):
        m = np.random.default_rng(n).normal(size=(n, 3))
        want = {"m": m.copy(), "out": np.zeros((n, 3))}
        wv = interp.run(prog, "f", want)
        # poison the pool so that a skipped zero fill shows
        junk = ViewStorage.from_values("junk", np.full((n, 3), 7.0))
        junk.device_ptr(krn.Device.get())
        del junk
        got = {"m": ViewStorage.from_values("m", m), "out": ViewStorage.zeros("out", (n, 3))}
        assert_bits(krn.execute(prog, "f", got, WIN).value, wv, f"n={n} value")
        assert_bits(got["out"].buffer, want["out"], f"n={n} out")


@pytest.mark.parametrize("cols", [1, 2, 3, 4])
@pytest.mark.parametrize("n", [1, 2, 3, 5, 42, 43, 127, 128, 129, 341, 342, 1023, 1024, 1025, 2731, 8192, 8193,
                               (1 << 20) - 1, 1 << 20, (1 << 20) + 1, (1 << 20) + 8192 * 3 + 17])
def test_fused_flat_reduction_of_rank2_views(cols, n):
    """`parallel_sum(q)` over a rank-2 View is the reference's tree over the FLATTENED buffer
    (leaf = row * C + column).  Fused into the producing kernel the 128 x C leaves of a warp step are
    C aligned subtrees; the objective must keep the reference's bits for every C, around the warp /
    block / multi-step boundaries, without q ever being stored."""
    from oracle import interp

    body = "\n".join(f"        q(i, {c}) = r(i) * m(i, {c}) + {c}.5;" for c in range(cols))
    src = f"""fn f(m: view<f64, 2>, r: view<f64, 1>) -> f64 {{
        let q: view<f64, 2> = view("q", extent(m, 0), extent(m, 1));
        parallel_for i in 0..extent(m, 0) {{
{body}
        }}
        s = parallel_sum(q);
        return s; }}"""
    prog = parse(src)
    plan = compiled.plan_for(prog.functions[0], True)
    assert plan.launch_count == 1 and not any(s[0] == "gather" for s in plan.steps)
    rng = np.random.default_rng(cols * 1000 + n % 997)
    m, r = rng.normal(size=(n, cols)), rng.normal(size=n)
    if n <= 3000:
        want = interp.run(prog, "f", {"m": m.copy(), "r": r.copy()})
    else:
        want = krn.execute(prog, "f", {"m": ViewStorage.from_values("m", m), "r": ViewStorage.from_values("r", r)},
                           STMT).value
    got = krn.execute(prog, "f", {"m": ViewStorage.from_values("m", m), "r": ViewStorage.from_values("r", r)}, WIN).value
    assert_bits(got, want, f"cols={cols} n={n}")


def test_fused_flat_reduction_needs_exactly_the_named_columns():
    """a View with more columns than the kernel names: the fused layout does not apply, the general
    route must still give the reference's value"""
    from oracle import interp

    src = """fn f(m: view<f64, 2>, r: view<f64, 1>) -> f64 {
        let q: view<f64, 2> = view("q", extent(m, 0), extent(m, 1));
        parallel_for i in 0..extent(m, 0) { q(i, 0) = r(i) * m(i, 0); q(i, 1) = m(i, 1); }
        s = parallel_sum(q);
        return s; }"""
    prog = parse(src)
    rng = np.random.default_rng(0)
    m, r = rng.normal(size=(300, 3)), rng.normal(size=300)
    want = interp.run(prog, "f", {"m": m.copy(), "r": r.copy()})
    got = krn.execute(prog, "f", {"m": ViewStorage.from_values("m", m), "r": ViewStorage.from_values("r", r)}, WIN).value
    assert_bits(got, want, "3 columns, 2 named")
