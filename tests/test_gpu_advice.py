"""Regression tests for defects found by review of round 1: scalar parameters that the
function redefines with device data, function-scope `if` blocks holding bulk statements, and lazily
zero shadows longer than the range of the fused headline kernels.  Every policy against the CPU
oracle, bit for bit."""

import numpy as np
import pytest

import paper_2507_13204_b200 as krn
from paper_2507_13204_b200 import ExecutionConfig, ViewStorage, parse
from conftest import assert_bits

pytestmark = pytest.mark.gpu

POLICIES = ("fused", "compiled", "statements")


def _both(src, fn, inputs, policy):
    from oracle import interp

    p = parse(src)
    want = {k: (np.array(v, dtype=np.float64) if isinstance(v, np.ndarray) else v) for k, v in inputs.items()}
    wv = interp.run(p, fn, want)
    got = {k: (ViewStorage.from_values(k, v) if isinstance(v, np.ndarray) else v) for k, v in inputs.items()}
    gv = krn.execute(p, fn, got, ExecutionConfig(policy=policy)).value
    if wv is None:
        assert gv is None
    else:
        assert_bits(gv, wv, f"{policy} value")
    for k, v in got.items():
        if isinstance(v, ViewStorage):
            assert_bits(v.buffer, want[k], f"{policy} {k}")


@pytest.mark.parametrize("policy", POLICIES)
def test_scalar_parameter_gathered_into(policy):
    """reference runtime.py:650: scalars[dst] = scalars.get(dst, 0.0) + total - the parameter's value
    is the base of the gather, and the kernel after it must read the NEW value"""
    src = """fn f(x: view<f64, 1>, y: view<f64, 1>, alpha: f64) -> f64 {
        alpha = parallel_sum(x);
        parallel_for i in 0..extent(x, 0) { y(i) = alpha * x(i); }
        return alpha; }"""
    rng = np.random.default_rng(1)
    for n in (1, 5, 1000, 70_000):
        _both(src, "f", {"x": rng.normal(size=n), "y": np.zeros(n), "alpha": 0.375}, policy)


@pytest.mark.parametrize("policy", POLICIES)
def test_scalar_parameter_reassigned_from_a_view(policy):
    src = """fn f(x: view<f64, 1>, y: view<f64, 1>, alpha: f64, beta: f64) -> f64 {
        alpha = alpha + x(0);
        beta = beta * 2.0;
        parallel_for i in 0..extent(x, 0) { y(i) = alpha * x(i) + beta; }
        if (extent(x, 0) > 3) { alpha = alpha - 1.0; }
        s = parallel_sum(y);
        return s + alpha; }"""
    rng = np.random.default_rng(2)
    for n in (1, 3, 4, 2000):
        _both(src, "f", {"x": rng.normal(size=n), "y": np.zeros(n), "alpha": 0.375, "beta": -1.5}, policy)


@pytest.mark.parametrize("policy", POLICIES)
def test_function_scope_if_with_bulk_statements(policy):
    """reference runtime.py:548-550 executes the body of a function-scope `if`, whatever it holds"""
    src = """fn g(x: view<f64, 1>, out: view<f64, 1>, alpha: f64) -> f64 {
        alpha = alpha + x(0);
        if (extent(x, 0) > 2) {
            let t: view<f64, 1> = view("t", extent(x, 0));
            parallel_for i in 0..extent(x, 0) { t(i) = alpha * x(i); }
            deep_copy(out, t);
            if (extent(x, 0) > 100) { parallel_sum(out, 0.5); }
            let c: f64 = 2.0;
            alpha += c;
        }
        if (extent(x, 0) < 2) { deep_copy(out, 7.0); }
        alpha = parallel_sum(out);
        return alpha; }"""
    rng = np.random.default_rng(3)
    for n in (1, 2, 3, 100, 101, 5000):
        _both(src, "g", {"x": rng.normal(size=n), "out": np.ones(n), "alpha": 0.5}, policy)


def test_headline_gradient_with_shadows_longer_than_x():
    """b, _d_x, _d_b may have MORE rows than x (only rows < extent(x, 0) are touched): the tails of
    lazily zero shadows must come back as zeros, and longer caller-filled shadows keep theirs"""
    from oracle import interp

    lap = krn.load_program("laplacian")
    gp = krn.differentiate(lap, "normRes1DLaplacianSQ", ("x", "b"))
    rng = np.random.default_rng(4)
    for n, extra in ((1, 3), (1000, 1), (5000, 777)):
        x, b = rng.normal(size=n), rng.normal(size=n + extra)
        want = {"x": x.copy(), "b": b.copy(), "_d_x": np.zeros(n + extra), "_d_b": np.zeros(n + 2 * extra)}
        interp.run(gp, "normRes1DLaplacianSQ_grad", want)
        for lazy in (True, False):
            got = {"x": ViewStorage.from_values("x", x), "b": ViewStorage.from_values("b", b)}
            if lazy:
                got["_d_x"] = ViewStorage.zeros("_d_x", (n + extra,))
                got["_d_b"] = ViewStorage.zeros("_d_b", (n + 2 * extra,))
            else:
                got["_d_x"] = ViewStorage.from_values("_d_x", np.zeros(n + extra))
                got["_d_b"] = ViewStorage.from_values("_d_b", np.zeros(n + 2 * extra))
            # poison the pool: a freshly allocated buffer must not be mistaken for zeros
            junk = ViewStorage.from_values("junk", np.full(n + 2 * extra, np.nan))
            junk.device_ptr(krn.Device.get())
            del junk
            krn.execute(gp, "normRes1DLaplacianSQ_grad", got)
            for k in want:
                assert_bits(got[k].buffer, want[k], f"n={n} lazy={lazy} {k}")


@pytest.mark.parametrize("fuse_neighbours", [True, False])
@pytest.mark.parametrize("n", [1, 5, 130, 1030, 70_001])
def test_neighbour_registers_of_a_view_that_is_still_lazily_zero(n, fuse_neighbours):
    """a local nobody has written is not allocated; a tile kernel that holds its stencil neighbours in
    registers still reads it through bounds-checked loads on the first and last steps of the range
    (found by the random-program test: the pointer must not be null)"""
    from oracle import interp

    src = """fn f(a: view<f64,1>) -> f64 {
        let t1: view<f64,1> = view("t1", extent(a, 0));
        let t2: view<f64,1> = view("t2", extent(a, 0));
        parallel_for i in 0..extent(a, 0) {
            t2(i) = t1(i) + a(i);
            if (i != 0) { t2(i) += 2.0 * t1(i - 1) + a(i - 1); }
            if (i != extent(a, 0) - 1) { t2(i) -= 0.125 * t1(i + 1); }
        }
        r = parallel_sum(t2);
        return r; }"""
    p = parse(src)
    a = np.random.default_rng(n).normal(size=n)
    want = {"a": a.copy()}
    wv = interp.run(p, "f", want)
    got = {"a": ViewStorage.from_values("a", a)}
    gv = krn.execute(p, "f", got, ExecutionConfig(policy="compiled", fuse_neighbours=fuse_neighbours)).value
    assert_bits(gv, wv, "value")
