"""GPU parity, execution semantics: the behaviours the reference pins in its
tests/test_runtime.py (cited per test), exercised through ``execute`` on the
device, plus the oracle on the same program where a value is not pinned."""

import math

import numpy as np
import pytest

import paper_2507_13204_b200 as krn
from paper_2507_13204_b200 import ExecutionConfig, NonFiniteDetected, OutOfBounds, ShapeMismatch, ViewStorage, parse
from conftest import assert_bits

pytestmark = pytest.mark.gpu


def run(program, fn, inputs, **cfg):
    return krn.execute(program, fn, inputs, ExecutionConfig(**cfg) if cfg else None)


def vec(name, values):
    return ViewStorage.from_values(name, np.asarray(values, dtype=np.float64))


def test_views_have_reference_semantics():
    """test_runtime.py:47-51"""
    lap = krn.load_program("laplacian")
    x, b = vec("x", [1.0, 1.0, 1.0]), vec("b", [0.0, 0.0, 0.0])
    assert run(lap, "normRes1DLaplacianSQ", {"x": x, "b": b}, policy="statements").value == 18.0
    assert x.buffer.tolist() == [3.0, 3.0, 3.0] and b.buffer.tolist() == [0.0, 0.0, 0.0]


def test_raw_arrays_are_wrapped_and_written_back():
    """runtime.py:495-497: raw arrays become ViewStorage inside the caller's dict"""
    lap = krn.load_program("laplacian")
    inputs = {"x": np.ones(3), "b": np.zeros(3)}
    run(lap, "normRes1DLaplacianSQ", inputs)
    assert isinstance(inputs["x"], ViewStorage) and inputs["x"].buffer.tolist() == [3.0, 3.0, 3.0]


def test_copy_is_independent_on_device():
    """test_runtime.py:54-58, with the View resident in HBM"""
    a = vec("a", [1.0, 2.0])
    a.device_ptr(krn.Device.get(), write=False)
    c = a.copy()
    c.buffer[0] = 9.0
    assert a.buffer[0] == 1.0 and c.buffer.tolist() == [9.0, 2.0]


def test_gather_accumulates_into_preset_scalar():
    """test_runtime.py:61-69"""
    src = "fn f(v: view<f64, 1>) -> f64 { let s: f64 = 2.0; s = parallel_sum(v); return s; }"
    assert run(parse(src), "f", {"v": vec("v", [1.0, 2.0, 3.0])}).value == 8.0


def test_broadcast_and_elementwise_accumulate():
    """test_runtime.py:72-82"""
    src = """fn f(v: view<f64, 1>, w: view<f64, 1>) -> f64 {
        parallel_sum(w, 1.5); parallel_sum(w, v); return w(0); }"""
    w = vec("w", [10.0, 10.0, 10.0])
    assert run(parse(src), "f", {"v": vec("v", [1.0, 2.0, 3.0]), "w": w}).value == 12.5
    assert w.buffer.tolist() == [12.5, 13.5, 14.5]


def test_deep_copy_forms():
    """test_runtime.py:85-98"""
    src = """fn f(a: view<f64, 1>, b: view<f64, 1>, c: f64) -> f64 {
        deep_copy(a, c); deep_copy(b, a); deep_copy(a, 0.0); return b(0); }"""
    a, b = vec("a", [1.0, 1.0]), vec("b", [0.0, 0.0])
    assert run(parse(src), "f", {"a": a, "b": b, "c": 7.0}).value == 7.0
    assert a.buffer.tolist() == [0.0, 0.0] and b.buffer.tolist() == [7.0, 7.0]


def test_counter_values_guards_and_extent_as_value():
    """counter read as a value is float(i) (runtime.py:245); extent as value (250).
    (The reference's sequential-scan test, test_runtime.py:101-115, relies on
    iteration order and is a data race on any parallel executor.)"""
    src = """fn f(v: view<f64, 1>) -> f64 {
        parallel_for i in 0..extent(v, 0) {
            v(i) = v(i) + i * extent(v, 0);
            if (i >= 2) { v(i) -= 0.5; }
            if (i == extent(v, 0) - 1) { v(i) = -v(i); }
        }
        return v(extent(v, 0) - 1); }"""
    v = vec("v", [1.0, 1.0, 1.0, 1.0])
    assert run(parse(src), "f", {"v": v}).value == -(1.0 + 12.0 - 0.5)
    assert v.buffer.tolist() == [1.0, 5.0, 8.5, -12.5]


def test_rank2_execution():
    """test_runtime.py:118-129"""
    m = ViewStorage.from_values("m", np.arange(6, dtype=np.float64).reshape(2, 3) + 1.0)
    r = vec("r", [2.0, 0.5])
    value = run(krn.load_program("rowscale_rank2"), "rowScaleEnergy", {"m": m, "r": r}).value
    expected = sum(s * (row[0] + row[1] + row[2] * row[2]) for row, s in zip([[1, 2, 3], [4, 5, 6]], [2.0, 0.5]))
    assert value == pytest.approx(expected, rel=1e-15)


def test_atomic_adds_are_exact():
    """test_runtime.py:150-164: 4000 contributions to one location"""
    src = """fn f(v: view<f64, 1>, acc: view<f64, 1>) -> f64 {
        parallel_for i in 0..extent(v, 0) { atomic_add(acc(0), 1.0); } return acc(0); }"""
    acc = vec("acc", [0.0])
    assert run(parse(src), "f", {"v": ViewStorage.zeros("v", (4000,)), "acc": acc}, threads=8).value == 4000.0


def test_atomics_are_deferred_to_the_kernel_boundary():
    """runtime.py:441-445: reads inside the kernel never see that kernel's atomic adds"""
    from oracle import interp

    src = """fn f(x: view<f64, 1>, idx: view<f64, 1>, out: view<f64, 1>) {
        parallel_for i in 0..extent(idx, 0) {
            atomic_add(x(idx(i)), 1.0);
            out(i) = x(idx(i));
        } }"""
    p = parse(src)
    idx = np.array([0.0, 0.0, 1.0, 2.0, 2.0, 2.0])
    want = {"x": np.array([10.0, 20.0, 30.0]), "idx": idx.copy(), "out": np.zeros(6)}
    interp.run(p, "f", want)
    got = {"x": vec("x", [10.0, 20.0, 30.0]), "idx": vec("idx", idx), "out": ViewStorage.zeros("out", (6,))}
    run(p, "f", got)
    assert got["out"].buffer.tolist() == want["out"].tolist() == [10.0, 10.0, 20.0, 30.0, 30.0, 30.0]
    assert got["x"].buffer.tolist() == want["x"].tolist() == [12.0, 21.0, 33.0]


def test_indirect_index_truncates_toward_zero():
    """runtime.py:335: int(value)"""
    src = """fn f(x: view<f64, 1>, idx: view<f64, 1>, out: view<f64, 1>) {
        parallel_for i in 0..extent(idx, 0) { out(i) = x(idx(i)); } }"""
    out = ViewStorage.zeros("out", (4,))
    run(parse(src), "f", {"x": vec("x", [5.0, 6.0, 7.0]), "idx": vec("idx", [0.9, 1.5, 2.999, -0.7]), "out": out})
    assert out.buffer.tolist() == [5.0, 6.0, 7.0, 5.0]
    with pytest.raises(ValueError):
        run(parse(src), "f", {"x": vec("x", [5.0]), "idx": vec("idx", [float("nan")]), "out": ViewStorage.zeros("out", (1,))})
    with pytest.raises(OverflowError):
        run(parse(src), "f", {"x": vec("x", [5.0]), "idx": vec("idx", [float("inf")]), "out": ViewStorage.zeros("out", (1,))})


def test_results_do_not_depend_on_threads_field():
    """test_runtime.py:167-185 (threads is accepted and ignored on the GPU)"""
    lap = krn.load_program("laplacian")
    gp = krn.differentiate(lap, "normRes1DLaplacianSQ", ("x", "b"))
    rng = np.random.default_rng(7)
    x0, b0 = rng.normal(size=257), rng.normal(size=257)
    outs = []
    for threads in (1, 2, 8):
        call = {"x": vec("x", x0), "b": vec("b", b0), "_d_x": ViewStorage.zeros("_d_x", (257,)),
                "_d_b": ViewStorage.zeros("_d_b", (257,))}
        run(gp, "normRes1DLaplacianSQ_grad", call, threads=threads)
        outs.append((call["_d_x"].buffer.copy(), call["_d_b"].buffer.copy()))
    for dx, db in outs[1:]:
        assert np.array_equal(dx, outs[0][0]) and np.array_equal(db, outs[0][1])


def test_out_of_bounds_read_and_write():
    """test_runtime.py:309-319 and the message format of runtime.py:302-305, 315-318"""
    src = "fn f(v: view<f64, 1>) -> f64 {\n parallel_for i in 0..extent(v, 0) {\n v(i) = v(i + 1);\n }\n return v(0);\n}"
    with pytest.raises(OutOfBounds, match=r"line 3: v\(2\) outside extent 2"):
        run(parse(src), "f", {"v": vec("v", [1.0, 2.0])})
    src2 = "fn f(m: view<f64, 2>) {\n parallel_for i in 0..extent(m, 0) {\n m(i, 3) = 1.0;\n }\n}"
    with pytest.raises(OutOfBounds, match=r"line 3: m\(\d, 3\) outside extents 2x3"):
        run(parse(src2), "f", {"m": ViewStorage.from_values("m", np.zeros((2, 3)))})
    # the headline program with a short b takes the statement path and reports like the reference
    lap = krn.load_program("laplacian")
    with pytest.raises(OutOfBounds, match=r"b\(2\) outside extent 2"):
        run(lap, "normRes1DLaplacianSQ", {"x": vec("x", [1.0, 1.0, 1.0]), "b": vec("b", [0.0, 0.0])})


def test_binding_errors():
    """test_runtime.py:322-349"""
    lap = krn.load_program("laplacian")
    with pytest.raises(ShapeMismatch, match="missing"):
        run(lap, "normRes1DLaplacianSQ", {"x": vec("x", [1.0])})
    with pytest.raises(ShapeMismatch, match="rank"):
        run(lap, "normRes1DLaplacianSQ", {"x": 3.0, "b": vec("b", [0.0])})
    with pytest.raises(KeyError):
        run(lap, "nope", {})
    src = "fn f(v: view<f64, 1>, w: view<f64, 1>) -> f64 { parallel_sum(w, v); return w(0); }"
    with pytest.raises(ShapeMismatch):
        run(parse(src), "f", {"v": vec("v", [1.0, 2.0, 3.0]), "w": vec("w", [0.0])})
    src = "fn f(v: view<f64, 1>, w: view<f64, 1>) { deep_copy(w, v); }"
    with pytest.raises(ShapeMismatch, match="deep_copy"):
        run(parse(src), "f", {"v": vec("v", [1.0, 2.0, 3.0]), "w": vec("w", [0.0])})


def test_division_by_zero_follows_ieee_and_check_finite():
    """test_runtime.py:352-375"""
    src = """fn f(v: view<f64, 1>) -> f64 {
        parallel_for i in 0..extent(v, 0) { v(i) = 1.0 / v(i); } return parallel_sum(v); }"""
    assert run(parse(src), "f", {"v": vec("v", [0.0, 1.0])}).value == math.inf
    with pytest.raises(NonFiniteDetected, match="'v'"):
        run(parse(src), "f", {"v": vec("v", [0.0, 1.0])}, check_finite=True)
    # finite data passes with the guard on, fused program included (falls back to statements)
    lap = krn.load_program("laplacian")
    assert run(lap, "normRes1DLaplacianSQ", {"x": np.ones(3), "b": np.zeros(3)}, check_finite=True).value == 18.0


def test_pairwise_sum_matches_reference_tree(pairwise_golden):
    """test_runtime.py:382-408 plus the stored reference results, bit for bit"""
    for n, want in zip(pairwise_golden["lengths"], pairwise_golden["sums"]):
        n = int(n)
        v = np.random.default_rng(n).normal(size=n) * 10.0 ** np.random.default_rng(n + 1).integers(-3, 4, size=n)
        assert_bits(krn.pairwise_sum(v), want, f"n={n}")
    rng = np.random.default_rng(3)
    values = rng.normal(size=1023) * 10.0 ** rng.integers(-6, 6, size=1023)
    assert krn.pairwise_sum(values) == pytest.approx(math.fsum(values), rel=1e-12)


def test_gather_signed_zero_and_large_tree():
    from oracle import cport

    src = "fn f(v: view<f64, 1>) -> f64 { return parallel_sum(v); }"
    p = parse(src)
    for n in (1, 2, 3, 4, 5, 8, 12, 16, 1024, 1025, 2048, 4096 + 1):
        v = np.full(n, -0.0)
        got = run(p, "f", {"v": vec("v", v)}).value
        assert_bits(got, 0.0 + cport.pairwise_sum(v), f"-0.0 n={n}")
    for n in ((1 << 20) + 1, (1 << 21) + 8192 * 3 + 77, 5_000_003):
        v = np.random.default_rng(n).normal(size=n)
        assert_bits(run(p, "f", {"v": vec("v", v)}).value, 0.0 + cport.pairwise_sum(v), f"n={n}")


def test_empty_views():
    src = """fn f(v: view<f64, 1>) -> f64 {
        let w: view<f64, 1> = view("w", extent(v, 0));
        parallel_for i in 0..extent(v, 0) { w(i) = v(i) * v(i); }
        return parallel_sum(w); }"""
    assert run(parse(src), "f", {"v": ViewStorage.zeros("v", (0,))}).value == 0.0
    lap = krn.load_program("laplacian")
    assert run(lap, "normRes1DLaplacianSQ", {"x": np.zeros(0), "b": np.zeros(0)}).value == 0.0


def test_function_scope_element_statements():
    """runtime.py:536-550: scalar lets/assignments, element writes, guards and atomic_add at function scope"""
    from oracle import interp

    src = """fn f(v: view<f64, 1>, c: f64) -> f64 {
        let a: f64 = c * c + v(0);
        a += 2.0;
        a -= v(1) / 4.0;
        v(2) = a;
        v(2) -= 1.0;
        atomic_add(v(0), a);
        if (extent(v, 0) > 2) { v(1) += 0.5; }
        if (extent(v, 0) > 5) { v(1) += 100.0; }
        return a * v(1); }"""
    p = parse(src)
    want = {"v": np.array([1.0, 2.0, 3.0]), "c": 1.5}
    wv = interp.run(p, "f", want)
    got = {"v": vec("v", [1.0, 2.0, 3.0]), "c": 1.5}
    assert_bits(run(p, "f", got).value, wv, "value")
    assert_bits(got["v"].buffer, want["v"], "v")


def test_ad_gradient_and_finite_differences_agree():
    """criterion 3 (test_acceptance.py:132-157) on two programs, on the device"""
    for stem, fn_name in (("safe_divide", "normalizedEnergy"), ("mean_shift", "shiftedEnergy")):
        prog = krn.load_program(stem)
        rng = np.random.default_rng(1)
        inputs = {"v": rng.normal(size=8)}
        ad = krn.ad_gradient(prog, fn_name, inputs, ("v",))
        fd = krn.finite_difference_gradient(prog, fn_name, inputs, ("v",))
        assert krn.check_gradient(ad["v"], fd["v"], atol=1e-9, rtol=1e-5).passed


def test_bench_ratio_runs():
    """test_verify.py:247-262"""
    lap = krn.load_program("laplacian")
    for policy in ("fused", "statements"):
        r = krn.bench_ratio(lap, "normRes1DLaplacianSQ", 10_000, ExecutionConfig(policy=policy), reps=3)
        assert r.n == 10_000 and r.reps == 3 and r.primal_s > 0 and r.grad_s > 0
        assert r.gradient_entries == 20_000 and math.isfinite(r.ratio)
    with pytest.raises(ValueError):
        krn.bench_ratio(lap, "normRes1DLaplacianSQ", 100, reps=2)


def test_compiled_modules_are_cached_on_disk(tmp_path, monkeypatch):
    """krn_module_compile keeps the cubin under $KRN_CACHE_DIR keyed by source/options/compiler; a
    damaged file is recompiled over, an empty KRN_CACHE_DIR switches the cache off"""
    import ctypes as C

    from paper_2507_13204_b200 import _cabi

    dev = krn.Device.get()
    src = ('#include "krn_prelude.cuh"\nextern "C" __global__ void cache_probe_%d(double *p) { p[0] = %d.0; }\n'
           % (id(tmp_path) % 100000, id(tmp_path) % 977))

    def compile_once():
        h = C.c_void_p()
        _cabi.check(dev.lib.krn_module_compile(dev.h, src.encode(), C.byref(h)))
        _cabi.check(dev.lib.krn_module_destroy(h))

    monkeypatch.setenv("KRN_CACHE_DIR", str(tmp_path / "cache"))
    compile_once()
    files = list((tmp_path / "cache").iterdir())
    assert len(files) == 1 and files[0].suffix == ".cubin" and files[0].stat().st_size > 0
    stamp = files[0].stat().st_mtime_ns
    compile_once()                                  # served from the cache: file untouched
    assert files[0].stat().st_mtime_ns == stamp and len(list((tmp_path / "cache").iterdir())) == 1
    files[0].write_bytes(b"not a cubin")            # damaged image: recompiled and replaced
    compile_once()
    assert files[0].stat().st_size > 100
    monkeypatch.setenv("KRN_CACHE_DIR", "")
    other = tmp_path / "cache2"
    compile_once()
    assert not other.exists()


def test_order_dependent_kernels_run_in_iteration_order():
    """The reference at threads=1 (its default) runs iterations 0..n-1 in order and its tests rely
    on it (tests/test_runtime.py:101-115: a scan completes).  Kernels whose index expressions allow
    two iterations to meet at a plainly written location are checked by the tag replay and, when
    they really do, run on one thread; otherwise in parallel.  Oracle = the sequential interpreter."""
    import paper_2507_13204_b200 as krn
    from oracle import interp

    scan = """fn f(v: view<f64, 1>) -> f64 {
        parallel_for i in 0..extent(v, 0) { if (i != 0) { v(i) = v(i - 1) + i; } }
        return v(extent(v, 0) - 1); }"""
    v = krn.ViewStorage.from_values("v", [0.0, 0.0, 0.0])
    assert krn.execute(krn.parse(scan), "f", {"v": v}).value == 3.0      # the reference's own case
    rng = np.random.default_rng(8)
    cases = [
        (scan, {"v": rng.normal(size=3000)}),
        ("""fn f(v: view<f64,1>, acc: view<f64,1>) -> f64 {
            parallel_for i in 0..extent(v,0) { acc(0) = v(i); acc(1) += v(i) * acc(0); } return acc(1); }""",
         {"v": rng.normal(size=777), "acc": np.zeros(2)}),
        # scatter through an index View: a permutation (parallel) and a map with repeats (in order)
        ("""fn f(v: view<f64,1>, idx: view<f64,1>, out: view<f64,1>) -> f64 {
            parallel_for i in 0..extent(idx,0) { out(idx(i)) = v(i) + out(idx(i)); } return out(0); }""",
         {"v": rng.normal(size=5000), "idx": rng.permutation(5000).astype(np.float64), "out": rng.normal(size=5000)}),
        ("""fn f(v: view<f64,1>, idx: view<f64,1>, out: view<f64,1>) -> f64 {
            parallel_for i in 0..extent(idx,0) { out(idx(i)) = v(i) + 0.5 * out(idx(i)); atomic_add(out(i), 1.0); }
            return out(0); }""",
         {"v": rng.normal(size=5000), "idx": rng.integers(0, 50, size=5000).astype(np.float64),
          "out": rng.normal(size=5000)}),
    ]
    for policy in ("fused", "compiled", "statements"):
        for src, data in cases:
            want = {k: a.copy() for k, a in data.items()}
            fo = interp.run(krn.parse(src), "f", want)
            call = {k: krn.ViewStorage.from_values(k, a) for k, a in data.items()}
            f = krn.execute(krn.parse(src), "f", call, krn.ExecutionConfig(policy=policy)).value
            assert f == fo, (policy, src)
            for k in data:
                assert np.array_equal(call[k].buffer, want[k]), (policy, k, src)
