"""GPU parity, accumulation policies for non-injective atomic_add targets
(hardware reductions, warp-aggregated, shared-memory privatised) under every
execution policy, on index maps from uniform to fully colliding.  Bar: relative
1e-12 against the CPU oracle (atomic order is not deterministic), and EXACT where
every partial sum is exactly representable."""

import numpy as np
import pytest

import paper_2507_13204_b200 as krn
from paper_2507_13204_b200 import ExecutionConfig, ViewStorage, parse

pytestmark = pytest.mark.gpu


def _index_maps(n, rows, rng):
    return {
        "uniform": rng.integers(0, rows, size=n),
        "all_zero": np.zeros(n, dtype=np.int64),
        "clustered": (np.arange(n) // 8) % rows,
        "hot_spot": np.where(rng.random(n) < 0.9, 3 % rows, rng.integers(0, rows, size=n)),
    }


@pytest.mark.parametrize("apol", ["auto", "ordered", "red", "warp", "smem", "lead"])
@pytest.mark.parametrize("policy", ["compiled", "statements"])
def test_gather_indirect_gradient_all_policies(policy, apol):
    from oracle import interp

    prog = krn.load_program("gather_indirect")
    gp = krn.differentiate(prog, "gatherSquares", ("x",))
    rng = np.random.default_rng(11)
    for n, rows in ((257, 257), (5000, 64), (5000, 5000), (3000, 6144), (2000, 7000)):
        x = rng.normal(size=rows)
        for label, idx in _index_maps(n, rows, rng).items():
            want = {"x": x.copy(), "idx": idx.astype(np.float64), "_d_x": np.zeros(rows)}
            interp.run(gp, "gatherSquares_grad", want)
            got = {"x": ViewStorage.from_values("x", x), "idx": ViewStorage.from_values("idx", idx.astype(np.float64)),
                   "_d_x": ViewStorage.zeros("_d_x", (rows,))}
            krn.execute(gp, "gatherSquares_grad", got, ExecutionConfig(policy=policy, atomic_policy=apol))
            if apol in ("auto", "ordered"):  # the reference's order: same bits
                assert np.array_equal(got["_d_x"].buffer, want["_d_x"]), (policy, apol, n, rows, label)
            err = np.abs(got["_d_x"].buffer - want["_d_x"])
            assert np.all(err <= 1e-12 * np.abs(want["_d_x"])), (policy, apol, n, rows, label, err.max())


@pytest.mark.parametrize("apol", ["ordered", "red", "warp", "smem", "lead"])
def test_integer_contributions_are_exact(apol):
    """reference tests/test_runtime.py:150-164, generalised: sums of small integers are exact in
    any order, so every policy must return the same bits"""
    src = """fn f(idx: view<f64, 1>, acc: view<f64, 1>) {
        parallel_for i in 0..extent(idx, 0) { atomic_add(acc(idx(i)), 1.0); atomic_add(acc(0), 2.0); } }"""
    p = parse(src)
    rng = np.random.default_rng(5)
    n, rows = 200_000, 97
    idx = rng.integers(0, rows, size=n)
    acc = ViewStorage.from_values("acc", np.full(rows, 0.5))
    krn.execute(p, "f", {"idx": ViewStorage.from_values("idx", idx.astype(np.float64)), "acc": acc},
                ExecutionConfig(atomic_policy=apol))
    want = 0.5 + np.bincount(idx, minlength=rows).astype(np.float64)
    want[0] += 2.0 * n
    assert np.array_equal(acc.buffer, want)


def test_rank2_target_privatised():
    from oracle import interp

    src = """fn f(idx: view<f64, 1>, v: view<f64, 1>, m: view<f64, 2>) {
        parallel_for i in 0..extent(idx, 0) { atomic_add(m(idx(i), 1), v(i)); atomic_add(m(idx(i), 2), -v(i)); } }"""
    p = parse(src)
    rng = np.random.default_rng(2)
    n, rows = 4000, 50
    idx, v = rng.integers(0, rows, size=n).astype(np.float64), rng.normal(size=n)
    want = {"idx": idx.copy(), "v": v.copy(), "m": np.ones((rows, 3))}
    interp.run(p, "f", want)
    for apol in ("red", "smem", "warp", "ordered"):
        got = {"idx": ViewStorage.from_values("idx", idx), "v": ViewStorage.from_values("v", v),
               "m": ViewStorage.from_values("m", np.ones((rows, 3)))}
        krn.execute(p, "f", got, ExecutionConfig(atomic_policy=apol))
        assert np.allclose(got["m"].buffer, want["m"], rtol=1e-12, atol=1e-12), apol
        if apol == "ordered":
            assert np.array_equal(got["m"].buffer, want["m"])


def test_privatised_rows_next_to_the_kernels_own_shared_memory():
    """a scatter into exactly the largest privatisable target (6144 rows = 48 KB) fused with a
    reduction (static shared memory for the block tree) and with a neighbour window: the host must
    not ask for more shared memory than a launch gets"""
    from oracle import interp

    src = """fn f(a: view<f64, 1>, idx: view<f64, 1>, acc: view<f64, 1>) -> f64 {
        let t: view<f64, 1> = view("t", extent(a, 0));
        parallel_for i in 0..extent(a, 0) { a(i) = 2.0 * a(i); }
        parallel_for i in 0..extent(a, 0) {
            t(i) = a(i);
            if (i != 0) { t(i) += a(i - 1); }
            atomic_add(acc(idx(i)), 1.0);
        }
        s = parallel_sum(t);
        return s; }"""
    p = parse(src)
    n, rows = 40_000, 6144
    rng = np.random.default_rng(3)
    a, idx = rng.normal(size=n), rng.integers(0, rows, size=n).astype(np.float64)
    want = {"a": a.copy(), "idx": idx.copy(), "acc": np.zeros(rows)}
    wv = interp.run(p, "f", want)
    for apol, det in (("auto", True), ("auto", False), ("smem", True)):
        got = {"a": ViewStorage.from_values("a", a), "idx": ViewStorage.from_values("idx", idx),
               "acc": ViewStorage.zeros("acc", (rows,))}
        v = krn.execute(p, "f", got, ExecutionConfig(policy="compiled", atomic_policy=apol,
                                                     deterministic_reduction=det)).value
        assert v == wv
        assert np.array_equal(got["acc"].buffer, want["acc"]) and np.array_equal(got["a"].buffer, want["a"])
