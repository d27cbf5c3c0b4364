"""GPU parity of check_finite on the FUSED path: the generated kernels test the values their
statements leave behind and the reference's checks (after every kernel / bulk statement the first
non-finite View in declaration order; after every gather its scalar; the return value:
/root/reference/pkg/src/krn/runtime.py:624, 641, 651, 665, 669-676) are replayed from the recorded
flags.  Bar: the same exception class and message as the CPU oracle, for non-finite values that
come in with the inputs, appear in the middle of a fused kernel, or only in a reduction - and
identical results, still fused, when nothing is wrong."""

import numpy as np
import pytest

import paper_2507_13204_b200 as krn
from paper_2507_13204_b200 import ExecutionConfig, NonFiniteDetected, ViewStorage, parse
from conftest import CORPUS, assert_bits

pytestmark = pytest.mark.gpu


def _outcome(run):
    try:
        return ("ok", run())
    except ArithmeticError as e:  # the oracle has its own NonFiniteDetected class: compare by name
        assert type(e).__name__ == "NonFiniteDetected"
        return ("NonFiniteDetected", str(e))


def _compare(program, fn_name, data, policy="compiled", expect_launches=None):
    from oracle import interp

    want_in = {k: (np.array(v) if isinstance(v, np.ndarray) else v) for k, v in data.items()}
    want = _outcome(lambda: interp.run(program, fn_name, want_in, check_finite=True))
    got_in = {k: (ViewStorage.from_values(k, v) if isinstance(v, np.ndarray) else v) for k, v in data.items()}
    dev = krn.Device.get()
    before = dev.launches()
    got = _outcome(lambda: krn.execute(program, fn_name, got_in, ExecutionConfig(policy=policy, check_finite=True)).value)
    launches = dev.launches() - before
    if want[0] == "ok":
        assert got[0] == "ok", (got, want)
        if want[1] is None:
            assert got[1] is None
        else:
            assert_bits(got[1], want[1], "value")
        for k, v in got_in.items():
            if isinstance(v, ViewStorage):
                assert_bits(v.buffer, want_in[k], k)
    else:
        assert got == want, (got, want)
    if expect_launches is not None:
        assert launches <= expect_launches, launches
    return want


def _inputs(fn, n, rng):
    data = {}
    for p in fn.params:
        if not p.is_view:
            data[p.name] = 0.75
        elif p.name == "idx":
            data[p.name] = rng.integers(0, n, size=n).astype(np.float64)
        elif p.type.rank == 2:
            data[p.name] = rng.normal(size=(n, 3))
        else:
            data[p.name] = rng.normal(size=n)
    return data


@pytest.mark.parametrize("stem", CORPUS)
def test_corpus_with_poisoned_inputs(stem):
    """every corpus program and its gradient: clean inputs pass (fused), and NaN / Inf placed in each
    View parameter in turn (first row, a middle row, last row) raise what the oracle raises"""
    prog = krn.load_program(stem)
    fn = prog.functions[0]
    wrt = tuple(p.name for p in fn.params if p.is_view and p.name != "idx")
    gp = krn.differentiate(prog, fn.name, wrt)
    gfn = gp.functions[-1]
    rng = np.random.default_rng(5)
    for n in (7, 1300):
        data = _inputs(fn, n, rng)
        gdata = dict(data)
        for sp, w in zip(gfn.params[len(fn.params):], wrt):
            gdata[sp.name] = rng.normal(size=np.shape(data[w]))
        for program, name, d in ((prog, fn.name, data), (gp, gfn.name, gdata)):
            assert _compare(program, name, d)[0] == "ok"
            for view in [k for k, v in d.items() if isinstance(v, np.ndarray) and k != "idx"]:
                for pos, poison in ((0, np.nan), (n // 2, np.inf), (n - 1, -np.inf)):
                    bad = {k: (np.array(v) if isinstance(v, np.ndarray) else v) for k, v in d.items()}
                    bad[view].reshape(-1)[pos * (bad[view].size // n)] = poison
                    _compare(program, name, bad)


def test_overflow_in_the_middle_of_a_fused_kernel_names_the_reference_view():
    lap = krn.load_program("laplacian")
    n = 5000
    x, b = np.full(n, 1.0), np.zeros(n)
    # 3x overflows nowhere, y = 2*3x - ... is finite, y*y overflows: the first bad View is y2 (after the
    # second kernel), not the return value
    x[1234] = 1e160
    assert _compare(lap, "normRes1DLaplacianSQ", {"x": x, "b": b}, expect_launches=3) == \
        ("NonFiniteDetected", "non-finite value in view 'y2'")
    # the scale kernel itself overflows: x, after the FIRST kernel
    x[:] = 1.0
    x[7] = 1e308
    assert _compare(lap, "normRes1DLaplacianSQ", {"x": x, "b": b}) == \
        ("NonFiniteDetected", "non-finite value in view 'x'")
    # every element finite, only the SUM overflows: the gather's scalar
    x[:] = 2.6e152 * (-1.0) ** np.arange(n)  # y = 4 * 3x in the interior, y*y ~ 1e307, 5000 of them
    want = _compare(lap, "normRes1DLaplacianSQ", {"x": x, "b": b})
    assert want[0] == "NonFiniteDetected" and want[1].startswith("non-finite scalar")


def test_dead_forward_sum_is_still_checked_in_the_gradient():
    """the verbatim forward `sum = parallel_sum(y2)` inside the gradient is dead, but the reference
    checks it: a gradient whose forward sum overflows raises although every View stays finite"""
    lap = krn.load_program("laplacian")
    gp = krn.differentiate(lap, "normRes1DLaplacianSQ", ("x", "b"))
    n = 4096
    data = {"x": 2.6e152 * (-1.0) ** np.arange(n), "b": np.zeros(n), "_d_x": np.zeros(n), "_d_b": np.zeros(n)}
    want = _compare(gp, "normRes1DLaplacianSQ_grad", data)
    assert want[0] == "NonFiniteDetected" and want[1].startswith("non-finite scalar")


def test_views_longer_than_the_range_and_output_parameters():
    """an output parameter the first statement overwrites may come in full of NaN; one that a LATER
    statement overwrites may not; rows beyond the range are checked too (statement path)"""
    src = """fn f(x: view<f64, 1>, y: view<f64, 1>, z: view<f64, 1>) -> f64 {
        parallel_for i in 0..extent(x, 0) { y(i) = 2.0 * x(i); }
        parallel_for i in 0..extent(x, 0) { z(i) = y(i) + 1.0; }
        s = parallel_sum(z);
        return s; }"""
    p = parse(src)
    n = 3000
    x = np.linspace(-1.0, 1.0, n)
    nan = np.full(n, np.nan)
    assert _compare(p, "f", {"x": x, "y": nan, "z": np.zeros(n)})[0] == "ok"
    assert _compare(p, "f", {"x": x, "y": np.zeros(n), "z": nan}) == \
        ("NonFiniteDetected", "non-finite value in view 'z'")
    longer = np.zeros(n + 5)
    longer[-1] = np.inf
    assert _compare(p, "f", {"x": x, "y": longer, "z": np.zeros(n)}) == \
        ("NonFiniteDetected", "non-finite value in view 'y'")


def test_cost_of_the_fused_check_is_small():
    """the tests themselves are a few ALU instructions per value; what the check costs is the forward
    reduction the reference checks and an unchecked plan drops as dead (one more launch, Views it
    reads materialised): well under 2x the unchecked time, several times faster than checking
    statement by statement"""
    import torch

    prog = krn.load_program("inplace_axpy")
    fn = prog.functions[0]
    wrt = tuple(p.name for p in fn.params if p.is_view)
    gp = krn.differentiate(prog, fn.name, wrt)
    gfn = gp.functions[-1]
    n = 1 << 25
    rng = np.random.default_rng(0)
    base = {p.name: (ViewStorage.from_values(p.name, rng.normal(size=n)) if p.is_view else 0.75) for p in fn.params}
    dev = krn.Device.get()
    for v in base.values():
        if isinstance(v, ViewStorage):
            v.device_ptr(dev, write=False)
    times = {}
    for check in (False, True, "statements"):
        best = 1e9
        for rep in range(5):
            call = {k: (v.copy() if isinstance(v, ViewStorage) else v) for k, v in base.items()}
            for sp, w in zip(gfn.params[len(fn.params):], wrt):
                call[sp.name] = ViewStorage.zeros(sp.name, (n,))
            dev.sync()
            e0, e1 = dev.event(), dev.event()
            dev.record(e0)
            krn.execute(gp, gfn.name, call, ExecutionConfig(policy="statements" if check == "statements" else "compiled",
                                                            check_finite=bool(check)))
            dev.record(e1)
            best = min(best, dev.elapsed_ms(e0, e1))
        times[check] = best
    assert times[True] <= 1.8 * times[False] + 0.05, times
    assert times[True] <= 0.5 * times["statements"], times
