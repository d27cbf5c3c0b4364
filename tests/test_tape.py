"""CPU tier: store-instead-of-reject (lang/tape.py, differentiate(tape=True)).  The reference
refuses these functions (NotFeasible), so there is no reference gradient to compare with: the
taped gradient is checked against central finite differences of the ORIGINAL primal evaluated by
the oracle, the rewritten forward part against the original primal bit for bit, and the default
(tape=False) must keep refusing exactly like the reference."""

import numpy as np
import pytest

import paper_2507_13204_b200 as krn
from conftest import assert_bits

CASES = {
    # self-overwrite, kernel-local scalar, neighbour read of a View overwritten by a later kernel
    "overwrites": (krn.load_program("taped_overwrites"), "tapedOverwrites", ("x", "a")),
    # quotient + product of Views that a later kernel rescales in place
    "quotient": (krn.parse("""fn f(u: view<f64, 1>, v: view<f64, 1>) -> f64 {
        let w: view<f64, 1> = view("w", extent(u, 0));
        parallel_for i in 0..extent(u, 0) { w(i) = u(i) / (2.0 + v(i) * v(i)); }
        parallel_for i in 0..extent(u, 0) { u(i) = u(i) * w(i); v(i) = v(i) - u(i); }
        parallel_for i in 0..extent(u, 0) { w(i) = w(i) * u(i) + v(i); }
        return parallel_sum(w); }"""), "f", ("u", "v")),
    # rank-2 rows, a column overwritten after use, function-scope scalar reused
    "rank2": (krn.parse("""fn f(m: view<f64, 2>, r: view<f64, 1>) -> f64 {
        let q: view<f64, 1> = view("q", extent(r, 0));
        parallel_for i in 0..extent(r, 0) { q(i) = m(i, 0) * m(i, 1) * r(i); }
        parallel_for i in 0..extent(r, 0) { m(i, 1) = m(i, 1) * m(i, 2); r(i) = r(i) * r(i); }
        parallel_for i in 0..extent(r, 0) { q(i) += m(i, 1) * r(i); }
        s = parallel_sum(q);
        return s; }"""), "f", ("m", "r")),
}


def _inputs(fn, n, rng):
    return {p.name: rng.uniform(0.5, 1.5, size=(n, 3) if p.type.rank == 2 else n) for p in fn.params if p.is_view}


@pytest.mark.parametrize("name", sorted(CASES))
def test_reference_behaviour_is_the_default(name):
    prog, fn, wrt = CASES[name]
    with pytest.raises(krn.NotFeasible, match="needed by the reverse pass but overwritten"):
        krn.differentiate(prog, fn, wrt)


@pytest.mark.parametrize("name", sorted(CASES))
def test_taped_gradient_against_finite_differences(name):
    from oracle import interp

    prog, fn_name, wrt = CASES[name]
    fn = prog.function(fn_name)
    gp = krn.differentiate(prog, fn_name, wrt, tape=True)
    gfn = gp.functions[-1]
    assert krn.validate(gp) == []
    krn.parse(krn.emit(gp))  # the emitted text is a well-formed program
    n = 6
    base = _inputs(fn, n, np.random.default_rng(3))

    def value(d):
        call = {k: v.copy() for k, v in d.items()}
        return interp.run(prog, fn_name, call), call

    v0, after = value(base)
    call = {k: v.copy() for k, v in base.items()}
    shadows = [p.name for p in gfn.params[len(fn.params):]]
    for s_, w in zip(shadows, wrt):
        call[s_] = np.zeros_like(base[w])
    interp.run(gp, gfn.name, call)
    # unlike a save/restore tape, the parameters still hold the forward results
    for k in base:
        assert_bits(call[k], after[k], f"{name}: {k} after the gradient call")
    h = 1e-6
    for s_, w in zip(shadows, wrt):
        fd = np.zeros(base[w].size)
        for k in range(fd.size):
            up, dn = {a: b.copy() for a, b in base.items()}, {a: b.copy() for a, b in base.items()}
            up[w].reshape(-1)[k] += h
            dn[w].reshape(-1)[k] -= h
            fd[k] = (value(up)[0] - value(dn)[0]) / (2 * h)
        got = call[s_].reshape(-1)
        assert np.all(np.abs(got - fd) <= 1e-6 * np.maximum(1.0, np.abs(fd))), (name, w, got, fd)


def test_snapshots_are_locals_that_are_never_rewritten():
    prog, fn_name, wrt = CASES["overwrites"]
    gp = krn.differentiate(prog, fn_name, wrt, tape=True)
    text = krn.emit(gp.functions[-1])
    assert "_tape_x(i) = x(i);" in text and "x(i) = _tape_x(i) * _tape_x(i);" in text
    assert "_tape_t(i) = t;" in text and "y(i) = _tape_t(i) * _tape_t(i);" in text
    assert "_tape_x2(i - 1) = x(i - 1);" in text           # neighbour read: snapshot at the same index
    assert "atomic_add(_d_x(i - 1)" in text                # ... and its adjoint is flagged like any other
    # a feasible function is left alone
    lap = krn.load_program("laplacian")
    a = krn.emit(krn.differentiate(lap, "normRes1DLaplacianSQ", ("x", "b")).functions[-1])
    b = krn.emit(krn.differentiate(lap, "normRes1DLaplacianSQ", ("x", "b"), tape=True).functions[-1])
    assert a == b


def test_what_cannot_be_snapshotted_still_raises():
    # the needed value is read through an index View that is itself overwritten in the same kernel
    p = krn.parse("""fn f(x: view<f64, 1>, idx: view<f64, 1>) -> f64 {
        let y: view<f64, 1> = view("y", extent(idx, 0));
        parallel_for i in 0..extent(idx, 0) { y(i) = x(idx(i)) * x(idx(i)); x(i) = 0.0; }
        return parallel_sum(y); }""")
    with pytest.raises(krn.NotFeasible):
        krn.differentiate(p, "f", ("x",), tape=True)


def test_random_programs_taped_gradient_against_finite_differences():
    """random programs the reference refuses (in-place updates of Views whose values an earlier
    statement's reversal needs): the taped gradient must agree with central differences of the
    ORIGINAL primal (oracle interpreter, n = 4)"""
    import warnings

    from hypothesis import HealthCheck, assume, given, settings, strategies as st

    from oracle import interp
    from test_gpu_random_programs import _inputs as fuzz_inputs, programs

    checked = [0]

    import os

    # the default run draws the same 120 programs every time; KRN_FUZZ=<n> explores n fresh ones
    @settings(max_examples=int(os.environ.get("KRN_FUZZ", "120")), deadline=None, suppress_health_check=list(HealthCheck),
              derandomize="KRN_FUZZ" not in os.environ, database=None)
    @given(programs(), st.integers(0, 10**6))
    def run(prog, seed):
        text, use_idx, use_c, use_m = prog
        assume(not use_idx)
        program = krn.parse(text)
        wrt = ("a", "b") + (("m",) if use_m else ())
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            try:
                krn.differentiate(program, "f", wrt)
                assume(False)  # feasible without a tape: covered elsewhere
            except krn.NotFeasible:
                pass
            try:
                gp = krn.differentiate(program, "f", wrt, tape=True)
            except krn.NotFeasible:
                assume(False)
        gfn = gp.functions[-1]
        n = 4
        base = fuzz_inputs(n, use_idx, use_c, seed, use_m)

        def value(d):
            call = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in d.items()}
            with np.errstate(all="ignore"):
                return interp.run(program, "f", call)

        v0 = value(base)
        assume(np.isfinite(v0) and abs(v0) < 1e6)
        call = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in base.items()}
        shadows = [p.name for p in gfn.params[len(program.functions[0].params):]]
        active = [s_[3:] for s_ in shadows]
        for s_ in shadows:
            call[s_] = np.zeros_like(base[s_[3:]])
        with np.errstate(all="ignore"):
            interp.run(gp, gfn.name, call)
        h = 1e-5
        for w in active:
            got = call["_d_" + w].reshape(-1)
            for k in range(got.size):
                up = {a: (b.copy() if isinstance(b, np.ndarray) else b) for a, b in base.items()}
                dn = {a: (b.copy() if isinstance(b, np.ndarray) else b) for a, b in base.items()}
                up[w].reshape(-1)[k] += h
                dn[w].reshape(-1)[k] -= h
                fd = (value(up) - value(dn)) / (2 * h)
                scale = max(1.0, abs(fd), abs(v0))
                assert abs(got[k] - fd) <= 2e-5 * scale, (text, w, k, got[k], fd)
        checked[0] += 1

    run()
    assert checked[0] >= 10  # the generator does produce functions that need a tape
