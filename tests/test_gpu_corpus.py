"""GPU parity, corpus: every benchmark program and its generated gradient,
through the reference-facing API (``execute``), against outputs of the
reference itself (tests/golden/corpus.npz) and against the CPU oracle on fresh
seeded inputs.  Bar: bit-exact for every program - gather_indirect's gradient
included: under the default configuration (deterministic_reduction=True) its
atomic_add queue is applied in the reference's order (atomic_policy "ordered",
csrc/krn_ordered.cu).  The hardware-atomic policies (rel 1e-12) are covered by
tests/test_gpu_atomics.py."""

import numpy as np
import pytest

import paper_2507_13204_b200 as krn
from conftest import CORPUS, SIZES, assert_bits, corpus_case

pytestmark = pytest.mark.gpu

ATOMIC_ORDER: set = set()  # nothing: the default accumulation policy is the reference's order


def _views(inputs):
    return {k: krn.ViewStorage.from_values(k, v) if isinstance(v, np.ndarray) else v for k, v in inputs.items()}


@pytest.mark.parametrize("policy", ["fused", "compiled", "statements"])
@pytest.mark.parametrize("n", SIZES)
@pytest.mark.parametrize("stem", CORPUS)
def test_primal_matches_reference(corpus_golden, stem, n, policy):
    inputs, wrt, key = corpus_case(corpus_golden, stem, n)
    prog = krn.load_program(stem)
    fn = prog.functions[0]
    call = _views(inputs)
    res = krn.execute(prog, fn.name, call, krn.ExecutionConfig(policy=policy))
    assert_bits(res.value, corpus_golden[key + "/primal/value"], f"{key} value")
    for name, v in call.items():
        if isinstance(v, krn.ViewStorage):
            assert_bits(v.buffer, corpus_golden[f"{key}/primal/after/{name}"], f"{key} {name}")


@pytest.mark.parametrize("policy", ["fused", "compiled", "statements"])
@pytest.mark.parametrize("n", SIZES)
@pytest.mark.parametrize("stem", CORPUS)
def test_gradient_matches_reference(corpus_golden, stem, n, policy):
    inputs, wrt, key = corpus_case(corpus_golden, stem, n)
    prog = krn.load_program(stem)
    fn = prog.functions[0]
    gp = krn.differentiate(prog, fn.name, wrt)
    gfn = gp.functions[-1]
    call = _views(inputs)
    for sp, primal in zip(gfn.params[len(fn.params):], wrt):
        call[sp.name] = krn.ViewStorage.zeros(sp.name, np.shape(inputs[primal]))
    res = krn.execute(gp, gfn.name, call, krn.ExecutionConfig(policy=policy))
    assert res.value is None
    for name, v in call.items():
        if not isinstance(v, krn.ViewStorage):
            continue
        want = corpus_golden[f"{key}/grad/after/{name}"]
        if stem in ATOMIC_ORDER and name.startswith("_d_"):
            got = v.buffer
            assert np.all(np.abs(got - want) <= 1e-12 * np.abs(want)), f"{key} {name}"
        else:
            assert_bits(v.buffer, want, f"{key} {name}")


@pytest.mark.parametrize("stem", CORPUS)
def test_gradient_matches_oracle_on_fresh_inputs(stem):
    """Sizes the stored vectors do not cover, checked against the CPU oracle."""
    from oracle import interp

    prog = krn.load_program(stem)
    fn = prog.functions[0]
    for n in (5, 64, 129, 1000):
        rng = np.random.default_rng(77 + n)
        inputs = {}
        for p in fn.params:
            if not p.is_view:
                inputs[p.name] = float(rng.uniform(0.5, 1.5))
            elif p.name == "idx":
                inputs[p.name] = rng.integers(0, n, size=n).astype(np.float64)
            elif p.type.rank == 2:
                inputs[p.name] = rng.normal(size=(n, 3))
            else:
                inputs[p.name] = rng.normal(size=n)
        wrt = tuple(p.name for p in fn.params if p.is_view and p.name != "idx")
        gp = krn.differentiate(prog, fn.name, wrt)
        gfn = gp.functions[-1]
        want = {k: np.array(v) if isinstance(v, np.ndarray) else v for k, v in inputs.items()}
        call = _views(inputs)
        for sp, primal in zip(gfn.params[len(fn.params):], wrt):
            want[sp.name] = np.zeros(np.shape(inputs[primal]))
            call[sp.name] = krn.ViewStorage.zeros(sp.name, np.shape(inputs[primal]))
        interp.run(gp, gfn.name, want)
        krn.execute(gp, gfn.name, call, krn.ExecutionConfig(policy="statements"))
        for name, v in call.items():
            if not isinstance(v, krn.ViewStorage):
                continue
            if stem in ATOMIC_ORDER and name.startswith("_d_"):
                assert np.all(np.abs(v.buffer - want[name]) <= 1e-12 * np.abs(want[name])), (stem, n, name)
            else:
                assert_bits(v.buffer, want[name], f"{stem} n={n} {name}")
