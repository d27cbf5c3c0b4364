"""CPU tier: the additional programs (paper_2507_13204_b200/extra_programs/) against vectors the
REFERENCE produced for them (tests/golden/extra.npz, oracle/make_golden_extra.py): the oracle
restatement and this repository's reverse-mode transform must reproduce them exactly."""

import os

import numpy as np
import pytest

import paper_2507_13204_b200 as krn
from conftest import GOLDEN as GOLDEN_DIR, assert_bits

EXTRA = sorted(f[:-4] for f in os.listdir(os.path.join(os.path.dirname(krn.PROGRAMS_DIR), "extra_programs"))
               if f.endswith(".krn"))
SIZES = (1, 2, 5, 130, 1030)


@pytest.fixture(scope="module")
def extra_golden():
    return np.load(os.path.join(GOLDEN_DIR, "extra.npz"))


def case(golden, stem, n):
    key = f"{stem}/n{n}"
    inputs = {k.split("/in/")[1]: golden[k] for k in golden.files if k.startswith(key + "/in/")}
    fn = krn.load_program(stem).functions[0]
    for p in fn.params:
        if not p.is_view:
            inputs[p.name] = float(inputs[p.name])
    wrt = tuple(str(golden[f"{stem}/wrt"]).split(","))
    return key, inputs, wrt


def test_emitted_gradient_text_equals_the_reference():
    for stem in EXTRA:
        path = os.path.join(GOLDEN_DIR, "grad_text_extra", stem + ".krn")
        prog = krn.load_program(stem)
        fn = prog.functions[0]
        wrt = tuple(p.name for p in fn.params if p.is_view and p.name != "idx")
        if not os.path.exists(path):
            with pytest.raises((krn.NotFeasible, ValueError)):
                krn.differentiate(prog, fn.name, wrt)
            continue
        assert krn.emit(krn.differentiate(prog, fn.name, wrt).functions[-1]) == open(path).read(), stem


@pytest.mark.parametrize("n", SIZES)
@pytest.mark.parametrize("stem", EXTRA)
def test_oracle_reproduces_the_reference(extra_golden, stem, n):
    from oracle import interp

    key, inputs, wrt = case(extra_golden, stem, n)
    prog = krn.load_program(stem)
    fn = prog.functions[0]
    arrays = {k: np.array(v) if isinstance(v, np.ndarray) else v for k, v in inputs.items()}
    value = interp.run(prog, fn.name, arrays)
    want = extra_golden[f"{key}/primal/value"]
    if value is None:
        assert np.isnan(want)
    else:
        assert_bits(value, want, f"{key} value")
    for k in arrays:
        if isinstance(arrays[k], np.ndarray):
            assert_bits(arrays[k], extra_golden[f"{key}/primal/after/{k}"], f"{key} {k}")
    if not bool(extra_golden[f"{stem}/has_grad"]):
        return
    gp = krn.differentiate(prog, fn.name, wrt)
    gfn = gp.functions[-1]
    arrays = {k: np.array(v) if isinstance(v, np.ndarray) else v for k, v in inputs.items()}
    for p in gfn.params[len(fn.params):]:
        arrays[p.name] = np.array(extra_golden[f"{key}/grad/in/{p.name}"])
    interp.run(gp, gfn.name, arrays)
    for k in arrays:
        if isinstance(arrays[k], np.ndarray):
            assert_bits(arrays[k], extra_golden[f"{key}/grad/after/{k}"], f"{key} grad {k}")
