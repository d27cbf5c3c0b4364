"""CPU tier: the oracle (oracle/interp.py, oracle/krn_oracle.c) against outputs of
the reference itself (tests/golden, written by oracle/make_golden.py) and the
reference's known-answer tests."""

import numpy as np
import pytest

import paper_2507_13204_b200 as krn
from oracle import cport, interp
from conftest import CORPUS, SIZES, assert_bits, corpus_case

FN = "normRes1DLaplacianSQ"


@pytest.mark.parametrize("stem", CORPUS)
def test_interp_matches_reference_corpus(corpus_golden, stem):
    prog = krn.load_program(stem)
    fn = prog.functions[0]
    for n in SIZES:
        inputs, wrt, key = corpus_case(corpus_golden, stem, n)
        call = {k: np.array(v) if isinstance(v, np.ndarray) else v for k, v in inputs.items()}
        value = interp.run(prog, fn.name, call)
        assert_bits(value, corpus_golden[key + "/primal/value"], key)
        for k, v in call.items():
            if isinstance(v, np.ndarray):
                assert_bits(v, corpus_golden[f"{key}/primal/after/{k}"], f"{key} {k}")
        gp = krn.differentiate(prog, fn.name, wrt)
        gfn = gp.functions[-1]
        call = {k: np.array(v) if isinstance(v, np.ndarray) else v for k, v in inputs.items()}
        for sp, primal in zip(gfn.params[len(fn.params):], wrt):
            call[sp.name] = np.zeros(np.shape(inputs[primal]))
        assert interp.run(gp, gfn.name, call) is None
        for k, v in call.items():
            if isinstance(v, np.ndarray):
                assert_bits(v, corpus_golden[f"{key}/grad/after/{k}"], f"{key} grad {k}")


def test_c_port_matches_reference_headline(laplacian_golden):
    g = laplacian_golden
    for tag in sorted({k.split("/")[0] for k in g.files}):
        if f"{tag}/x" in g.files:
            x, b = g[f"{tag}/x"], g[f"{tag}/b"]
        else:
            n = int(tag.split("_n")[1])
            rng = np.random.default_rng(0)
            x, b = rng.uniform(-1.0, 1.0, n), rng.uniform(-1.0, 1.0, n)
        n = x.size
        xc = x.copy()
        with np.errstate(all="ignore"):
            f = cport.laplacian_primal(xc, b.copy())
            dx = g[f"{tag}/dx0"].copy() if f"{tag}/dx0" in g.files else np.zeros(n)
            db = g[f"{tag}/db0"].copy() if f"{tag}/db0" in g.files else np.zeros(n)
            xg = x.copy()
            cport.laplacian_grad(xg, b.copy(), dx, db, float(g[f"{tag}/seed"]))
        assert_bits(f, g[f"{tag}/f"], tag)
        assert_bits(xc, g[f"{tag}/x_after"], tag)
        assert_bits(xg, g[f"{tag}/x_after"], tag)
        assert_bits(dx, g[f"{tag}/dx"], tag)
        assert_bits(db, g[f"{tag}/db"], tag)


def test_golden_values_quoted_in_survey(laplacian_golden):
    """f at N=1000 and N=10000 for the bench inputs"""
    assert float(laplacian_golden["bench_n1000/f"]) == 19156.501489526854
    assert float(laplacian_golden["bench_n10000/f"]) == 189292.31519333157
    assert laplacian_golden["bench_n1000/dx"][:3].tolist() == [56.89983467454396, -34.50904364043208, 23.083696603425363]


def test_pairwise_tree(pairwise_golden):
    for n, want in zip(pairwise_golden["lengths"], pairwise_golden["sums"]):
        n = int(n)
        v = np.random.default_rng(n).normal(size=n) * 10.0 ** np.random.default_rng(n + 1).integers(-3, 4, size=n)
        assert_bits(interp.pairwise_sum(v), want, f"interp n={n}")
        assert_bits(cport.pairwise_sum(v), want, f"c n={n}")
    for n in (1, 2, 3, 4, 5, 8, 12, 16):
        assert_bits(cport.pairwise_sum(np.full(n, -0.0)), pairwise_golden[f"negzero_{n}"], f"-0.0 n={n}")
        assert_bits(interp.pairwise_sum(np.full(n, -0.0)), pairwise_golden[f"negzero_{n}"], f"-0.0 n={n}")


def test_known_answers_from_reference_tests():
    """reference tests/test_runtime.py:41-51, 61-69, 72-82, 132-143, 352-362"""
    lap = krn.load_program("laplacian")
    x, b = np.ones(3), np.zeros(3)
    assert interp.run(lap, FN, {"x": x, "b": b}) == 18.0 and x.tolist() == [3.0, 3.0, 3.0]
    gp = krn.differentiate(lap, FN, ("x", "b"))
    call = {"x": np.ones(3), "b": np.zeros(3), "_d_x": np.zeros(3), "_d_b": np.zeros(3)}
    interp.run(gp, FN + "_grad", call)
    assert call["_d_x"].tolist() == [36.0, -36.0, 36.0] and call["_d_b"].tolist() == [-6.0, 0.0, -6.0]
    acc = krn.parse("fn f(v: view<f64,1>) -> f64 { let s: f64 = 2.0; s = parallel_sum(v); return s; }")
    assert interp.run(acc, "f", {"v": np.array([1.0, 2.0, 3.0])}) == 8.0
    bc = krn.parse("fn f(v: view<f64,1>, w: view<f64,1>, c: f64) { parallel_sum(v, c); parallel_sum(v, w); }")
    v = np.array([1.0, 2.0, 3.0])
    interp.run(bc, "f", {"v": v, "w": np.array([10.0, 10.0, 10.0]), "c": 1.5})
    assert v.tolist() == [12.5, 13.5, 14.5]
    div = krn.parse("fn f(v: view<f64,1>) -> f64 { parallel_for i in 0..extent(v,0) { v(i) = 1.0 / v(i); } return v(0); }")
    assert interp.run(div, "f", {"v": np.array([0.0])}) == float("inf")
    oob = krn.parse("fn f(v: view<f64,1>) {\n parallel_for i in 0..extent(v,0) {\n v(i + 1) = 1.0;\n }\n}")
    with pytest.raises(interp.OutOfBounds, match=r"line 3: v\(4\) outside extent 4"):
        interp.run(oob, "f", {"v": np.zeros(4)})
    with pytest.raises(interp.ShapeMismatch):
        interp.run(lap, FN, {"x": np.ones(3)})
    with pytest.raises(KeyError):
        interp.run(lap, "nope", {})


def test_analytic_oracle_frozen_values():
    """reference tests/test_verify.py:31-51"""
    f, gx, gb = krn.laplacian_oracle([1.0, 1.0, 1.0], [0.0, 0.0, 0.0])
    assert f == 18.0 and gx.tolist() == [36.0, -36.0, 36.0] and gb.tolist() == [-6.0, 0.0, -6.0]
    f, gx, gb = krn.laplacian_oracle([1.0], [0.0])
    assert f == 36.0 and gx.tolist() == [72.0] and gb.tolist() == [-12.0]
