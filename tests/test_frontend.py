"""CPU tier: the kernel-language front-end against fixtures produced by the
reference (tests/golden/grad_text) and the reference's documented behaviour
(reference tests/test_adjoint.py, test_analysis.py, test_parser.py)."""

import os
import warnings

import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import paper_2507_13204_b200 as krn
from paper_2507_13204_b200.lang import nodes as N
from conftest import CORPUS, GOLDEN


def _wrt(fn):
    return tuple(p.name for p in fn.params if p.is_view and p.name != "idx")


@pytest.mark.parametrize("stem", CORPUS)
def test_gradient_text_matches_reference(stem):
    prog = krn.load_program(stem)
    fn = prog.functions[0]
    gp = krn.differentiate(prog, fn.name, _wrt(fn))
    want = open(os.path.join(GOLDEN, "grad_text", stem + ".krn")).read()
    assert krn.emit(gp.functions[-1]) == want


@pytest.mark.parametrize("stem", CORPUS)
def test_round_trip_and_closure(stem):
    """criterion 7: parse(emit(p)) == p, and diff output re-parses and re-validates"""
    prog = krn.load_program(stem)
    assert krn.parse(krn.emit(prog)) == prog
    fn = prog.functions[0]
    gp = krn.differentiate(prog, fn.name, _wrt(fn))
    again = krn.parse(krn.emit(gp))
    assert again == gp and krn.validate(again) == []


def test_laplacian_structure():
    """criterion 1: 2 forward + 2 reverse kernels, one seed, one broadcast, atomics on _d_x only"""
    prog = krn.load_program("laplacian")
    g = krn.differentiate(prog, "normRes1DLaplacianSQ", ("x", "b")).functions[-1]
    loops = [s for s in g.body if N.kind(s) == "ParallelFor"]
    assert len(loops) == 4
    atomics = [s for s in N.walk_statements(g.body) if N.kind(s) == "AtomicAdd"]
    assert {a.target.view for a in atomics} == {"_d_x"} and len(atomics) == 3
    seeds = [s for s in g.body if N.kind(s) == "AssignScalar" and s.name == "_d_sum"]
    assert len(seeds) == 1 and seeds[0].op == "+=" and seeds[0].rhs == N.Literal(1.0)
    bcast = [s for s in g.body if N.kind(s) == "ParallelSumInto"]
    assert len(bcast) == 1 and bcast[0].dst == "_d_y2" and bcast[0].src == N.ScalarVar("_d_sum")
    assert [p.name for p in g.params] == ["x", "b", "_d_x", "_d_b"] and g.returns is None


def test_analyses_on_corpus():
    lap = krn.load_program("laplacian").functions[0]
    act = krn.activity(N.desugar_function(lap), ("x", "b"))
    assert act.active_views == {"x", "b", "y", "y2"} and act.active_scalars == {"sum"}
    flags = krn.race_analysis(lap).flags
    assert [(f.kernel, f.view, f.rule) for f in flags] == [(1, "x", 2)]
    assert flags[0].indices == ("(j + 1)", "(j - 1)", "(j)")
    gi = krn.load_program("gather_indirect").functions[0]
    assert [(f.view, f.rule) for f in krn.race_analysis(gi).flags] == [("x", 1)]
    rs = krn.load_program("rowscale_rank2").functions[0]
    assert {f.view for f in krn.race_analysis(rs).flags} == {"m", "q"}
    assert krn.activity(lap, ()).active_views == frozenset()
    with pytest.raises(krn.UnknownParameter):
        krn.activity(lap, ("nope",))


def test_failure_modes():
    bad = krn.parse("fn f(x: view<f64,1>) -> f64 { let y: view<f64,1> = view(\"y\", extent(x,0));"
                    " parallel_for i in 0..extent(x,0) { x(i) = x(i) * x(i); y(i) = x(i); }"
                    " return parallel_sum(y); }")
    with pytest.raises(krn.NotFeasible):
        krn.differentiate(bad, "f", ("x",))
    lap = krn.load_program("laplacian")
    with pytest.raises(krn.UnknownFunction):
        krn.differentiate(lap, "missing", ("x",))
    const = krn.parse("fn f(x: view<f64,1>, b: view<f64,1>) -> f64 { return parallel_sum(b); }")
    with warnings.catch_warnings(record=True) as w:
        warnings.simplefilter("always")
        g = krn.differentiate(const, "f", ("x",))
    assert any(issubclass(i.category, krn.InactiveReturn) for i in w)
    assert g.functions[-1].name == "f_grad"
    with pytest.raises(krn.ParseError):
        krn.parse("fn f( { ")
    with pytest.raises(krn.ValidationError):
        krn.parse("fn f(x: view<f64,1>) -> f64 { parallel_for i in 0..extent(x,0) { x(i, i) = 1.0; } return 0.0; }")
    with pytest.raises(krn.ParseError):  # nested parallelism
        krn.parse("fn f(x: view<f64,1>) { parallel_for i in 0..3 { parallel_for j in 0..3 { x(i) = 1.0; } } }")
    with pytest.raises(ValueError):
        krn.differentiate(krn.load_program("fill_scale"), "fillScale", ("c",))


def test_index_normalisation_commutes():
    from paper_2507_13204_b200.lang.dataflow import normalize_index

    a = krn.parse("fn f(x: view<f64,1>) { parallel_for j in 0..extent(x,0) { x(j + 1) = x(1 + j); } }")
    stmt = a.functions[0].body[0].body[0]
    assert normalize_index(stmt.target.indices[0]) == normalize_index(stmt.rhs.indices[0])
    assert krn.race_analysis(a.functions[0]).flags == ()


@settings(max_examples=200, deadline=None, derandomize=True, database=None)
@given(st.text(alphabet="fn xyz(){}:<>,;=+-*/.0123456789\"view f64 let if in return parallel_for _sum\n", max_size=120))
def test_parser_never_crashes(text):
    try:
        krn.parse(text)
    except (krn.ParseError, krn.ValidationError):
        pass
