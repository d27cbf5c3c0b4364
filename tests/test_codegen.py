"""CPU tier: host logic of the statement path - accumulation policy per atomic
target, generated module shape, plan steps."""

import numpy as np

import paper_2507_13204_b200 as krn
from paper_2507_13204_b200 import codegen
from paper_2507_13204_b200.lang import nodes as N
from paper_2507_13204_b200.runtime import _plan_for
from conftest import CORPUS


def _grad(stem):
    prog = krn.load_program(stem)
    fn = prog.functions[0]
    wrt = tuple(p.name for p in fn.params if p.is_view and p.name != "idx")
    return krn.differentiate(prog, fn.name, wrt).functions[-1]


def _loops(fn):
    return [s for s in fn.body if N.kind(s) == "ParallelFor"]


def test_atomic_policies():
    lap = _loops(_grad("laplacian"))[2]
    sites = codegen.plan_atomics(lap)
    assert [(s.view, s.offset, s.mode) for s in sites] == [
        ("_d_x", 1, "gather"), ("_d_x", -1, "gather"), ("_d_x", 0, "gather")]
    gi = _loops(_grad("gather_indirect"))[1]
    assert [s.mode for s in codegen.plan_atomics(gi)] == ["atomic", "atomic"]
    rs = _loops(_grad("rowscale_rank2"))[1]
    sites = codegen.plan_atomics(rs)
    assert {s.mode for s in sites} == {"gather"}
    assert sorted({(s.view, s.column) for s in sites}) == [("_d_m", 0), ("_d_m", 1), ("_d_m", 2),
                                                          ("_d_q", 0), ("_d_q", 1), ("_d_q", 2)]
    # a target that the kernel also reads through an indirect index must be staged
    p = krn.parse("fn f(x: view<f64,1>, idx: view<f64,1>) { parallel_for i in 0..extent(idx,0) {"
                  " atomic_add(x(idx(i)), x(i)); } }")
    assert [s.mode for s in codegen.plan_atomics(p.functions[0].body[0])] == ["staged_atomic"]


def test_adjacent_atomics_on_one_location_merge():
    """The product rule emits two atomic_adds to _d_x(idx(i)) back to back: one reduction with the
    sum of both values (hardware-atomic sites only; gather-mode sites stay separate, they are
    bit-identical to the interpreter)."""
    gi = _loops(_grad("gather_indirect"))[1]
    sites = codegen.plan_atomics(gi)
    assert [(s.mode, len(s.merged), s.absorbed) for s in sites] == [("atomic", 1, False), ("atomic", 0, True)]
    src = _plan_for(_grad("gather_indirect")).source
    assert sum("krn_scatter(E," in ln and "__device__" not in ln for ln in src.splitlines()) == 1
    lap = _loops(_grad("laplacian"))[2]
    assert all(not s.merged and not s.absorbed for s in codegen.plan_atomics(lap))
    # different locations, a statement in between, or different guards: not merged
    p = krn.parse("""fn f(x: view<f64,1>, idx: view<f64,1>, v: view<f64,1>) { parallel_for i in 0..extent(idx,0) {
        atomic_add(x(idx(i)), v(i)); atomic_add(x(idx(i) + 1), v(i));
        let t: f64 = v(i);
        atomic_add(x(idx(i) + 1), t);
        if (i != 0) { atomic_add(x(idx(i) + 1), t); atomic_add(x(idx(i) + 1), 2.0 * t); atomic_add(x(idx(i) + 1), t); }
    } }""")
    sites = codegen.plan_atomics(p.functions[0].body[0])
    assert [(len(s.merged), s.absorbed) for s in sites] == [(0, False), (0, False), (0, False), (2, False),
                                                            (0, True), (0, True)]


def test_every_corpus_function_plans():
    for stem in CORPUS:
        prog = krn.load_program(stem)
        for fn in (prog.functions[0], _grad(stem)):
            plan = _plan_for(fn)
            assert plan.source.count('extern "C" __global__') >= 1
            kinds = [s[0] for s in plan.steps]
            assert kinds.count("kernel") == len(_loops(fn))


def test_literals_are_exact():
    for v in (0.1, 1.5, -0.25, 3.0, 1e-300, 5e-324, -0.0):
        text = codegen.c_double(v).strip("()")
        assert float.fromhex(text) == v and np.signbit(float.fromhex(text)) == np.signbit(v)


def test_order_dependent_kernels_are_recognised():
    """carries_across_iterations: index expressions that let two iterations meet at one location
    with a plain write among the accesses (reference scan, tests/test_runtime.py:101-115)."""
    def flag(body, params="v: view<f64,1>, w: view<f64,1>, m: view<f64,2>, idx: view<f64,1>"):
        p = krn.parse("fn f(%s) { parallel_for i in 0..extent(v,0) { %s } }" % (params, body))
        return codegen.carries_across_iterations(p.functions[0].body[0])

    assert flag("if (i != 0) { v(i) = v(i - 1) + i; }")          # scan
    assert flag("w(0) = v(i);")                                   # every iteration writes one location
    assert flag("w(idx(i)) = v(i);")                              # through a View: nothing known
    assert flag("w(i) = v(i); w(i + 1) += 1.0;")                  # two writes one row apart
    assert flag("m(i, 0) = m(i + 1, 0);")
    assert not flag("v(i) = 3.0 * v(i);")
    assert not flag("w(i) = v(i + 1) - v(i - 1);")                # neighbours of a View that is only read
    assert not flag("m(i, 0) = v(i); m(i, 1) = m(i, 0) * m(i, 2);")   # literal columns of the own row
    assert not flag("w(2 * i) = v(i); w(2 * i + 1) = v(i);")      # interleaved, never the same element
    assert not flag("atomic_add(w(idx(i)), v(i)); v(i) = 0.0;")   # atomics are not plain writes
    for stem in CORPUS:
        prog = krn.load_program(stem)
        for fn in (prog.functions[0], _grad(stem)):
            assert not _plan_for(fn).carried


def test_injective_affine_targets_are_updated_directly():
    """general affine gather form (row N2): sites `a*i + c` on one View with one writing iteration per
    location are 'direct'; sites that share a residue mod a with different constants are not"""
    from paper_2507_13204_b200 import compiled

    def modes(stem, wrt):
        prog = krn.load_program(stem)
        g = krn.differentiate(prog, prog.functions[0].name, wrt).functions[-1]
        out = {}
        for loop in _loops(g):
            for st in codegen.plan_atomics(loop):
                out.setdefault(st.view, set()).add(st.mode)
        return g, out

    g, m = modes("stride2_scatter", ("fine", "w"))
    assert m == {"_d_fine": {"direct"}, "_d_w": {"gather"}}
    assert compiled.plan_for(g).launch_count == 1  # the in-order update lives inside the window kernel
    g, m = modes("stride2_collide", ("fine", "w"))
    assert m == {"_d_fine": {"atomic"}, "_d_w": {"gather"}}  # 2i - 1 and 2i + 1 meet: the ordered queue
    g, m = modes("rank2_row_offset", ("m", "r"))
    assert m == {"_d_m": {"gather"}} and compiled.plan_for(g).launch_count == 1
    # reversal: one site, a = -1 -> direct; two sites on a reversed index with different constants -> not
    p = krn.parse("""fn f(v: view<f64,1>, a: view<f64,1>, b: view<f64,1>) {
        parallel_for i in 0..extent(v, 0) {
            atomic_add(a(extent(v, 0) - 1 - i), v(i));
            atomic_add(b(extent(v, 0) - 1 - i), v(i));
            if (i != 0) { atomic_add(b(extent(v, 0) - i), v(i)); }
        } }""")
    got = {st.view: st.mode for st in codegen.plan_atomics(p.functions[0].body[0])}
    assert got == {"a": "direct", "b": "atomic"}
    # a kernel that also READS the target must not update it early (deferral)
    p = krn.parse("""fn f(v: view<f64,1>, a: view<f64,1>) {
        parallel_for i in 0..extent(v, 0) { v(i) = a(2 * i); atomic_add(a(2 * i + 1), v(i)); } }""")
    assert [st.mode for st in codegen.plan_atomics(p.functions[0].body[0])] == ["staged_atomic"]


def test_ordered_queue_layout():
    """records of the ordered policy: groups per iteration in program order, merged sites share a
    record, sites on the literal columns of one row share a ROW record"""
    gi = _loops(_grad("gather_indirect"))[1]
    sites = codegen.plan_atomics(gi)
    assert codegen.assign_ordered([sites]) == [dict(view="_d_x", groups=1, width=2, key_off=0, val_off=0, cols=None,
                                                    guarded=False)]
    assert sites[0].ord == (0, 0, 1, 2, 0) and sites[1].absorbed
    prog = krn.load_program("gather_rows_rank2")
    g = krn.differentiate(prog, "rowGather", ("q", "w")).functions[-1]
    sites = codegen.plan_atomics(_loops(g)[1])
    assert [(s.lanes, s.absorbed) for s in sites] == [(True, False), (False, True), (False, True)]
    assert codegen.assign_ordered([sites]) == [dict(view="_d_q", groups=1, width=3, key_off=0, val_off=0, cols=(0, 1, 2),
                                                    guarded=False)]
    # two targets, a guarded site, lane groups with DIFFERENT column sets: back to one record per site
    p = krn.parse("""fn f(idx: view<f64,1>, v: view<f64,1>, m: view<f64,2>, a: view<f64,1>) {
        parallel_for i in 0..extent(idx, 0) {
            atomic_add(m(idx(i), 0), v(i)); atomic_add(m(idx(i), 2), v(i));
            if (i != 0) { atomic_add(a(idx(i)), v(i)); }
            atomic_add(m(idx(i), 1), v(i)); atomic_add(m(idx(i), 2), v(i));
        } }""")
    sites = codegen.plan_atomics(p.functions[0].body[0])
    entries = codegen.assign_ordered([sites])
    assert entries == [dict(view="m", groups=4, width=1, key_off=0, val_off=0, cols=None, guarded=False),
                       dict(view="a", groups=1, width=1, key_off=4, val_off=4, cols=None, guarded=True)]
    assert not any(s.absorbed or s.lanes for s in sites)
    src = codegen.ModuleBuilder(p.functions[0])
    src.kernel(p.functions[0].body[0], "k0")
    text = src.source()
    assert text.count("krn_ord_put(E, 0, 0, 4, 1,") == 4 and text.count("krn_ord_put(E, 4, 4, 1, 1, 0,") == 1
