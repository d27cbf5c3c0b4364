"""CPU tier: decisions of the fusion pass (grouping, promotion, dead code, host
scalars, bounds-check elision) on the corpus - no device needed."""

import paper_2507_13204_b200 as krn
from paper_2507_13204_b200 import compiled, fusion
from conftest import CORPUS


def _grad(stem):
    prog = krn.load_program(stem)
    fn = prog.functions[0]
    wrt = tuple(p.name for p in fn.params if p.is_view and p.name != "idx")
    return fn, krn.differentiate(prog, fn.name, wrt).functions[-1]


def _shape(fn, windows=False):
    an = fusion.Analysis(fn)
    out = []
    for item in fusion.form_groups(fusion.build_ops(fn, an, windows), an, windows):
        if item[0] == "group":
            g = item[1]
            out.append("G[" + ",".join(o.what for o in g.ops) + ("+gather" if g.gather else "") + "]")
        else:
            out.append(item[0])
    return an, out


def test_headline_schedule():
    fn, g = _grad("laplacian")
    an, shape = _shape(fn)
    # the in-place scale cannot fuse with the stencil that reads its neighbours' results
    assert [s for s in shape if s.startswith("G[")] == ["G[kernel]", "G[kernel+gather]"]
    an, shape = _shape(g)
    assert an.host_scalars == {"_d_sum"}  # the seed never needs a device kernel
    groups = [s for s in shape if s.startswith("G[")]
    # forward stencil + seed broadcast + its reversal in one kernel; the dead forward reduction is gone;
    # the deferred atomics' apply loop fuses with the reversal of the scale kernel
    assert groups == ["G[kernel]", "G[kernel,suminto,kernel]", "G[apply,kernel]"]
    assert "gather" not in shape


def test_headline_schedule_with_halo_recompute():
    """window_plan: the in-place scale, the stencil, the seed broadcast, the stencil's reversal,
    the deferred atomics' apply loop and the scale's reversal become ONE kernel; every warp
    re-runs 2 iterations either side for the scale and 1 for the stencil and its reversal."""
    fn, g = _grad("laplacian")
    _, shape = _shape(fn, True)
    assert [s for s in shape if s.startswith("G[")] == ["G[kernel,kernel+gather]"]
    an, shape = _shape(g, True)
    assert [s for s in shape if s.startswith("G[")] == ["G[kernel,kernel,suminto,kernel,apply,kernel]"]
    group = [i[1] for i in fusion.form_groups(fusion.build_ops(g, an, True), an, True) if i[0] == "group"][0]
    wp = fusion.window_plan(group.ops, an)
    assert wp.halo == [(2, 2), (1, 1), (1, 1), (1, 1), (0, 0), (0, 0)] and (wp.hlo, wp.hhi) == (2, 2)
    assert wp.windowed == ["x"]
    # contributions to _d_x(j +- 1) cross lanes (windows); the one to _d_x(j) stays in a register
    assert len(wp.stage_windows) == 2 and len(wp.stage_regs) == 1
    assert wp.phases == [[0], [1, 2, 3], [4, 5]]
    plan = compiled.plan_for(g, True)
    assert plan.windowed and plan.launch_count == 1
    recipe = [s[2] for s in plan.steps if s[0] == "group"][0]
    views = {p["view"]: p for p in recipe["promoted"]}
    # x is read on halo rows and stored: out of place; so is _d_b (touched by a halo statement)
    assert sorted(recipe["alt"]) == ["_d_b", "x"] and not views["_d_x"]["alt"]
    for v in ("y", "y2", "_d_y", "_d_y2"):
        assert not views[v]["store"]
    assert not recipe["stage_cols"]  # nothing staged through global memory


def test_window_plan_refuses_side_effects_on_halo_iterations():
    # the first kernel would have to re-run on halo iterations, but it scatters with hardware atomics
    p = krn.parse("""fn f(x: view<f64,1>, idx: view<f64,1>, acc: view<f64,1>, y: view<f64,1>) {
        parallel_for i in 0..extent(x, 0) { x(i) = 2.0 * x(i); atomic_add(acc(idx(i)), 1.0); }
        parallel_for i in 0..extent(x, 0) { if (i != 0) { y(i) = x(i - 1); } } }""")
    _, shape = _shape(p.functions[0], True)
    assert [s for s in shape if s.startswith("G[")] == ["G[kernel]", "G[kernel]"]
    # an unguarded neighbour read cannot be proven in range: no window, two launches, checks kept
    p = krn.parse("""fn f(x: view<f64,1>, y: view<f64,1>) {
        parallel_for i in 0..extent(x, 0) { x(i) = 2.0 * x(i); }
        parallel_for i in 0..extent(x, 0) { y(i) = x(i + 1); } }""")
    _, shape = _shape(p.functions[0], True)
    assert [s for s in shape if s.startswith("G[")] == ["G[kernel]", "G[kernel]"]


def test_promotion_and_dead_stores():
    _, g = _grad("laplacian")
    plan = compiled.plan_for(g, False)
    recipes = [s[2] for s in plan.steps if s[0] == "group"]
    middle = {p["view"]: p for p in recipes[1]["promoted"]}
    # y, y2, _d_y, _d_y2 live and die inside the kernel: never loaded from nor stored to memory
    for v in ("y", "y2"):
        assert not middle[v]["load"] and not middle[v]["store"]
    for v in ("_d_y", "_d_y2"):
        assert not middle[v]["store"]
    assert middle["_d_b"]["store"] and middle["b"]["load"] and not middle["b"]["store"]
    assert "x" not in middle and recipes[1]["elided_views"] == ["_d_x", "x"]
    assert len(recipes[1]["stage_cols"]) == 3
    last = {p["view"]: p for p in recipes[2]["promoted"]}
    assert last["_d_x"]["store"]


def test_every_corpus_function_compiles_to_a_plan():
    for stem in CORPUS:
        for fn in _grad(stem):
            plan = compiled.plan_for(fn)
            assert plan.source.count('extern "C" __global__') >= 1
            statements = sum(1 for s in fn.body if type(s).__name__ in
                             ("ParallelFor", "DeepCopy", "ParallelSum", "ParallelSumInto"))
            launches = sum(1 for s in plan.steps if s[0] in ("group", "kernel", "gather", "deepcopy", "suminto"))
            assert launches <= statements


def test_rank2_rows_become_register_columns():
    fn, g = _grad("rowscale_rank2")
    _, shape = _shape(g)  # pointwise-only fusion leaves rank-2 statements alone
    assert "raw" in shape and not any(s.startswith("G[") for s in shape)
    # the window generator keeps m(i, c), q(i, c), _d_q(i, c), _d_m(i, c) in register columns: the
    # forward kernel, the seed broadcast (unrolled over the 3 columns), the reversal and the apply
    # loops of its (conservatively flagged, in fact injective) atomics are one launch
    an, shape = _shape(g, True)
    assert [s for s in shape if s.startswith("G[")] == ["G[kernel,suminto,kernel,apply,apply]"]
    plan = compiled.plan_for(g, True)
    recipe = [s[2] for s in plan.steps if s[0] == "group"][0]
    views = {p["view"]: p for p in recipe["promoted"]}
    assert views["m"]["cols"] == [0, 1, 2] and not views["m"]["store"]
    assert not any(views["q"]["col_load"].values()) and not views["q"]["store"]       # dead intermediate
    assert not any(views["_d_q"]["col_load"].values())                                   # fresh local: +0.0
    assert all(views["_d_m"]["col_store"].values()) and views["_d_r"]["store"]
    assert not recipe["stage_cols"] and plan.launch_count == 1
    # primal: the flat reduction (its tree interleaves the columns) is folded into the kernel too:
    # the warp's 128 x 3 leaves are three aligned subtrees; q is never stored
    _, shape = _shape(fn, True)
    assert shape == ["declview", "G[kernel+gather]", "return"]
    plan = compiled.plan_for(fn, True)
    recipe = [s[2] for s in plan.steps if s[0] == "group"][0]
    assert recipe["gather_cols"] == 3 and not {p["view"]: p for p in recipe["promoted"]}["q"]["store"]


def test_read_only_neighbour_reads_can_use_a_window(monkeypatch):
    """off by default (measured: no gain), kept selectable"""
    fn, _ = _grad("stencil_smooth")
    an = fusion.Analysis(fn)
    group = [i[1] for i in fusion.form_groups(fusion.build_ops(fn, an, True), an, True) if i[0] == "group"][0]
    assert not group.windowed
    monkeypatch.setattr(fusion, "READONLY_WINDOWS", True)
    group = [i[1] for i in fusion.form_groups(fusion.build_ops(fn, an, True), an, True) if i[0] == "group"][0]
    wp = fusion.window_plan(group.ops, an)
    assert group.windowed and wp.windowed == ["u"] and (wp.hlo, wp.hhi) == (1, 1)
    assert wp.halo == [(0, 0), (0, 0)]  # nothing is recomputed: the window only replaces repeated loads


def test_dead_fills_and_scalars_disappear():
    """the tail of a generated gradient zeroes shadows of locals nobody reads again and reverses
    scalars that are never used: no kernels for those; `dst += src` over whole Views counts over
    the source's extent when that is the open group's range (their extents must agree anyway)"""
    _, g = _grad("copy_chain")
    plan = compiled.plan_for(g)
    groups = [s for s in plan.steps if s[0] == "group"]
    assert plan.launch_count == 1 and len(groups) == 1
    # the forward `deep_copy(t, 0.0)` and `t(i) += ...` only feed the dead forward sum: dropped too
    assert [o.what for o in groups[0][1].ops] == ["deepcopy", "suminto", "kernel", "suminto"]
    stored = [p["view"] for p in groups[0][2]["promoted"] if p["store"]]
    assert stored == ["_d_src"]  # 16 B/row: read src, write _d_src
    fn, g = _grad("mean_shift")
    assert compiled.plan_for(fn).launch_count == 2       # gather, then fill + kernel + gather
    plan = compiled.plan_for(g)
    # forward `total = parallel_sum(v); deep_copy(w, total); w(i) += ...` feeds nothing the reverse sweep
    # reads: what is left is the reversal kernel with its gather, then the broadcast of the gathered scalar
    assert plan.launch_count == 2 and not any(s[0] == "scalars" for s in plan.steps)


def test_dead_statements_that_could_raise_are_kept():
    """a dead kernel whose accesses are not provably in range must still run: it may have to report
    OutOfBounds like the reference (an indirect read, a neighbour read, a shorter View)"""
    p = krn.parse("""fn f(v: view<f64,1>, idx: view<f64,1>, u: view<f64,1>) -> f64 {
        let t: view<f64,1> = view("t", extent(v, 0));
        let w: view<f64,1> = view("w", extent(v, 0));
        parallel_for i in 0..extent(v, 0) { t(i) = v(idx(i)); }
        parallel_for i in 0..extent(v, 0) { w(i) = u(i); }
        parallel_for i in 0..extent(v, 0) { w(i) = v(i) + 1.0; }
        s = parallel_sum(v);
        return s; }""")
    an = fusion.Analysis(p.functions[0])
    ops = fusion.build_ops(p.functions[0], an, True)
    kernels = [op[1] for op in ops if op[0] == "loop" and op[1].what == "kernel"]
    # t(i) = v(idx(i)): indirect read - kept; w(i) = u(i): u may be shorter than v - kept;
    # w(i) = v(i) + 1.0: provably in range and dead - dropped
    assert len(kernels) == 2


def test_a_fill_that_is_read_later_is_kept():
    p = krn.parse("""fn f(v: view<f64,1>) -> f64 {
        let t: view<f64,1> = view("t", extent(v, 0));
        deep_copy(t, 2.0);
        parallel_for i in 0..extent(v, 0) { v(i) = v(i) * t(i); }
        deep_copy(t, 3.0);
        s = parallel_sum(t);
        deep_copy(t, 4.0);
        return s; }""")
    an = fusion.Analysis(p.functions[0])
    ops = fusion.build_ops(p.functions[0], an, True)
    fills = [op[1].origin.src.value for op in ops if op[0] == "loop" and op[1].what == "deepcopy"]
    assert fills == [2.0, 3.0]  # the last one is dead, the others are read


def test_side_reduction_over_a_view_the_group_never_touches():
    """tracked plans keep side reductions in the open group; their source must be promoted even when no
    statement of the group reads or writes it (a fresh zero local) - found by the random-program test"""
    p = krn.parse("""fn f(a: view<f64,1>, b: view<f64,1>, m: view<f64,2>) -> f64 {
        let t0: view<f64,1> = view("t0", extent(a, 0));
        let q: view<f64,2> = view("q", extent(a, 0), extent(m, 1));
        parallel_for i in 0..extent(a, 0) { q(i, 0) = a(i); }
        parallel_for i in 0..extent(a, 0) { a(i) = 0.5 * a(i) + b(i); }
        r = parallel_sum(t0);
        return r; }""")
    plan = compiled.plan_for(p.functions[0], True, True)
    assert plan is not None and plan.launch_count == 1
    # the same shape without the rank-2 local: the plain tile kernel
    p = krn.parse("""fn f(a: view<f64,1>, b: view<f64,1>) -> f64 {
        let t0: view<f64,1> = view("t0", extent(a, 0));
        parallel_for i in 0..extent(a, 0) { a(i) = 0.5 * a(i) + b(i); }
        r = parallel_sum(t0);
        return r; }""")
    plan = compiled.plan_for(p.functions[0], False, True)
    assert plan is not None and plan.launch_count == 1


def test_read_only_stencil_neighbours_become_registers():
    """a read-only View read at i - 1, i, i + 1 under guards is loaded with one 256-bit access per lane;
    the neighbours come from the adjacent lanes (interior steps), the layout stays the vector one"""
    from paper_2507_13204_b200 import tilegen

    fn = krn.load_program("stencil_smooth").functions[0]
    plan = compiled.plan_for(fn, False)
    recipe = [st[2] for st in plan.steps if st[0] == "group"][0]
    u = [p for p in recipe["promoted"] if p["view"] == "u"][0]
    assert u["nbr"] == (1, 1) and u["load"] and not u["store"]
    src = plan.source
    assert "KRN_NBR(P0" in src and "__shfl_up_sync" in src and "#define KRN_IT(e) (j0 + (e))" in src
    assert "u" in recipe["elided_views"]  # the host must verify extent(u) >= n before it launches
    # an unguarded neighbour read has no margin that proves it in range: bounds-checked loads stay
    p = krn.parse("""fn f(u: view<f64,1>) -> f64 {
        let d: view<f64,1> = view("d", extent(u, 0));
        parallel_for i in 0..extent(u, 0) - 1 { d(i) = u(i + 1) - u(i); }
        s = parallel_sum(d);
        return s; }""")
    plan = compiled.plan_for(p.functions[0], False)
    assert "= KRN_NBR(" not in plan.source and "* KRN_NBR(" not in plan.source and "KRN_NBR(P0" not in plan.source


def test_side_reduction_whose_source_a_later_loop_reads_at_neighbours():
    """tracked plans: the dead sum's source is untouched when the reduction joins the group, then a later
    loop reads it at i - 1 / i + 1 (found by the random-program test): no tile kernel with the source
    outside its registers; the window kernel captures the value from global memory"""
    p = krn.parse("""fn f(a: view<f64,1>, b: view<f64,1>) -> f64 {
        let t0: view<f64,1> = view("t0", extent(a, 0));
        let t1: view<f64,1> = view("t1", extent(a, 0));
        parallel_for i in 0..extent(a, 0) { t1(i) = t0(i); if (i != 0) { t1(i) += 1.5 * t0(i - 1); } }
        s0 = parallel_sum(a);
        parallel_for i in 0..extent(a, 0) { t1(i) = a(i); if (i != 0) { t1(i) += 0.125 * a(i - 1); } }
        r = parallel_sum(t0);
        return r; }""")
    for windows in (True, False):
        plan = compiled.plan_for(p.functions[0], windows, True)
        assert plan is not None and plan.launch_count <= 2
