"""CUDA generation for a fused group of loop-shaped statements (fusion.py).

Shape of a tile kernel: every thread owns 4 consecutive iterations j0..j0+3.

    prologue   each *promoted* View (rank 1, touched only at the running index by every
               statement of the group) is read once: one LDG.E.256 on the fast path,
               guarded scalar loads on the ragged tail; a View the host knows to be all
               +0.0 is not read at all (zero_mask bit)
    body       the statements of the group, per iteration, in program order; promoted
               Views are registers, every other access goes through the bounds-checked
               accessors of the statement path; staged atomic contributions go to
               per-site register columns
    epilogue   promoted Views that were written AND are read by anything after the group
               (or belong to the caller) are stored once (STG.E.256); staging columns are
               stored; a trailing `s = parallel_sum(v)` is folded with the reference's
               tree (block partial + last-block final pass, csrc/krn_prelude.cuh)

The generated text only uses helpers of the statement path's preamble and of the
hand-written prelude, and is compiled with the same flags (--fmad=false).
"""

from __future__ import annotations

import re

from .lang import nodes as N
from .lang.dataflow import normalize_index
from .lang.nodes import kind, walk_statements

STRIDE_PAD = 8  # staging columns are padded so that column starts stay 32-byte aligned



# Tree over a warp's steps (`steps` is a power of two <= 16).  After krn_warp_tree* every lane
# holds the node of the step, so lane 0 parks it in shared memory at [warp][step]; the block's
# epilogue folds the 8 * steps parked nodes - consecutive tree nodes, in order - with
# krn_smem_tree.  One predicated STS per step: no registers held across steps and no
# run-time-indexed stack, which the compiler can only keep in local memory (STL/LDL in the step
# loop).  Measured on B200 at 134 M rows against that stack: affine_weighted primal 0.340 -> 0.324 ms,
# sum_squares 0.186 -> 0.180, copy_chain 0.188 -> 0.180, mean_shift 0.367 -> 0.354 (stencil_smooth
# 0.229 -> 0.233, safe_divide 0.256 -> 0.260, headline window kernel unchanged); a binary counter
# in named registers costs the window kernels a block of occupancy (headline primal 0.526 -> 0.597).
_TREE_DECL = "    __shared__ double s_nodes[128];  // [warp][step]: nodes of the block's reduction tree"
_TREE_PUSH = "        if (lane_ == 0) s_nodes[(threadIdx.x >> 5) * steps + t] = node;"
_TREE_SMEM = 128 * 8 + 32 * 8  # s_nodes + krn_final_tree's scratch




class Untrackable(ValueError):
    """check_finite cannot be folded into this fused group (a statement writes a View through
    global memory, or scatters with hardware atomics): the call takes the statement path."""


def _tracked_writes(b, loop, in_kernel) -> tuple:
    """(checkpoint number, Views the statement writes) of one op of a tracked (check_finite) plan;
    every written View must live in registers / windows of the kernel."""
    if any(st.mode != "gather" for st in loop.sites):
        raise Untrackable("hardware-atomic sites")
    if loop.what == "apply":
        written = [loop.apply_of[0]]
    else:
        written = sorted({a.view for a in loop.accesses() if a.write and not a.atomic})
    for v in written:
        if v not in in_kernel:
            raise Untrackable(f"{v} is written through global memory")
    return b.track[id(loop.origin)], written


def _first_access_is_full_store(group, view, ops_with_full_range, col=None) -> bool:
    """True when, in program order, the first statement of the group touching `view`
    (column `col` of it, for a rank-2 View) is an unguarded top-level `view(i) = rhs` whose
    rhs does not read it, in a statement that runs over the whole range of the group."""
    def hit(n):
        if kind(n) != "ViewAccess" or n.view != view:
            return False
        return col is None or (len(n.indices) == 2 and kind(n.indices[1]) == "IntLiteral" and n.indices[1].value == col)

    for loop in group.ops:
        if loop.what == "apply":
            if loop.apply_of[0] == view:
                return False
            continue
        for s in loop.body:  # top level only
            touches = False
            for inner in walk_statements([s]):
                for e in N.statement_exprs(inner):
                    for n in N.walk_expr(e):
                        if hit(n):
                            touches = True
            if not touches:
                continue
            if (kind(s) == "AssignView" and s.op == "=" and hit(s.target) and id(loop) in ops_with_full_range
                    and not any(hit(n) for n in N.walk_expr(s.rhs))):
                return True
            return False
    return False


def _columns(group, view) -> dict:
    """rank-2 View -> {column: written?} over the statements of the group"""
    cols: dict = {}
    for loop in group.ops:
        if loop.what == "apply":
            if loop.apply_of[0] == view:
                for st in loop.apply_of[1]:
                    cols[st.column] = True
            continue
        for a in loop.accesses():
            if a.view == view and len(a.indices) == 2 and kind(a.indices[1]) == "IntLiteral":
                c = a.indices[1].value
                cols[c] = cols.get(c, False) or (a.write and not a.atomic)
    return cols


def plan_group(builder, group, an, live_after: set) -> dict:
    """Decide what is promoted, loaded and stored; returns the recipe dict (without text)."""
    accessed: dict = {}  # view -> [all pointwise?, written?]
    direct_atomic: set = set()
    for loop in group.ops:
        if loop.what == "apply":
            v = loop.apply_of[0]
            e = accessed.setdefault(v, [True, False])
            e[1] = True
            continue
        staged = {st.view for st in loop.sites if st.mode == "gather"}
        for a in loop.accesses():
            if a.atomic and a.view in staged:
                continue
            if a.atomic:
                direct_atomic.add(a.view)
            pw = len(a.indices) == 1 and kind(a.indices[0]) == "Counter" and a.indices[0].name == loop.counter
            e = accessed.setdefault(a.view, [True, False])
            e[0] = e[0] and pw
            e[1] = e[1] or a.write
    if group.gather is not None:
        accessed.setdefault(group.gather[0].src, [True, False])
    for sstmt, _, _ in group.sides:
        accessed.setdefault(sstmt.src, [True, False])
    full_range = {id(l) for l in group.ops if l.shift == 0}
    promoted = []
    for v, (pw, written) in accessed.items():
        if pw and builder.rank.get(v) == 1 and v not in direct_atomic:
            # a local View nothing has touched yet is +0.0 everywhere: nothing to load
            load = not _first_access_is_full_store(group, v, full_range) and v not in group.fresh
            store = written and (v in live_after)
            promoted.append(dict(view=v, load=load, store=store, written=written))
    # Read-only Views read at i + c (|c| <= 4) - stencil neighbours: loaded like a promoted View (one
    # 256-bit access per lane and step); the values beyond the lane's own four come from the adjacent
    # lanes by shuffle, the warp's two ends from global memory.  Interior steps only (the guards'
    # margins must cover the offsets, so that every such read is in range there); the other steps
    # keep the bounds-checked loads.
    if an is not None and group.ops and all(l.what == "kernel" and l.shift == 0 for l in group.ops):
        from .codegen import _unit_affine

        lo_m, up_m = _guard_margins(group, an)
        for v, (pw, written) in accessed.items():
            if pw or written or builder.rank.get(v) != 1 or v in direct_atomic or v in group.fresh:
                continue
            offs = []
            for loop in group.ops:
                for a in loop.accesses():
                    if a.view != v:
                        continue
                    c = _unit_affine(a.indices[0], loop.counter) if len(a.indices) == 1 and not a.atomic else None
                    offs.append(c)
            if offs and all(c is not None and abs(c) <= 4 for c in offs) and -min(offs) <= lo_m and max(offs) <= up_m:
                promoted.append(dict(view=v, load=True, store=False, written=False,
                                     nbr=(max(0, -min(offs)), max(0, max(offs)))))
    stage_cols = []
    for loop in group.ops:
        if loop.what == "kernel":
            stage_cols += [(id(loop), st.index) for st in loop.sites if st.mode == "gather"]
    # thread -> iteration mapping.  "vector": 4 consecutive iterations per thread, promoted Views
    # move with one 256-bit access.  "strided": lane L of a warp takes iterations L, L+32, L+64,
    # L+96 of the warp's 128, so that EVERY access of the form v(i + c) is coalesced (stencil
    # neighbours, staging columns read by an apply loop); chosen when the group has such accesses
    # to Views it cannot promote.
    promoted_names = {p["view"] for p in promoted}
    strided = any(l.what == "apply" for l in group.ops)
    for loop in group.ops:
        if loop.what == "apply":
            continue
        for a in loop.accesses():
            if a.view in promoted_names or len(a.indices) != 1:
                continue
            try:
                const, terms = normalize_index(a.indices[0])
            except (TypeError, ValueError):
                continue
            if terms == ((("counter", loop.counter), 1),):
                strided = True
    if strided and any(p.get("nbr") for p in promoted):
        # neighbour registers are elements of the VECTOR layout; something else forces the strided one
        # (another View read at i + c that cannot be held in registers): plain loads for all of them
        promoted = [p for p in promoted if not p.get("nbr")]
    return dict(promoted=promoted, stage_cols=stage_cols, max_shift=max(l.shift for l in group.ops),
                has_user_ops=any(l.what != "apply" for l in group.ops), strided=strided)


def _specialise_interior_chunks(L: list, start: int, end: int, cond: str, subst: dict) -> None:
    """L[start:end] is the text of the step loop.  Almost every warp's whole chunk (all its steps,
    halo included) lies inside the range, far from both ends; for those warps the per-step
    classification (`full`, `live`, `interior`, tail activity: 64-bit compares on every step) is
    decided ONCE: the loop is emitted twice, the first copy with those flags as compile-time
    constants (the compiler drops every slow-path branch), selected by `cond` per warp."""
    general = L[start:end]
    fast = []
    for line in general:
        for old, new in subst.items():
            if line.strip() == old:
                line = line.replace(old, new)
        fast.append(line)
    L[start:end] = ([f"    const bool chunk_interior_ = {cond};", "    if (chunk_interior_) {"] + fast +
                    ["    } else {"] + general + ["    }"])



_FIN_CALL = re.compile(r"krn_fin\(E, ([^,;]+), ([^;]+)\);")


def _defer_finite_flags(text: str) -> str:
    """check_finite tests of a fused kernel without branches or stores in the element loops: every
    test site ORs one bit into a per-thread mask (an fp64 compare that sets a predicate and a predicated
    LOP3, against test + branch + store per value) and the thread writes the flags of its set bits once,
    when it is done.  Up to 64 distinct (statement, View) flags per kernel; beyond that the immediate
    form stays."""
    slots: list = []
    for m in _FIN_CALL.finditer(text):
        if m.group(1) not in slots:
            slots.append(m.group(1))
    if not slots or len(slots) > 64:
        return text
    text = _FIN_CALL.sub(lambda m: f"KRN_FINB({slots.index(m.group(1))}, {m.group(2)});", text)
    head = text.index("{\n", text.index('extern "C" __global__')) + 2
    flush = ["    if (finbits_) {"]
    flush += [f"        if (finbits_ >> {k} & 1ull) E.fin[{slot}] = 1;" for k, slot in enumerate(slots)]
    flush += ["    }"]
    tail = text.rindex("}")
    return text[:head] + "    unsigned long long finbits_ = 0ull;\n" + text[head:tail] + "\n".join(flush) + "\n" + text[tail:]


def tile_kernel(builder, group, name: str, plan: dict, an=None) -> dict:
    b = builder
    elided: set = set()
    promoted = plan["promoted"]
    regs = {p["view"]: f"P{b.vid(p['view'])}" for p in promoted}
    has_stage = bool(plan["stage_cols"]) or any(l.what == "apply" for l in group.ops)
    gather = group.gather
    L: list = []
    w = L.append
    w(f"#ifndef KRN_MINB_{name}\n#define KRN_MINB_{name}\n#endif")  # see window_kernel
    w(f'extern "C" __global__ void __launch_bounds__(256 KRN_MINB_{name}) {name}(Env E, krn_i64 n, krn_i64 n_launch, '
      "krn_i64 n_safe, unsigned zero_mask, double *stage, krn_i64 ld, double *partials, double *scratch, "
      "unsigned int *ticket, double *red_out, int accumulate, int steps"
      ", double *side_out0, int side_acc0, double *side_out1, int side_acc1)")
    w("{")
    w("    (void)side_out0; (void)side_acc0; (void)side_out1; (void)side_acc1;")
    sides = list(group.sides)
    for j in range(len(sides)):
        w(f"    __shared__ double s_side{j}[128];  // [warp][step]: nodes of side reduction {j}")
    strided = plan["strided"]
    # a warp owns 128*steps consecutive iterations, a block 1024*steps (an aligned power-of-two
    # chunk of the reduction tree); `steps` > 1 amortises block start-up and the block-level
    # combine on bandwidth-bound sizes
    direct = sorted({st.view for l in group.ops for st in l.sites if st.mode == "atomic"})
    from . import codegen
    ordered = codegen.assign_ordered([l.sites for l in group.ops if l.what == "kernel"])
    if direct:
        w("    krn_priv_begin(E);")
    w("    const int lane_ = threadIdx.x & 31;")
    w("    const krn_i64 wbase = ((krn_i64)blockIdx.x * 8 + (threadIdx.x >> 5)) * 128 * steps;")
    w(_TREE_DECL)
    # Memory-level parallelism: the loads of B consecutive steps are issued before the first of them
    # is consumed (a kernel with one or two operand streams otherwise keeps a single 1 KB request per
    # warp in flight; measured on B200: 4.5 -> 6 TB/s for a one-stream reduction).  B shrinks with
    # the number of loaded Views so the register file still holds 3+ blocks per SM.
    nload = sum(1 for p in promoted if p["load"])
    B = 2 if 1 <= nload <= 2 else 1  # measured on B200: 2 gains 1-3%, deeper batches cost occupancy
    # (tracked - check_finite - kernels: B = 1, 2, 4 measured equal within 1 %)
    if (nload == 1 and gather is not None and not any(p["store"] or p.get("nbr") for p in promoted)):
        # one operand stream that ends in the reduction, nothing stored: 4 loads in flight per lane
        # (measured at 134 M rows: sum_squares / copy_chain / fill_scale primal 0.180 -> 0.174 ms; with
        # stores or neighbour registers in the kernel 4 is slower, 8 is slower everywhere)
        B = 4
    if strided:
        w("#define KRN_IT(e) (j0 + (e) * 32 + lane_)")
    else:
        w("#define KRN_IT(e) (j0 + (e))")

    def geometry():
        w("    const int t = t0 + b_;")
        w("    if (t >= steps) break;")
        if strided:
            w("    const krn_i64 j0 = wbase + (krn_i64)t * 128;  // the warp's first iteration of this step")
            w("    const bool full = j0 + 128 <= n_safe;")
        else:
            w("    const krn_i64 j0 = wbase + (krn_i64)t * 128 + 4 * lane_;")
            w("    const bool full = j0 + 4 <= n_safe;")
        w("    const bool live = j0 < n_launch;")

    loop_start = len(L)
    if gather is not None:
        # steps is 1 or 8 (compiled.py): unrolled, so that the step index - and with it the shape of
        # the binary-counter tree over the steps - is known at compile time (registers, no local memory)
        w("#pragma unroll")
        w(f"    for (int tt_ = 0; tt_ < {8 // B}; ++tt_) {{")
        w(f"    const int t0 = tt_ * {B};")
        w("    if (t0 >= steps) break;")
    else:
        w(f"    for (int t0 = 0; t0 < steps; t0 += {B}) {{")
    # ---- prologue: loads of the whole batch -------------------------------------------
    init_tests: list = []  # tested in the compute part: a test right behind its load would serialise the batch's loads
    nbrs = {p["view"]: p["nbr"] for p in promoted if p.get("nbr")}
    # interior step: every iteration of the warp (and every iteration an apply loop looks back or
    # ahead to) lies far enough inside the range for the index guards to be decided at compile time
    LO, UP = _guard_margins(group, an) if an is not None else (0, 0)
    OFF = max([abs(st.offset) for l in group.ops if l.what == "apply" for st in l.apply_of[1]] + [0])
    span = 128 if strided else 4
    interior_line = f"    const bool interior = full && j0 >= {LO + OFF} && j0 + {span + UP + OFF} <= n;"
    for k_, p in enumerate(promoted):
        if p["load"]:
            w(f"    double {regs[p['view']]}b_[{B}][4];")
        if p.get("nbr"):
            w(f"    double {regs[p['view']]}Lb_[{B}][4], {regs[p['view']]}Rb_[{B}][4];  // elements j0-1.., j0+4.. (warp ends)")
    w("#pragma unroll")
    w(f"    for (int b_ = 0; b_ < {B}; ++b_) {{")
    geometry()
    if nbrs:
        w(interior_line)
    for k_, p in enumerate(promoted):
        if not p["load"]:
            continue
        r, v = regs[p["view"]] + "b_[b_]", b.vid(p["view"])
        w(f"    for (int e = 0; e < 4; ++e) {r}[e] = 0.0;")
        w(f"    if (live && !(zero_mask & {1 << k_}u)) {{")
        if strided:
            w(f"        if (full) {{ for (int e = 0; e < 4; ++e) {r}[e] = E.v[{v}][KRN_IT(e)]; }}")
        else:
            # read-only operands take the non-coherent path (LDG.E.256.CONSTANT), read-modify-write ones may not
            ld = "krn_ld4_rmw" if p["written"] else "krn_ld4_stream"
            w(f"        if (full) {{ krn_d4 q = {ld}(E.v[{v}] + j0); {r}[0] = q.a; {r}[1] = q.b; {r}[2] = q.c; {r}[3] = q.d; }}")
        w(f"        else {{ for (int e = 0; e < 4; ++e) if (KRN_IT(e) < E.e0[{v}] && KRN_IT(e) < n_launch) {r}[e] = E.v[{v}][KRN_IT(e)]; }}")
        if b.track is not None and p["view"] not in b.touched_before:  # initial status of a loaded View (checkpoint 0)
            init_tests.append((v, regs[p["view"]]))
            b.init_tested.add(p["view"])
        w("    }")
        if p.get("nbr"):
            # the values just outside the warp's 128 elements: lane 0 / lane 31 fetch them with the
            # batch's other loads (in range on an interior step); the other lanes shuffle (below)
            rs, (na, nb_) = regs[p["view"]], p["nbr"]
            w(f"    for (int e = 0; e < 4; ++e) {{ {rs}Lb_[b_][e] = 0.0; {rs}Rb_[b_][e] = 0.0; }}")
            w(f"    if (interior && !(zero_mask & {1 << k_}u)) {{")
            if na:
                w("        if (lane_ == 0) { " + " ".join(f"{rs}Lb_[b_][{k - 1}] = E.v[{v}][j0 - {k}];" for k in range(1, na + 1)) + " }")
            if nb_:
                w("        if (lane_ == 31) { " + " ".join(f"{rs}Rb_[b_][{k}] = E.v[{v}][j0 + {4 + k}];" for k in range(nb_)) + " }")
            w("    }")
    w("    }")
    # ---- the steps of the batch, one after the other ------------------------------------------
    w("#pragma unroll")
    w(f"    for (int b_ = 0; b_ < {B}; ++b_) {{")
    geometry()
    for p in promoted:
        if p["load"]:
            w(f"    double (&{regs[p['view']]})[4] = {regs[p['view']]}b_[b_];")
        else:
            w(f"    double {regs[p['view']]}[4] = {{0.0, 0.0, 0.0, 0.0}};")
    for (_, idx) in plan["stage_cols"]:
        w(f"    double T{idx}[4] = {{0.0, 0.0, 0.0, 0.0}};")
    for j in range(len(sides)):
        w(f"    double SG{j}[4] = {{0.0, 0.0, 0.0, 0.0}};  // side reduction {j}: the source as it is at that statement")
    for v, r in init_tests:  # (slots that were not loaded hold 0.0)
        w(f"    for (int e = 0; e < 4; ++e) krn_fin(E, {v}, {r}[e]);")
    # ---- body ------------------------------------------------------------------------
    w(interior_line)
    if nbrs:
        # neighbour registers need the whole warp on the fast path (shuffles)
        w("    const bool interior_w = __all_sync(KRN_FULL_MASK, interior);")
        for p in promoted:
            if not p.get("nbr"):
                continue
            r, (na, nb_) = regs[p["view"]], p["nbr"]
            w(f"    double (&{r}L)[4] = {r}Lb_[b_]; double (&{r}R)[4] = {r}Rb_[b_];")
            w("    if (interior_w) {")
            for k in range(1, na + 1):
                w(f"        {{ const double s_ = __shfl_up_sync(KRN_FULL_MASK, {r}[{4 - k}], 1); if (lane_ != 0) {r}L[{k - 1}] = s_; }}")
            for k in range(nb_):
                w(f"        {{ const double s_ = __shfl_down_sync(KRN_FULL_MASK, {r}[{k}], 1); if (lane_ != 31) {r}R[{k}] = s_; }}")
            w("    }")

    def emit_body(interior: bool):
        w("#pragma unroll")
        w("    for (int e = 0; e < 4; ++e) {")
        w("        const krn_i64 i = KRN_IT(e);")
        w("        bool bad = false;")
        if not interior:
            w("        if (i >= n_launch) continue;")
        b.promoted = {v_: r_ for v_, r_ in regs.items() if v_ not in nbrs}
        b.nbr = {v_: regs[v_] for v_ in nbrs} if interior else {}
        try:
            for k_op, loop in enumerate(list(group.ops) + [None]):
                for j, (sstmt, _, pos) in enumerate(sides):
                    if pos == k_op:
                        w(f"        SG{j}[e] = {regs[sstmt.src]}[e];")
                if loop is None:
                    break
                if loop.what == "apply":
                    view, sites, producer = loop.apply_of
                    v, r = b.vid(view), regs.get(view)
                    order = sorted(sites, key=lambda st: (-st.offset, st.index))
                    conds = [f"i < E.e0[{v}]"] if not (interior and r) else []
                    if not interior:
                        conds.append(f"i < n + {loop.shift}")
                    w(f"        if ({' && '.join(conds) if conds else 'true'}) {{  // deferred atomic adds landing on row i, reference order")
                    tgt = f"{r}[e]" if r else f"E.v[{v}][i]"
                    w(f"            double acc = {tgt};")
                    if interior and an is not None:
                        try:
                            b.interior = dict(counter=producer.counter, trip=an.trip(producer.upper), sym=an.trip,
                                              lo=LO, up=UP)
                        except (TypeError, ValueError):
                            b.interior = None
                    try:
                        for st in order:
                            parts = ([] if interior else ["i >= 0", "i < n"]) + \
                                    [b.compare(g, {producer.counter}) for g in st.guards]
                            guard = " && ".join(x for x in parts if x != "(true)") or "true"
                            w(f"            {{ const krn_i64 k_ = i; {{ const krn_i64 i = k_ - ({st.offset}); "
                              f"if ({guard}) acc = acc + stage[{st.index} * ld + i]; }} }}")
                    finally:
                        b.interior = None
                    w(f"            {tgt} = acc;")
                    w("        }")
                    if b.track is not None:
                        cp, written = _tracked_writes(b, loop, regs)
                        for tv in written:
                            w(f"        krn_fin(E, {cp} * NV + {b.vid(tv)}, {regs[tv]}[e]);")
                    continue
                sites = {id(st.stmt): st for st in loop.sites}
                body: list = []
                local = {loop.counter}
                b.counter = loop.counter
                if an is not None:
                    try:
                        trip = an.trip(loop.upper)
                        b.elide = dict(counter=loop.counter, trip=trip, sym=an.trip, views=elided)
                        if interior:
                            b.interior = dict(counter=loop.counter, trip=trip, sym=an.trip, lo=LO, up=UP)
                    except (TypeError, ValueError):
                        b.elide = None
                try:
                    for s in loop.body:
                        b.element(s, local, body, "            ", sites, True)
                finally:
                    b.elide = None
                    b.interior = None
                w("        if (i < n) {" if (plan["max_shift"] and not interior) else "        {")
                L.extend(body)
                w("        }")
                if b.track is not None:
                    cp, written = _tracked_writes(b, loop, regs)
                    for tv in written:
                        w(f"        krn_fin(E, {cp} * NV + {b.vid(tv)}, {regs[tv]}[e]);")
        finally:
            b.promoted = {}
            b.nbr = {}
            b.counter = None
        w("    }")

    w("    if (interior_w) {" if nbrs else "    if (interior) {")
    emit_body(True)
    w("    } else if (live) {")
    emit_body(False)
    w("    }")
    # ---- epilogue -----------------------------------------------------------------------
    for p in promoted:
        if not p["store"]:
            continue
        r, v = regs[p["view"]], b.vid(p["view"])
        w("    if (live) {")
        if strided:
            w(f"        if (full) {{ for (int e = 0; e < 4; ++e) E.v[{v}][KRN_IT(e)] = {r}[e]; }}")
        else:
            w(f"        if (full) {{ krn_d4 q = {{{r}[0], {r}[1], {r}[2], {r}[3]}}; krn_st4(E.v[{v}] + j0, q); }}")
        w(f"        else {{ for (int e = 0; e < 4; ++e) if (KRN_IT(e) < E.e0[{v}] && KRN_IT(e) < n_launch) E.v[{v}][KRN_IT(e)] = {r}[e]; }}")
        w("    }")
    for (_, idx) in plan["stage_cols"]:
        if strided:
            w(f"    if (live) {{ for (int e = 0; e < 4; ++e) if (KRN_IT(e) < n_launch) stage[{idx} * ld + KRN_IT(e)] = T{idx}[e]; }}")
        else:
            w(f"    if (live) {{ krn_d4 q = {{T{idx}[0], T{idx}[1], T{idx}[2], T{idx}[3]}}; krn_st4(stage + {idx} * ld + j0, q); }}")
    if gather is not None:
        src = gather[0].src
        r = regs[src]
        w("    {")
        w("        double R[4];")
        w(f"        if (full) {{ for (int e = 0; e < 4; ++e) R[e] = {r}[e]; }}")
        w("        else { for (int e = 0; e < 4; ++e) R[e] = (KRN_IT(e) < n) ? "
          f"{r}[e] : krn_tree_pad((krn_u64)KRN_IT(e), (krn_u64)n); }}")
        if strided:
            # element e of the 32 lanes = 32 consecutive leaves: four 32-leaf subtrees, then two levels
            w("        double node = krn_warp_tree4(R[0], R[1], R[2], R[3]);")
        else:
            w("        double node = krn_warp_tree((R[0] + R[1]) + (R[2] + R[3]));")
        w(_TREE_PUSH)
        w("    }")
    for j in range(len(sides)):
        w("    {")
        w("        double R[4];")
        w(f"        if (full) {{ for (int e = 0; e < 4; ++e) R[e] = SG{j}[e]; }}")
        w("        else { for (int e = 0; e < 4; ++e) R[e] = (KRN_IT(e) < n) ? "
          f"SG{j}[e] : krn_tree_pad((krn_u64)KRN_IT(e), (krn_u64)n); }}")
        w("        double node = " + ("krn_warp_tree4(R[0], R[1], R[2], R[3]);" if strided else
                                      "krn_warp_tree((R[0] + R[1]) + (R[2] + R[3]));"))
        w(f"        if (lane_ == 0) s_side{j}[(threadIdx.x >> 5) * steps + t] = node;")
        w("    }")
    w("    }  // step of the batch")
    w("    }  // steps")
    _specialise_interior_chunks(
        L, loop_start, len(L),
        f"wbase >= {LO + OFF} && wbase + (krn_i64)128 * steps + {UP + OFF} <= n && wbase + (krn_i64)128 * steps <= n_safe",
        {"const bool full = j0 + 128 <= n_safe;": "const bool full = true;",
         "const bool full = j0 + 4 <= n_safe;": "const bool full = true;",
         "const bool live = j0 < n_launch;": "const bool live = true;",
         f"const bool interior = full && j0 >= {LO + OFF} && j0 + {span + UP + OFF} <= n;": "const bool interior = true;"})
    w("#undef KRN_IT")
    if direct:
        w("    krn_priv_end(E);")
    if gather is not None or sides:
        _emit_reduce_epilogue(w, gather is not None, len(sides), "threadIdx.x >> 5")
    w("}")
    b.parts.append(_defer_finite_flags("\n".join(L)))
    return dict(name=name, promoted=promoted, stage_cols=plan["stage_cols"], has_stage=has_stage,
                gather=gather, max_shift=plan["max_shift"], elided_views=sorted(elided), atomic_views=direct,
                ordered=ordered, static_smem=(_TREE_SMEM if (gather is not None or sides) else 0) + 1024 * len(sides))


def _emit_reduce_epilogue(w, main: bool, nsides: int, warp_expr: str, partial_slots: int = 1):
    """Block partial(s) -> arrival ticket -> the last block folds the partials of every reduction of the
    kernel (the fused gather and the side reductions of a check_finite plan), one after the other."""
    w("    {")
    w(f"        const int warp = {warp_expr};")
    w("        __syncthreads();")
    w("        if (warp == 0) {")
    if main:
        w("            { double v = krn_smem_tree(s_nodes, 8 * steps, lane_); if (lane_ == 0) partials[blockIdx.x] = v; }")
    for j in range(nsides):
        w(f"            {{ double v = krn_smem_tree(s_side{j}, 8 * steps, lane_); "
          f"if (lane_ == 0) partials[(krn_i64)gridDim.x * {partial_slots + j} + blockIdx.x] = v; }}")
    w("        }")
    w("        if (krn_last_block(ticket, gridDim.x)) {")
    if main:
        w("            { double root = krn_final_tree(partials, scratch, gridDim.x);")
        w("              if (threadIdx.x == 0) *red_out = (accumulate ? *red_out : 0.0) + root; }")
    for j in range(nsides):
        w("            __syncthreads();  // krn_final_tree's scratch is reused")
        w(f"            {{ double root = krn_final_tree(partials + (krn_i64)gridDim.x * {partial_slots + j}, scratch, gridDim.x);")
        w(f"              if (threadIdx.x == 0) *side_out{j} = (side_acc{j} ? *side_out{j} : 0.0) + root; }}")
    w("        }")
    w("    }")


# ---------------------------------------------------------------------------------------
# window kernels: groups whose statements exchange values between NEIGHBOURING iterations
# (fusion.window_plan).  Same decomposition as the strided tile kernel - a warp owns 128
# consecutive iterations per step, lane L takes L, L+32, L+64, L+96 - plus one extra slot
# (e = 4) in which the first HLO + HHI lanes re-run the iterations just outside the warp's
# 128 whose results the warp reads.  Views written by one statement and read at i + c by a
# later one live in a warp-private shared-memory window [j0 - HLO, j0 + 128 + HHI); pointwise
# Views stay in registers (5 per lane instead of 4).  No value crosses a warp, so there is no
# block or grid barrier: __syncwarp() between phases is all.  A View that is loaded on halo
# positions and stored by the kernel is written OUT OF PLACE (`alt` pointers; the host swaps
# the buffers afterwards) because the neighbouring warp may still need the old contents.


def plan_window_group(builder, group, an, live_after: set) -> dict:
    from . import fusion

    wp = fusion.window_plan(group.ops, an)
    if wp is None:
        raise ValueError("group has no window plan")
    G = wp.facts
    full_range = {id(l) for l in group.ops if l.shift == 0}
    if group.gather is not None and group.gather[0].src not in G:
        G[group.gather[0].src] = fusion.Facts(rd=True)
    for sstmt, _, _ in group.sides:
        if sstmt.src not in G:
            G[sstmt.src] = fusion.Facts(rd=True)
    promoted, windows = [], []
    for v, f in G.items():
        if v.startswith("__stage"):
            continue
        is_window = v in wp.windowed
        if not is_window and not (f.pw and not f.at):
            continue
        load = not _first_access_is_full_store(group, v, full_range) and v not in group.fresh
        store = f.wr and (v in live_after)
        halo = v in wp.halo_views
        rec = dict(view=v, load=load, store=store, written=f.wr, halo=halo,
                   alt=bool(load and store and (halo or is_window)))
        # an untouched local kept in a window: the window itself must read as +0.0
        rec["zero_init"] = is_window and v in group.fresh and not _first_access_is_full_store(group, v, full_range)
        if builder.rank.get(v) == 2:
            # register columns: each literal column is loaded unless its first access overwrites it,
            # and stored when the group wrote it
            cols = _columns(group, v)
            fresh = v in group.fresh
            rec["cols"] = sorted(cols)
            rec["col_load"] = {c: not fresh and not _first_access_is_full_store(group, v, full_range, c) for c in cols}
            rec["col_store"] = {c: bool(cols[c]) and store for c in cols}
            rec["load"] = any(rec["col_load"].values())
            rec["alt"] = False
        (windows if is_window else promoted).append(rec)
    if sum(1 for r in promoted + windows if r["alt"]) > fusion.MAX_ALT:
        raise ValueError("too many out-of-place outputs")
    stage_cols = []  # columns that travel through global memory (apply loop in another launch)
    for loop in group.ops:
        if loop.what == "kernel":
            for st in loop.sites:
                name = fusion.stage_name(st.index, loop)
                if st.mode == "gather" and name not in wp.stage_windows and name not in wp.stage_regs:
                    stage_cols.append((id(loop), st.index))
    gather_cols = 0
    if group.gather is not None and builder.rank.get(group.gather[0].src) == 2:
        rec = next(p for p in promoted if p["view"] == group.gather[0].src)
        gather_cols = len(rec["cols"])
        if rec["cols"] != list(range(gather_cols)):
            raise ValueError("flat reduction of a rank-2 View needs every column in registers")
    return dict(promoted=promoted, windows=windows, stage_cols=stage_cols, wp=wp,
                max_shift=max(l.shift for l in group.ops), strided=True, window=True, gather_cols=gather_cols)


def _guard_margins(group, an) -> tuple:
    """(lo, up): the largest margins any guard of the group needs to be decided statically
    (`i != 0` -> lo 1, `i < n - 2` -> up 2, ...)."""
    from . import codegen

    lo = up = 0
    for loop in group.ops:
        conds = []
        if loop.what == "apply":
            producer = loop.apply_of[2]
            counter, upper = producer.counter, producer.upper
            for st in loop.apply_of[1]:
                conds += list(st.guards)
        else:
            counter, upper = loop.counter, loop.upper
            for s_ in walk_statements(loop.body):
                if kind(s_) == "If":
                    conds.append(s_.cond)
        try:
            trip = an.trip(upper)
        except (TypeError, ValueError):
            continue
        for c in conds:
            l, u = codegen.guard_interval([c], counter, trip, an.trip)
            lo, up = max(lo, l), max(up, u)
    return lo, up


def window_kernel(builder, group, name: str, plan: dict, an) -> dict:
    from . import fusion

    b, wp = builder, plan["wp"]
    promoted, windows = plan["promoted"], plan["windows"]
    elided: set = set()
    HLO, HHI = wp.hlo, wp.hhi
    WN = 128 + HLO + HHI
    regs = {p["view"]: f"P{b.vid(p['view'])}" for p in promoted}
    wins = {p["view"]: f"W{b.vid(p['view'])}" for p in windows}
    in_kernel_views = set(regs) | set(wins)
    # zero_mask bits / alt pointers: promoted first, then windows
    bit = {p["view"]: k for k, p in enumerate(promoted + windows)}
    alts = [p["view"] for p in promoted + windows if p["alt"]]
    outp = {v: f"alt{k}" for k, v in enumerate(alts)}
    stage_reg_sites, stage_win_sites = set(), {}
    for loop in group.ops:
        if loop.what != "kernel":
            continue
        for st in loop.sites:
            nm = fusion.stage_name(st.index, loop)
            if nm in wp.stage_windows:
                stage_win_sites[st.index] = f"TW{st.index}"
            elif nm in wp.stage_regs or (id(loop), st.index) in plan["stage_cols"]:
                stage_reg_sites.add(st.index)
    gather = group.gather
    direct = sorted({st.view for l in group.ops for st in l.sites if st.mode == "atomic"})
    from . import codegen
    ordered = codegen.assign_ordered([l.sites for l in group.ops if l.what == "kernel"])
    LO, UP = _guard_margins(group, an)
    L: list = []
    w = L.append
    # the occupancy bound is a macro the host may define ahead of the source after looking at the
    # compiled kernel's register count (compiled.retuned_source)
    w(f"#ifndef KRN_MINB_{name}\n#define KRN_MINB_{name}\n#endif")
    w(f'extern "C" __global__ void __launch_bounds__(256 KRN_MINB_{name}) {name}(Env E, krn_i64 n, krn_i64 n_launch, '
      "krn_i64 n_safe, unsigned zero_mask, double *stage, krn_i64 ld, double *partials, double *scratch, "
      "unsigned int *ticket, double *red_out, int accumulate, int steps, double *alt0, double *alt1, "
      "double *alt2, double *alt3, double *side_out0, int side_acc0, double *side_out1, int side_acc1)")
    w("{")
    w("    (void)alt0; (void)alt1; (void)alt2; (void)alt3;")
    w("    (void)side_out0; (void)side_acc0; (void)side_out1; (void)side_acc1;")
    sides = list(group.sides)
    for j in range(len(sides)):
        w(f"    __shared__ double s_side{j}[128];  // [warp][step]: nodes of side reduction {j}")
    w("    const int lane_ = threadIdx.x & 31, warp_ = threadIdx.x >> 5;")
    for wn in list(wins.values()) + list(stage_win_sites.values()):
        w(f"    __shared__ double {wn}_[8][{WN}];")
        w(f"    double *{wn} = {wn}_[warp_];")
    if plan.get("gather_cols"):
        w(f"    __shared__ double G_all_[8][{128 * plan['gather_cols']}];")
        w("    double *G_ = G_all_[warp_];")
        w(f"    __shared__ double s_gn[{64 * plan['gather_cols']}];  // [warp][step][subtree]: the block's tree nodes, in order")
    # which lanes of the halo slot run statement k (it covers [j0 - hlo_k, j0 + 128 + hhi_k))
    for k, (hlo, hhi) in enumerate(wp.halo):
        if hlo or hhi:
            w(f"    const bool h{k}_ = lane_ >= {HLO - hlo} && lane_ < {HLO + hhi};")
    if direct:
        w("    krn_priv_begin(E);")
    w("    const krn_i64 wbase = ((krn_i64)blockIdx.x * 8 + warp_) * 128 * steps;")
    w(_TREE_DECL)
    w("    int wq_[5];  // window position of each slot's iteration")
    w(f"    for (int e = 0; e < 4; ++e) wq_[e] = e * 32 + lane_ + {HLO};")
    w(f"    wq_[4] = lane_ < {HLO} ? lane_ : 128 + lane_;")
    loop_start = len(L)
    w("    for (int t = 0; t < steps; ++t) {")
    w("    const krn_i64 j0 = wbase + (krn_i64)t * 128;  // the warp's first own iteration of this step")
    w(f"    const krn_i64 wlo = j0 - {HLO};                // iteration held by window position 0")
    w("    const bool full = j0 + 128 <= n_safe;")
    w("    const bool live = j0 < n_launch;")
    w("    // interior step: the whole window lies inside the range, far enough from both ends for every")
    w("    // index guard to be decided at compile time")
    w(f"    const bool interior = full && wlo >= {LO} && j0 + {128 + HHI + UP} <= n;")
    w("    krn_i64 it_[5]; bool act_[5];")
    w("    for (int e = 0; e < 4; ++e) { it_[e] = j0 + e * 32 + lane_; act_[e] = live && it_[e] < n_launch; }")
    w(f"    it_[4] = lane_ < {HLO} ? wlo + lane_ : j0 + 128 + (lane_ - {HLO});")
    w(f"    act_[4] = live && lane_ < {HLO + HHI} && it_[4] >= 0 && it_[4] < n_launch;")
    # ---- prologue: registers ------------------------------------------------------------
    late_tests: list = []  # check_finite tests of loaded values: a test right behind its load would serialise the loads
    for p in promoted:
        r, v = regs[p["view"]], b.vid(p["view"])
        if "cols" in p:
            # rank-2 View, rows at the running index: one register column per literal column; the
            # lanes of a warp read rows 24 B (n1 = 3) apart, the columns of a row share its sectors (L1)
            for c in p["cols"]:
                w(f"    double {r}c{c}[5] = {{0.0, 0.0, 0.0, 0.0, 0.0}};")
            lc = [c for c in p["cols"] if p["col_load"][c]]
            if lc:
                w(f"    if (live && !(zero_mask & {1 << bit[p['view']]}u)) {{")
                w(f"        const krn_i64 ld_ = E.e1[{v}];")
                w("        for (int e = 0; e < 4; ++e) {")
                w(f"            if (full || (act_[e] && it_[e] < E.e0[{v}])) {{")
                for c in lc:
                    w(f"                {r}c{c}[e] = E.v[{v}][it_[e] * ld_ + {c}];")
                    if b.track is not None and p["view"] not in b.touched_before:
                        late_tests.append(f"    for (int e = 0; e < 4; ++e) krn_fin(E, {v}, {r}c{c}[e]);")
                w("            }")
                w("        }")
                w("    }")
                if b.track is not None and p["view"] not in b.touched_before:
                    b.init_tested.add(p["view"])
            continue
        w(f"    double {r}[5] = {{0.0, 0.0, 0.0, 0.0, 0.0}};")
        if p["load"]:
            w(f"    if (live && !(zero_mask & {1 << bit[p['view']]}u)) {{")
            w(f"        if (full) {{ for (int e = 0; e < 4; ++e) {r}[e] = E.v[{v}][it_[e]]; }}")
            w(f"        else {{ for (int e = 0; e < 4; ++e) if (act_[e] && it_[e] < E.e0[{v}]) {r}[e] = E.v[{v}][it_[e]]; }}")
            if p["halo"]:
                w(f"        if (act_[4] && it_[4] < E.e0[{v}]) {r}[4] = E.v[{v}][it_[4]];")
            if b.track is not None and p["view"] not in b.touched_before:  # initial status: own rows only (checkpoint 0)
                late_tests.append(f"    for (int e = 0; e < 4; ++e) krn_fin(E, {v}, {r}[e]);")
                b.init_tested.add(p["view"])
            w("    }")
    for idx in sorted(stage_reg_sites):
        w(f"    double T{idx}[5] = {{0.0, 0.0, 0.0, 0.0, 0.0}};")
    for j in range(len(sides)):
        w(f"    double SG{j}[4] = {{0.0, 0.0, 0.0, 0.0}};  // side reduction {j}: the source as it is at that statement")
    # window contents: fetched into registers here so that every global load of the step is in
    # flight before the first one is consumed
    NQ = (WN + 31) // 32
    for p in windows:
        if not p["load"]:
            continue
        wn, v = wins[p["view"]], b.vid(p["view"])
        w(f"    double {wn}r[{NQ}];")
        w("#pragma unroll")
        w(f"    for (int u = 0; u < {NQ}; ++u) {wn}r[u] = 0.0;")
        w(f"    if (live && !(zero_mask & {1 << bit[p['view']]}u)) {{")
        w("        if (interior) {")
        w("#pragma unroll")
        w(f"            for (int u = 0; u < {NQ}; ++u) if (lane_ + 32 * u < {WN}) {wn}r[u] = E.v[{v}][wlo + lane_ + 32 * u];")
        w("        } else {")
        w("#pragma unroll")
        w(f"            for (int u = 0; u < {NQ}; ++u) {{ const krn_i64 g_ = wlo + lane_ + 32 * u; "
          f"if (lane_ + 32 * u < {WN} && g_ >= 0 && g_ < E.e0[{v}] && g_ < n_launch) {wn}r[u] = E.v[{v}][g_]; }}")
        w("        }")
        if b.track is not None and p["view"] not in b.touched_before:  # own positions of the window only: [HLO, HLO + 128)
            late_tests.append("#pragma unroll\n"
                              f"    for (int u = 0; u < {NQ}; ++u) if (lane_ + 32 * u >= {HLO} && lane_ + 32 * u < {HLO + 128}) "
                              f"krn_fin(E, {v}, {wn}r[u]);")
            b.init_tested.add(p["view"])
        w("    }")
    for line in late_tests:  # behind every load of the step (slots that were not loaded hold 0.0)
        w(line)

    def emit_apply(view, sites, producer, interior: bool):
        """`acc = target(row); acc += contributions landing on the row, reference order; target = acc`,
        once per literal column for a rank-2 target."""
        v = b.vid(view)
        order = sorted(sites, key=lambda st: (-st.offset, st.index))
        try:
            ptrip = an.trip(producer.upper)
        except (TypeError, ValueError):
            ptrip = None
        rank2 = b.rank.get(view) == 2
        for col in (sorted({st.column for st in sites}) if rank2 else [None]):
            if rank2 and view in regs:
                tgt, head = f"{regs[view]}c{col}[e]", "{"
            elif rank2:
                tgt, head = f"E.v[{v}][i * E.e1[{v}] + {col}]", f"if ({col} < E.e1[{v}]) {{"
            elif view in regs:
                tgt, head = f"{regs[view]}[e]", "{"
            elif view in wins:
                tgt, head = f"{wins[view]}[wq]", "{"
            else:
                tgt, head = f"E.v[{v}][i]", "{"
            w(f"            {head}")
            w(f"            double acc = {tgt};")
            if interior and ptrip is not None:
                b.interior = dict(counter=producer.counter, trip=ptrip, sym=an.trip, lo=LO, up=UP)
            try:
                for st in order:
                    if rank2 and st.column != col:
                        continue
                    parts = ([] if interior else ["i >= 0", "i < n"]) + \
                            [b.compare(g, {producer.counter}) for g in st.guards]
                    guard = " && ".join(x for x in parts if x != "(true)") or "true"
                    nm = fusion.stage_name(st.index, producer)
                    if nm in wp.stage_windows:
                        src = f"TW{st.index}[wq - ({st.offset})]"
                    elif nm in wp.stage_regs:
                        src = f"T{st.index}[e]"
                    else:
                        src = f"stage[{st.index} * ld + i]"
                    w(f"            {{ const krn_i64 k_ = i; {{ const krn_i64 i = k_ - ({st.offset}); (void)i; "
                      f"if ({guard}) acc = acc + {src}; }} }}")
            finally:
                b.interior = None
            w(f"            {tgt} = acc;")
            w("            }")

    def emit_side_capture(position):
        """side reductions that sit before op `position`: copy the source's current value (own slots)"""
        for j, (sstmt, _, pos) in enumerate(sides):
            if pos == position:
                if sstmt.src in regs:
                    val = f"{regs[sstmt.src]}[e]"
                elif sstmt.src in wins:
                    val = f"{wins[sstmt.src]}[wq]"
                else:
                    # a View the group only reads, at i + c somewhere (global loads): its own row, in range
                    # because the reduction's extent IS the group's trip count
                    val = f"E.v[{b.vid(sstmt.src)}][i]"
                w(f"        if (e < 4) SG{j}[e] = {val};")

    def emit_tests(loop):
        """check_finite plans: the Views this statement wrote, tested on the iteration's own slot"""
        if b.track is None:
            return
        cp, written = _tracked_writes(b, loop, in_kernel_views)
        for tv in written:
            v = b.vid(tv)
            if tv in wins:
                w(f"        if (e < 4) krn_fin(E, {cp} * NV + {v}, {wins[tv]}[wq]);")
                continue
            rec = next(p for p in promoted if p["view"] == tv)
            if "cols" in rec:
                cols = sorted(c for c, wr in _columns(type("G", (), {"ops": [loop]})(), tv).items() if wr) \
                    if loop.what != "apply" else sorted({st.column for st in loop.apply_of[1]})
                for c in cols:
                    w(f"        if (e < 4) krn_fin(E, {cp} * NV + {v}, {regs[tv]}c{c}[e]);")
            else:
                w(f"        if (e < 4) krn_fin(E, {cp} * NV + {v}, {regs[tv]}[e]);")

    def emit_step(interior: bool):
        # ---- windows in (values were fetched into registers by the prologue, all loads in flight at once)
        loaded = False
        for p in windows:
            if p["zero_init"]:
                loaded = True
                w(f"    for (int q = lane_; q < {WN}; q += 32) {wins[p['view']]}[q] = 0.0;")
            if not p["load"]:
                continue
            loaded = True
            wn = wins[p["view"]]
            w("#pragma unroll")
            w(f"    for (int u = 0; u < {NQ}; ++u) if (lane_ + 32 * u < {WN}) {wn}[lane_ + 32 * u] = {wn}r[u];")
        if loaded:
            w("    __syncwarp();")
        # ---- phases ----------------------------------------------------------------------------
        b.promoted, b.windows, b.stage_windows, b.in_tile = regs, wins, stage_win_sites, True
        try:
            for phase in wp.phases:
                slots = 5 if any(wp.halo[k] != (0, 0) for k in phase) else 4
                w("#pragma unroll")
                w(f"    for (int e = 0; e < {slots}; ++e) {{")
                if interior:
                    if slots == 5:
                        w(f"        if (e == 4 && lane_ >= {HLO + HHI}) continue;")
                else:
                    w("        if (!act_[e]) continue;")
                w("        const krn_i64 i = it_[e];")
                w("        const int wq = wq_[e]; (void)wq;")
                w("        bool bad = false;")
                for k in phase:
                    emit_side_capture(k)
                    loop = group.ops[k]
                    hlo, hhi = wp.halo[k]
                    conds = []
                    if slots == 5:
                        conds.append(f"(e < 4 || h{k}_)" if (hlo or hhi) else "e < 4")
                    if loop.what == "apply":
                        view, sites, producer = loop.apply_of
                        v = b.vid(view)
                        if not interior:
                            conds.append(f"i < n + {loop.shift}")
                        if not (interior and view in in_kernel_views):
                            conds.append(f"i < E.e0[{v}]")
                        w(f"        if ({' && '.join(conds) if conds else 'true'}) {{  // deferred atomic adds landing on row i, reference order")
                        emit_apply(view, sites, producer, interior)
                        w("        }")
                        emit_tests(loop)
                        continue
                    sites = {id(st.stmt): st for st in loop.sites}
                    body: list = []
                    local = {loop.counter}
                    b.counter = loop.counter
                    try:
                        trip = an.trip(loop.upper)
                        b.elide = dict(counter=loop.counter, trip=trip, sym=an.trip, views=elided)
                        if interior:
                            b.interior = dict(counter=loop.counter, trip=trip, sym=an.trip, lo=LO, up=UP)
                    except (TypeError, ValueError):
                        b.elide = None
                    try:
                        for s_ in loop.body:
                            b.element(s_, local, body, "            ", sites, True)
                    finally:
                        b.elide = None
                        b.interior = None
                        b.counter = None
                    if plan["max_shift"] and not interior:
                        conds.append("i < n")
                    # `continue` inside the body must only leave this statement's block
                    w(f"        if ({' && '.join(conds) if conds else 'true'}) do {{")
                    L.extend(x.replace("continue;", "break;") for x in body)
                    w("        } while (0);")
                    w("        if (bad) continue;")
                    emit_tests(loop)
                if phase is wp.phases[-1]:
                    emit_side_capture(len(group.ops))
                w("    }")
                w("    __syncwarp();")
        finally:
            b.promoted, b.windows, b.stage_windows, b.in_tile = {}, {}, {}, False
        # ---- windows out ---------------------------------------------------------------------------
        for p in windows:
            if not p["store"]:
                continue
            wn, v = wins[p["view"]], b.vid(p["view"])
            dst = outp.get(p["view"], f"E.v[{v}]")
            if interior:
                w(f"    for (int e = 0; e < 4; ++e) {dst}[it_[e]] = {wn}[wq_[e]];")
            else:
                w(f"    for (int e = 0; e < 4; ++e) if (act_[e] && it_[e] < E.e0[{v}]) {dst}[it_[e]] = {wn}[wq_[e]];")

    w("    if (interior) {")
    emit_step(True)
    w("    } else if (live) {")
    emit_step(False)
    w("    }")
    # ---- epilogue ---------------------------------------------------------------------------------
    for p in promoted:
        if not p["store"]:
            continue
        r, v = regs[p["view"]], b.vid(p["view"])
        if "cols" in p:
            sc = [c for c in p["cols"] if p["col_store"][c]]
            if sc:
                w("    if (live) {")
                w(f"        const krn_i64 ld_ = E.e1[{v}];")
                w("        for (int e = 0; e < 4; ++e) {")
                w(f"            if (full || (act_[e] && it_[e] < E.e0[{v}])) {{")
                for c in sc:
                    w(f"                E.v[{v}][it_[e] * ld_ + {c}] = {r}c{c}[e];")
                w("            }")
                w("        }")
                w("    }")
            continue
        dst = outp.get(p["view"], f"E.v[{v}]")
        w("    if (live) {")
        w(f"        if (full) {{ for (int e = 0; e < 4; ++e) {dst}[it_[e]] = {r}[e]; }}")
        w(f"        else {{ for (int e = 0; e < 4; ++e) if (act_[e] && it_[e] < E.e0[{v}]) {dst}[it_[e]] = {r}[e]; }}")
        w("    }")
    for (_, idx) in plan["stage_cols"]:
        w(f"    if (live) {{ for (int e = 0; e < 4; ++e) if (act_[e]) stage[{idx} * ld + it_[e]] = T{idx}[e]; }}")
    gcols = plan.get("gather_cols", 0)
    if gather is not None and gcols:
        # flat reduction of a rank-2 View (leaf index = row * C + column): the warp's 128 x C leaves
        # are laid out in flat order in shared memory; they are C aligned 128-leaf subtrees of the
        # reference's tree over the flattened buffer (runtime.py:643-651: pairwise_sum(view.flat))
        src, r = gather[0].src, regs[gather[0].src]
        w("    {")
        w("        for (int e = 0; e < 4; ++e) {")
        w("            const bool in_ = full || it_[e] < n;")
        for c in range(gcols):
            w(f"            G_[(e * 32 + lane_) * {gcols} + {c}] = in_ ? {r}c{c}[e] : "
              f"krn_tree_pad((krn_u64)(it_[e] * {gcols} + {c}), (krn_u64)(n * {gcols}));")
        w("        }")
        w("        __syncwarp();")
        for k in range(gcols):
            w(f"        {{ const double nd_ = krn_warp_tree4(G_[{128 * k} + lane_], G_[{128 * k + 32} + lane_], "
              f"G_[{128 * k + 64} + lane_], G_[{128 * k + 96} + lane_]); "
              f"if (lane_ == 0) s_gn[(warp_ * steps + t) * {gcols} + {k}] = nd_; }}")
        w("    }")
    elif gather is not None:
        src = gather[0].src
        w("    {")
        w("        double R[4];")
        val = f"{regs[src]}[e]" if src in regs else f"{wins[src]}[wq_[e]]"
        w(f"        if (full) {{ for (int e = 0; e < 4; ++e) R[e] = {val}; }}")
        w(f"        else {{ for (int e = 0; e < 4; ++e) R[e] = (it_[e] < n) ? {val} : krn_tree_pad((krn_u64)it_[e], (krn_u64)n); }}")
        w("        double node = krn_warp_tree4(R[0], R[1], R[2], R[3]);")
        w(_TREE_PUSH)
        w("    }")
    for j in range(len(sides)):
        w("    {")
        w("        double R[4];")
        w(f"        if (full) {{ for (int e = 0; e < 4; ++e) R[e] = SG{j}[e]; }}")
        w(f"        else {{ for (int e = 0; e < 4; ++e) R[e] = (it_[e] < n) ? SG{j}[e] : krn_tree_pad((krn_u64)it_[e], (krn_u64)n); }}")
        w("        double node = krn_warp_tree4(R[0], R[1], R[2], R[3]);")
        w(f"        if (lane_ == 0) s_side{j}[warp_ * steps + t] = node;")
        w("    }")
    w("    __syncwarp();")
    w("    }  // steps")
    _specialise_interior_chunks(
        L, loop_start, len(L),
        f"wbase >= {LO + HLO} && wbase + (krn_i64)128 * steps + {HHI + UP} <= n && wbase + (krn_i64)128 * steps <= n_safe",
        {"const bool full = j0 + 128 <= n_safe;": "const bool full = true;",
         "const bool live = j0 < n_launch;": "const bool live = true;",
         f"const bool interior = full && wlo >= {LO} && j0 + {128 + HHI + UP} <= n;": "const bool interior = true;",
         "for (int e = 0; e < 4; ++e) { it_[e] = j0 + e * 32 + lane_; act_[e] = live && it_[e] < n_launch; }":
             "for (int e = 0; e < 4; ++e) { it_[e] = j0 + e * 32 + lane_; act_[e] = true; }",
         f"act_[4] = live && lane_ < {HLO + HHI} && it_[4] >= 0 && it_[4] < n_launch;": f"act_[4] = lane_ < {HLO + HHI};"})
    if direct:
        w("    krn_priv_end(E);")
    if gather is not None and gcols:
        C_ = gcols
        w("    {")
        # lane 0 of every warp parked its C x steps nodes at [warp][step][subtree]: 8 * steps * C
        # consecutive nodes of the tree, in order.  Warp 0 folds log2(8 * steps) levels, every level
        # in parallel (read all pairs, then write), down to the block's C nodes.
        w("        __syncthreads();")
        w("        if (warp_ == 0) {")
        w(f"            for (int cnt = {8 * C_} * steps; cnt > {C_}; cnt >>= 1) {{")
        w(f"                double pair_[{C_}];")
        w("#pragma unroll")
        w(f"                for (int u = 0; u < {C_}; ++u) {{ const int i = lane_ + 32 * u; "
          "if (i < cnt / 2) pair_[u] = s_gn[2 * i] + s_gn[2 * i + 1]; }")
        w("                __syncwarp();")
        w("#pragma unroll")
        w(f"                for (int u = 0; u < {C_}; ++u) {{ const int i = lane_ + 32 * u; "
          "if (i < cnt / 2) s_gn[i] = pair_[u]; }")
        w("                __syncwarp();")
        w("            }")
        w(f"            if (lane_ < {C_}) partials[(krn_i64)blockIdx.x * {C_} + lane_] = s_gn[lane_];")
        w("        }")
        w("        if (krn_last_block(ticket, gridDim.x)) {")
        w("            // nodes past the end of the flattened View were computed from padding leaves and equal")
        w("            // the padding of the tree over the partials: only the real ones are folded")
        w(f"            const krn_u64 span_ = (krn_u64)1024 * steps, m_ = ((krn_u64)n * {C_} + span_ - 1) / span_;")
        w("            double root = krn_final_tree(partials, scratch, m_);")
        w("            if (threadIdx.x == 0) *red_out = (accumulate ? *red_out : 0.0) + root;")
        w("        }")
        w("    }")
    elif gather is not None or sides:
        _emit_reduce_epilogue(w, gather is not None, len(sides), "warp_")
    w("}")
    b.parts.append(_defer_finite_flags("\n".join(L)))
    every = promoted + windows
    return dict(name=name, promoted=every, stage_cols=plan["stage_cols"], has_stage=bool(plan["stage_cols"]),
                gather=gather, max_shift=plan["max_shift"],
                elided_views=sorted(elided | {p["view"] for p in windows}), atomic_views=direct, ordered=ordered,
                window=True, alt=alts, hlo=HLO, hhi=HHI, gather_cols=gcols,
                static_smem=8 * 8 * WN * (len(wins) + len(stage_win_sites))
                + (_TREE_SMEM if (gather is not None or sides) else 0) + 1024 * len(sides) + 8 * (8 * 128 + 8) * gcols)
