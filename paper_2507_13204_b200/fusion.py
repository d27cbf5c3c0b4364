"""Automatic fusion of a function's statements into fewer, wider kernels
(the paper lists kernel fusion as future work,
PAPER.md:837).

The statement path (one launch per statement, like the reference's interpreter
and like Kokkos) moves every intermediate View through HBM.  This pass keeps
the reference's semantics bit for bit and removes the traffic that is only an
artefact of statement granularity:

* consecutive loop-shaped statements over the same range are merged into one
  kernel when every View they share is touched *pointwise* (always at the
  running index), so a value written by one statement and read by the next
  travels in a register;
* Views that are pointwise in a group are loaded once with a 256-bit access,
  kept in registers, and stored once - or not at all when nothing after the
  group reads them (dead intermediates such as ``y2``);
* zero-initialised Views (``DeclView``, ``ViewStorage.zeros``) are never
  materialised ahead of a kernel that only touches them pointwise: the kernel is
  told they read as +0.0;
* ``s = parallel_sum(v)`` fuses into the kernel that produces ``v`` (the block
  tree of csrc/krn_prelude.cuh), and disappears when ``s`` is never read (the
  verbatim forward reduction inside a generated gradient);
* function-scope scalars whose value the host can know (literals, parameters and
  arithmetic on them: seeds, ``base = c*c``) are evaluated on the host and passed
  as kernel arguments instead of running one-thread kernels.

Deferred ``atomic_add`` keeps its two policies (codegen.plan_atomics).  In gather
mode the staging columns are ordinary pointwise Views of the producing group, and
the apply loop is a synthetic statement that may itself fuse with what follows
(e.g. the reversal of the in-place scale kernel).

Fusion legality (what "pointwise" buys): iterations of a ``parallel_for`` are
independent, and a kernel boundary is only observable through a View that some
iteration reads or writes at an index other than its own.  If every shared View
is accessed at exactly the running index by both statements, iteration i of the
second statement depends only on iteration i of the first, and running them back
to back inside one thread is indistinguishable from two launches.

Anything outside the supported shape (rank-2 Views, staged atomics, differing
ranges) simply stays an unfused statement and runs through the statement path.
"""

from __future__ import annotations

import dataclasses as _dc

from . import codegen
from .lang import nodes as N
from .lang.dataflow import normalize_index
from .lang.nodes import kind, walk_expr, walk_statements

K = "__k"  # counter of synthetic loops


@_dc.dataclass
class Access:
    view: str
    indices: tuple
    write: bool
    atomic: bool = False


@_dc.dataclass
class LoopOp:
    """A loop-shaped statement: a parallel_for, a bulk builtin rewritten as one, or
    the apply loop of gather-mode atomics."""

    counter: str
    upper: object  # index expression (trip count)
    body: tuple
    origin: object  # the source statement (for shape checks / fallback)
    what: str  # "kernel" | "deepcopy" | "suminto" | "apply"
    sites: list = _dc.field(default_factory=list)  # atomic sites of a kernel
    apply_of: object = None  # (view, sites) for an apply loop
    shift: int = 0  # apply loops run over upper + shift rows
    need_cols: dict = _dc.field(default_factory=dict)  # rank-2 bulk statements: view -> exact extent 1 assumed

    def accesses(self) -> list:
        out: list = []

        def index_accesses(e):
            for n in walk_expr(e):
                if kind(n) == "ViewAccess":
                    out.append(Access(n.view, tuple(n.indices), False))

        def value(e):
            for n in walk_expr(e):
                if kind(n) == "ViewAccess":
                    out.append(Access(n.view, tuple(n.indices), False))

        for s in walk_statements(self.body):
            k = kind(s)
            if k == "AssignView":
                out.append(Access(s.target.view, tuple(s.target.indices), True))
                if s.op != "=":
                    out.append(Access(s.target.view, tuple(s.target.indices), False))
                for i in s.target.indices:
                    index_accesses(i)
                value(s.rhs)
            elif k == "AtomicAdd":
                out.append(Access(s.target.view, tuple(s.target.indices), True, True))
                for i in s.target.indices:
                    index_accesses(i)
                value(s.value)
            elif k == "DeclScalar":
                value(s.init)
            elif k == "AssignScalar":
                value(s.rhs)
        return out


def guarded_accesses(loop: "LoopOp") -> list:
    """(Access, guards) for every access of a user loop: the enclosing If conditions decide
    which neighbour reads are provably in range."""
    out: list = []

    def reads(e, guards):
        for n in walk_expr(e):
            if kind(n) == "ViewAccess":
                out.append((Access(n.view, tuple(n.indices), False), guards))

    def walk(body, guards):
        for s in body:
            k = kind(s)
            if k == "If":
                walk(s.body, guards + (s.cond,))
            elif k == "AssignView":
                out.append((Access(s.target.view, tuple(s.target.indices), True), guards))
                if s.op != "=":
                    out.append((Access(s.target.view, tuple(s.target.indices), False), guards))
                for i in s.target.indices:
                    reads(i, guards)
                reads(s.rhs, guards)
            elif k == "AtomicAdd":
                out.append((Access(s.target.view, tuple(s.target.indices), True, True), guards))
                for i in s.target.indices:
                    reads(i, guards)
                reads(s.value, guards)
            elif k == "DeclScalar":
                reads(s.init, guards)
            elif k == "AssignScalar":
                reads(s.rhs, guards)

    walk(loop.body, ())
    return out


def group_columns(ops: list, view: str) -> set:
    """Literal columns with which the loops of a group touch rank-2 `view` (apply targets included)."""
    cols: set = set()
    for loop in ops:
        if loop.what == "apply":
            if loop.apply_of[0] == view:
                cols |= {st.column for st in loop.apply_of[1]}
            continue
        for a in loop.accesses():
            if a.view == view and len(a.indices) == 2 and kind(a.indices[1]) == "IntLiteral":
                cols.add(a.indices[1].value)
    return cols


def stage_name(index: int, producer) -> str:
    return f"__stage{index}@{id(producer)}"


MAX_HALO = 32      # halo iterations of a warp step are handled by the 32 lanes in one extra slot
MAX_WINDOWS = 5    # 8 warps x (128 + halo) doubles each: 5 windows stay under 48 KB of static shared memory
MAX_ALT = 4        # out-of-place output pointers a window kernel accepts
MAX_GATHER_COLS = 4  # a fused flat reduction of a rank-2 View stages 128 x C leaves per warp in shared memory
# Also serve neighbour reads of READ-ONLY Views from a window.  Measured on B200 (stencil_smooth,
# 67 M rows): no gain for the primal, -10% for the gradient - the three L1-cached loads per row are
# all in flight at once, the window adds a shared-memory round trip - so it stays off.
READONLY_WINDOWS = False


@_dc.dataclass
class Facts:
    """How one loop (or a whole group) touches one View."""

    pw: bool = True        # every access at exactly the running index
    wr: bool = False
    at: bool = False       # direct (non-staged) atomic target
    affine: bool = True    # every access is `counter + c` on a rank-1 View, writes at c = 0, reads proven in range
    offsets: frozenset = frozenset()
    rd: bool = False
    direct: bool = False   # touched ONLY by "direct" atomic sites (one writing iteration per location)

    def merged(self, o: "Facts") -> "Facts":
        return Facts(self.pw and o.pw, self.wr or o.wr, self.at or o.at, self.affine and o.affine,
                     self.offsets | o.offsets, self.rd or o.rd, self.direct and o.direct)


def loop_facts(loop: "LoopOp", an: "Analysis") -> dict:
    """view -> Facts; staging columns of gather-mode atomics appear as pseudo views
    (`stage_name`): written pointwise by the producer, read at -offset by the apply loop."""
    out: dict = {}

    def note(view, pw, wr, at, affine, c, rd, direct=False):
        f = out.get(view, Facts(direct=True))
        offs = f.offsets | ({c} if c is not None else set())
        out[view] = Facts(f.pw and pw, f.wr or wr, f.at or at, f.affine and affine, frozenset(offs), f.rd or rd,
                          f.direct and direct)

    if loop.what == "apply":
        view, sites, producer = loop.apply_of
        note(view, True, True, False, True, 0, True)
        for st in sites:
            note(stage_name(st.index, producer), st.offset == 0, False, False, True, -st.offset, True)
        return out
    try:
        trip = an.trip(loop.upper)
    except (TypeError, ValueError):
        trip = None
    staged_views = {st.view for st in loop.sites if st.mode == "gather"}
    direct_views = {st.view for st in loop.sites if st.mode == "direct"}
    for st in loop.sites:
        if st.mode == "gather":
            note(stage_name(st.index, loop), True, True, False, True, 0, False)
    for a, guards in guarded_accesses(loop):
        if a.atomic and a.view in staged_views:
            continue
        if a.atomic and a.view in direct_views:
            note(a.view, False, True, True, False, None, False, direct=True)
            continue
        pw = _is_pointwise(a, loop.counter)
        c = codegen._unit_affine(a.indices[0], loop.counter) if len(a.indices) == 1 else None
        affine = c is not None and an.rank.get(a.view, 1) == 1
        if pw and len(a.indices) == 2:
            affine, c = True, 0  # rank-2 row at the running index, literal column: register columns
        if affine and c != 0:
            if a.write or trip is None:
                affine = False
            else:
                lo, up = codegen.guard_interval(guards, loop.counter, trip, an.trip)
                affine = lo + c >= 0 and c - up <= 0
        note(a.view, pw, a.write, a.atomic, affine, c if affine else None, not a.write)
    return out


@_dc.dataclass
class WindowPlan:
    halo: list            # per op: (lo, hi) iterations it runs beyond the warp's own 128
    hlo: int              # window geometry: positions [j0 - hlo, j0 + 128 + hhi)
    hhi: int
    windowed: list        # Views kept in warp-private shared-memory windows
    stage_windows: list   # staging pseudo views kept in windows (read by a neighbour row)
    stage_regs: list      # staging pseudo views kept in registers (read by the same row)
    halo_views: set       # Views touched by an op that runs on halo iterations
    phases: list          # op indices, split where a window written by one op is read at an offset by the next
    facts: dict           # group-level Facts
    rank2: list = _dc.field(default_factory=list)  # rank-2 Views kept as register columns

    @property
    def needed(self) -> bool:
        return bool(self.windowed or self.stage_windows or self.stage_regs or self.rank2)


def window_plan(ops: list, an: "Analysis"):
    """Halo-recompute plan for running `ops` back to back in ONE kernel although some View
    written by one of them is read at a neighbouring index by a later one (stencil after an
    in-place update, deferred atomics gathered by the rows they land on).  Every warp owns
    128 consecutive iterations per step and recomputes the few iterations of its neighbours
    whose results it reads, so no value crosses a warp and no grid-wide barrier is needed.
    None when the shape is outside what the window kernel supports."""
    per = [loop_facts(o, an) for o in ops]
    G: dict = {}
    for f in per:
        for v, x in f.items():
            G[v] = G[v].merged(x) if v in G else x
    # (a View reached only through "direct" atomic sites is updated in global memory by its one
    # writing iteration - own iterations only, see below - and takes no part in the windows)
    windowed = [v for v, f in G.items() if f.wr and not f.pw and not v.startswith("__stage") and not f.direct]
    for v in windowed:
        f = G[v]
        if not f.affine or f.at or an.rank.get(v) != 1:
            return None
    # read-only Views read at neighbouring rows: one coalesced window load instead of one load per
    # neighbour (optional: dropped first when the kernel runs out of windows)
    readonly = [v for v, f in G.items() if not f.wr and not f.pw and f.affine and not f.at
                and an.rank.get(v, 1) == 1 and not v.startswith("__stage")] if READONLY_WINDOWS else []
    stage_w, stage_r = [], []
    for v, f in G.items():
        if v.startswith("__stage") and f.wr and f.rd:   # producer and apply loop in the same group
            (stage_r if f.pw else stage_w).append(v)
    promoted = {v for v, f in G.items() if f.pw and not f.at}
    in_kernel = promoted | set(windowed) | set(stage_w) | set(stage_r)
    m = len(ops)
    H = [[0, 0] for _ in ops]
    for k in range(m - 1, -1, -1):
        hlo, hhi = H[k]
        for v, f in per[k].items():
            if not f.rd or v not in in_kernel:
                continue
            for c in (f.offsets or {0}):
                for p in range(k):
                    if v in per[p] and per[p][v].wr:
                        H[p][0] = max(H[p][0], hlo - c)
                        H[p][1] = max(H[p][1], hhi + c)
    HLO = max(h[0] for h in H)
    HHI = max(h[1] for h in H)
    halo_views: set = set()
    for k, (hlo, hhi) in enumerate(H):
        if hlo == 0 and hhi == 0:
            continue
        # an op that runs on halo iterations must leave no trace outside registers and windows
        # ("direct" sites write global memory, but only from the iteration's OWN slot: codegen guards
        # them with e < 4 inside window kernels, so re-running the statement on halo rows is harmless)
        if any(st.mode not in ("gather", "direct") for st in ops[k].sites):
            return None
        for v, f in per[k].items():
            if f.wr and v not in in_kernel and not f.direct:
                return None
            halo_views.add(v)
    for k, (hlo, hhi) in enumerate(H):
        for v, f in per[k].items():
            if v in windowed or v in stage_w:
                for c in f.offsets:
                    HLO, HHI = max(HLO, hlo - c), max(HHI, hhi + c)
    if len(windowed) + len(stage_w) > MAX_WINDOWS:
        return None
    readonly = sorted(readonly)[:MAX_WINDOWS - len(windowed) - len(stage_w)]
    for k, (hlo, hhi) in enumerate(H):
        for v, f in per[k].items():
            if v in readonly:
                for c in f.offsets:
                    HLO, HHI = max(HLO, hlo - c), max(HHI, hhi + c)
    if HLO + HHI > MAX_HALO:
        return None
    windowed = windowed + readonly
    # phases: a __syncwarp() separates an op from an earlier one when a window carries a value
    # between different lanes (read-after-write or write-after-read at a non-zero offset)
    phases, cur, written, read_off = [], [], set(), set()
    for k in range(m):
        reads_k = {v for v, f in per[k].items() if (v in windowed or v in stage_w) and f.rd and any(c != 0 for c in f.offsets)}
        writes_k = {v for v, f in per[k].items() if (v in windowed or v in stage_w) and f.wr}
        if cur and ((reads_k & written) or (writes_k & read_off)):
            phases.append(cur)
            cur, written, read_off = [], set(), set()
        cur.append(k)
        written |= writes_k
        read_off |= reads_k
    if cur:
        phases.append(cur)
    rank2 = sorted(v for v in promoted if an.rank.get(v, 1) == 2)
    return WindowPlan([tuple(h) for h in H], HLO, HHI, sorted(windowed), sorted(stage_w), sorted(stage_r),
                      halo_views, phases, G, rank2)


def _is_pointwise(acc: Access, counter: str) -> bool:
    """the running row: v(i), or v(i, c) with a literal column c >= 0"""
    if not acc.indices or kind(acc.indices[0]) != "Counter" or acc.indices[0].name != counter:
        return False
    if len(acc.indices) == 1:
        return True
    return len(acc.indices) == 2 and kind(acc.indices[1]) == "IntLiteral" and acc.indices[1].value >= 0


@_dc.dataclass
class Group:
    ops: list
    gather: object = None  # (ParallelSum stmt, accumulate) fused at the end
    promoted: dict = _dc.field(default_factory=dict)  # view -> dict(load=, store=, written=)
    name: str = ""
    fresh: frozenset = frozenset()  # local Views still untouched (all +0.0) when the group starts
    windowed: bool = False  # formed through window_plan: runs as a window kernel (tilegen.window_kernel)
    # check_finite plans: gathers whose result nothing reads (the dead forward sum of a gradient) but whose
    # value the reference checks - reduced as a SIDE output of the kernel, which goes on:
    # (ParallelSum stmt, accumulate, number of ops of the group that precede it)
    sides: list = _dc.field(default_factory=list)


class Analysis:
    """Whole-function facts the grouping needs."""

    def __init__(self, fn):
        self.fn = fn
        self.rank = {p.name: p.type.rank for p in fn.params if p.is_view}
        self.params = {p.name for p in fn.params}
        self.extent_alias: dict = {}  # local view -> normalized declared extent (rank 1)
        for s in walk_statements(fn.body):
            if kind(s) == "DeclView":
                self.rank[s.name] = s.descriptor.rank
                # extent(local, 0) is the expression the View was declared with
                first_dynamic = kind(s.descriptor.extents[0]) != "StaticExtent"
                if first_dynamic and len(s.dyn_args) >= 1:
                    try:
                        self.extent_alias[s.name] = self.trip(s.dyn_args[0])
                    except (TypeError, ValueError):
                        pass
        self.host_scalars = self._host_scalars()
        self.live_scalars = self._live_scalars()
        # literal columns with which each rank-2 View is accessed anywhere in the function
        self.columns: dict = {}
        for s in walk_statements(fn.body):
            for e in N.statement_exprs(s):
                for n in walk_expr(e):
                    if kind(n) == "ViewAccess" and len(n.indices) == 2 and kind(n.indices[1]) == "IntLiteral":
                        self.columns.setdefault(n.view, set()).add(n.indices[1].value)
            if kind(s) in ("AssignView", "AtomicAdd") and len(s.target.indices) == 2 \
                    and kind(s.target.indices[1]) == "IntLiteral":
                self.columns.setdefault(s.target.view, set()).add(s.target.indices[1].value)

    # symbolic trip counts ------------------------------------------------------
    def trip(self, e):
        """Canonical (constant, terms) form with local-view extents replaced by the
        expression they were declared with."""
        const, terms = normalize_index(e)
        out_c, out_t = const, {}
        for atom, c in terms:
            if atom[0] == "extent" and atom[2] == 0 and atom[1] in self.extent_alias:
                ac, at = self.extent_alias[atom[1]]
                out_c += c * ac
                for a2, c2 in at:
                    out_t[a2] = out_t.get(a2, 0) + c * c2
            else:
                out_t[atom] = out_t.get(atom, 0) + c
        return out_c, tuple(sorted((a, c) for a, c in out_t.items() if c != 0))

    # host-evaluable scalars ------------------------------------------------------
    def _host_scalars(self) -> set:
        """Function-scope scalars every definition of which is literal/parameter
        arithmetic.  Decided per name (straight-line code, but one name may be
        assigned several times)."""
        device = set()
        defs: dict = {}
        for s in self.fn.body:
            k = kind(s)
            if k == "DeclScalar":
                defs.setdefault(s.name, []).append(s.init)
            elif k == "AssignScalar":
                defs.setdefault(s.name, []).append(s.rhs)
            elif k == "ParallelSum":
                device.add(s.dst)
            elif k == "If":
                for inner in walk_statements(s.body):
                    if kind(inner) in ("DeclScalar", "AssignScalar"):
                        device.add(inner.name)  # guarded function-scope scalars: keep on the device
        # A scalar PARAMETER starts out host-known (the caller's value) but stays so only while
        # every definition of it is host-evaluable too: `alpha = parallel_sum(x)` or
        # `alpha = alpha + x(0)` move it to the device (its slot is initialised with the caller's
        # value, compiled._CompiledRun.go), exactly like any other scalar.
        params = {p.name for p in self.fn.params if not p.is_view}
        changed = True
        cand = (set(defs) | params) - device
        while changed:
            changed = False
            for name in list(cand):
                for e in defs.get(name, ()):
                    ok = True
                    for n in walk_expr(e):
                        kk = kind(n)
                        if kk == "ViewAccess" or (kk == "ScalarVar" and n.name not in cand):
                            ok = False
                    if not ok:
                        cand.discard(name)
                        changed = True
                        break
        return cand

    def _live_scalars(self) -> set:
        """Scalars that are ever read (anywhere): a gather into a scalar outside this
        set is dead code."""
        live = set()
        for s in walk_statements(self.fn.body):
            for e in N.statement_exprs(s):
                for n in walk_expr(e):
                    if kind(n) == "ScalarVar":
                        live.add(n.name)
            if kind(s) == "AssignScalar" and s.op != "=":
                pass  # `s += e` reads s, but only to feed s itself
        return live


def _bulk_as_loop(stmt, an: Analysis, rank2: bool = False):
    """deep_copy / accumulate parallel_sum as an equivalent loop over the rows.  Rank-2 Views
    (`rank2`): one statement per column, for the columns 0..C-1 the function names literally;
    the host checks extent(dst, 1) == C before launching (LoopOp.need_cols)."""
    k = kind(stmt)
    op = "=" if k == "DeepCopy" else "+="
    what = "deepcopy" if k == "DeepCopy" else "suminto"
    rank = an.rank.get(stmt.dst)
    if isinstance(stmt.src, str) and an.rank.get(stmt.src) != rank:
        return None
    if rank == 1:
        tgt = N.ViewAccess(stmt.dst, (N.Counter(K),))
        rhs = N.ViewAccess(stmt.src, (N.Counter(K),)) if isinstance(stmt.src, str) else stmt.src
        return LoopOp(K, N.Extent(stmt.dst, 0), (N.AssignView(tgt, op, rhs),), stmt, what)
    if rank != 2 or not rank2:
        return None
    cols = set(an.columns.get(stmt.dst, ()))
    if isinstance(stmt.src, str):
        cols |= set(an.columns.get(stmt.src, ()))
    if not cols or cols != set(range(len(cols))) or len(cols) > 8:
        return None
    body = []
    for c in sorted(cols):
        tgt = N.ViewAccess(stmt.dst, (N.Counter(K), N.IntLiteral(c)))
        rhs = N.ViewAccess(stmt.src, (N.Counter(K), N.IntLiteral(c))) if isinstance(stmt.src, str) else stmt.src
        body.append(N.AssignView(tgt, op, rhs))
    need = {stmt.dst: len(cols)}
    if isinstance(stmt.src, str):
        need[stmt.src] = len(cols)
    return LoopOp(K, N.Extent(stmt.dst, 0), tuple(body), stmt, what, need_cols=need)


def build_ops(fn, an: Analysis, windows: bool = True, keep_dead: bool = False) -> list:
    """Statement list -> op list.  Ops are ('loop', LoopOp) | ('gather', stmt, acc) |
    ('scalars', [stmts]) | ('hostscalar', stmt) | ('declview', stmt) | ('return', expr) |
    ('raw', stmt) for statements the fusion pass does not model.  `keep_dead`: no dead-statement
    elimination (check_finite runs: a statement nothing reads may still produce the non-finite value
    the reference traps)."""
    ops: list = []
    bound = {p.name for p in fn.params if not p.is_view}
    run: list = []

    def flush():
        # `let s: f64 = 0.0;` of a device-resident scalar needs no kernel: the slot array is zero
        # filled at the start of every run (compiled._CompiledRun.go)
        import math

        live = [x for x in run if not (kind(x) == "DeclScalar" and kind(x.init) == "Literal"
                                       and x.init.value == 0.0 and math.copysign(1.0, x.init.value) > 0)]
        if live:
            ops.append(("scalars", live))
        run.clear()

    for s in fn.body:
        k = kind(s)
        if k in ("DeclScalar", "AssignScalar") and s.name in an.host_scalars:
            flush()
            bound.add(s.name)
            ops.append(("hostscalar", s))
            continue
        if k in codegen._ELEMENT:
            run.append(s)
            if k == "DeclScalar":
                bound.add(s.name)
            continue
        flush()
        if k == "DeclView":
            ops.append(("declview", s))
        elif k == "ParallelFor":
            sites = codegen.plan_atomics(s)
            modes = {st.mode for st in sites}
            # rank-2 Views: only rows at the running index with literal columns, and only in the
            # window generator (register columns); anything else stays an unfused statement
            # (a rank-2 View indexed any other way - m(idx(i), c) - is accessed in global memory
            # through the checked accessors, like an indirectly indexed rank-1 View)
            probe = LoopOp(s.counter, s.upper, s.body, s, "kernel")
            rank2 = not windows and any(an.rank.get(a.view, 1) != 1 for a in probe.accesses())
            if rank2 or "staged_atomic" in modes:
                ops.append(("raw", s))
                continue
            loop = LoopOp(s.counter, s.upper, tuple(s.body), s, "kernel", sites)
            ops.append(("loop", loop))
            targets: dict = {}
            for st in sites:
                if st.mode == "gather":
                    targets.setdefault(st.view, []).append(st)
            for view, group in targets.items():
                shift = max(0, max(st.offset for st in group))
                ops.append(("loop", LoopOp(K, s.upper, (), s, "apply", apply_of=(view, group, loop), shift=shift)))
        elif k in ("DeepCopy", "ParallelSumInto"):
            loop = _bulk_as_loop(s, an, windows)
            ops.append(("loop", loop) if loop is not None else ("raw", s))
        elif k == "ParallelSum":
            if s.dst not in an.live_scalars and not keep_dead:
                bound.add(s.dst)
                continue  # the sum is never read: dead statement
            ops.append(("gather", s, s.dst in bound))
            bound.add(s.dst)
        elif k == "Return":
            ops.append(("return", s.value))
        else:
            raise TypeError(f"cannot execute {k}")
    flush()
    return ops if keep_dead else _drop_dead_fills(ops, fn, an)


def _op_views(op) -> set:
    tag = op[0]
    out: set = set()

    def of_stmt(s):
        k = kind(s)
        if k in ("DeepCopy", "ParallelSumInto"):
            out.add(s.dst)
            if isinstance(s.src, str):
                out.add(s.src)
        elif k == "ParallelSum":
            out.add(s.src)
        for inner in walk_statements([s]):
            for e in N.statement_exprs(inner):
                for n in walk_expr(e):
                    if kind(n) in ("ViewAccess", "Extent"):
                        out.add(n.view)

    if tag == "loop":
        loop = op[1]
        if loop.what == "apply":
            out.add(loop.apply_of[0])
        else:
            for s in loop.body:
                of_stmt(s)
            of_stmt(loop.origin) if loop.what in ("deepcopy", "suminto") else None
    elif tag in ("raw", "gather", "hostscalar", "declview"):
        of_stmt(op[1])
    elif tag == "scalars":
        for s in op[1]:
            of_stmt(s)
    elif tag == "return":
        for n in walk_expr(op[1]):
            if kind(n) in ("ViewAccess", "Extent"):
                out.add(n.view)
    return out


def _cannot_raise(loop: "LoopOp", an) -> bool:
    """True when no access of the loop can leave its View and no bulk statement can meet
    mismatching extents - i.e. executing the statement is unobservable apart from the values it
    writes.  Proven for accesses at exactly the running index (literal column 0 of a rank-2 row
    excluded: column extents are run-time data) over a range that IS the View's first extent."""
    if loop.what == "apply":
        return False
    try:
        trip = an.trip(loop.upper)
    except (TypeError, ValueError):
        return False
    if loop.what in ("deepcopy", "suminto") and isinstance(loop.origin.src, str):
        try:
            if an.trip(N.Extent(loop.origin.src, 0)) != an.trip(N.Extent(loop.origin.dst, 0)):
                return False  # ShapeMismatch is decided at run time
        except (TypeError, ValueError):
            return False
    if loop.sites:
        return False
    for a in loop.accesses():
        if an.rank.get(a.view, 1) != 1 or len(a.indices) != 1:
            return False
        if kind(a.indices[0]) != "Counter" or a.indices[0].name != loop.counter:
            return False
        try:
            if an.trip(N.Extent(a.view, 0)) != trip:
                return False
        except (TypeError, ValueError):
            return False
    return True


def _drop_dead_fills(ops: list, fn, an=None) -> list:
    """Dead statements: a statement all of whose results nothing reads afterwards, and whose
    execution cannot raise, is unobservable - locals die at the return (runtime.py: DeclView
    storage is dropped).  The generated gradients carry such statements: the verbatim forward
    sweep computes Views only the (dead) forward reduction reads (`w` and `total` in
    mean_shift_grad), and the reversal of `deep_copy(t, 0.0)` zeroes the shadow of a View that is
    never used again.  Backward liveness over the op list: fills of dead locals, loop-shaped
    statements that write only dead locals through provably in-range accesses (`_cannot_raise`),
    gathers into scalars nobody reads, and pure scalar statements."""
    local = {s.name for s in walk_statements(fn.body) if kind(s) == "DeclView"}
    needed: set = set()
    needed_scalars: set = set()
    kept: list = []

    def scalar_reads(op) -> set:
        out: set = set()
        stmts = op[1] if op[0] == "scalars" else [op[1].origin] + list(op[1].body) if op[0] == "loop" else \
            [op[1]] if op[0] in ("raw", "gather", "hostscalar", "declview") else []
        exprs = [op[1]] if op[0] == "return" else []
        for s in walk_statements([x for x in stmts if x is not None and kind(x) != "ParallelFor"] +
                                 [x for x in stmts if x is not None and kind(x) == "ParallelFor"]):
            exprs += list(N.statement_exprs(s))
            if kind(s) == "AssignScalar" and s.op != "=":
                out.add(s.name)
        for e in exprs:
            for n in walk_expr(e):
                if kind(n) == "ScalarVar":
                    out.add(n.name)
        return out

    for op in reversed(ops):
        if op[0] == "scalars":
            # function-scope scalar statements nothing reads afterwards (the tail of a generated
            # gradient reverses scalars that are never used again): dead unless they touch a View
            stmts = list(walk_statements(op[1]))
            pure = all(kind(x) in ("DeclScalar", "AssignScalar", "If") for x in stmts) and not any(
                kind(n) == "ViewAccess" for x in stmts for e in N.statement_exprs(x) for n in walk_expr(e))
            written = {x.name for x in stmts if kind(x) in ("DeclScalar", "AssignScalar")}
            if pure and not (written & needed_scalars):
                continue
        if op[0] == "gather" and op[1].dst not in needed_scalars:
            continue  # a sum nobody reads (a gather cannot raise)
        stmt = op[1].origin if op[0] == "loop" and op[1].what == "deepcopy" else op[1] if op[0] == "raw" else None
        if stmt is not None and kind(stmt) == "DeepCopy" and not isinstance(stmt.src, str):
            if stmt.dst in local and stmt.dst not in needed:
                continue  # dead
            needed_scalars |= scalar_reads(op)
            needed.discard(stmt.dst)  # fully overwritten here: earlier contents are not needed
            kept.append(op)
            continue
        if op[0] == "loop" and an is not None and op[1].what in ("kernel", "suminto", "deepcopy"):
            written = {a.view for a in op[1].accesses() if a.write}
            if written and written <= local and not (written & needed) and _cannot_raise(op[1], an):
                continue  # writes only locals nothing reads afterwards
        needed_scalars |= scalar_reads(op)
        if op[0] == "gather" and not op[2]:
            needed_scalars.discard(op[1].dst)  # assigned here (not accumulated): earlier values are dead
            needed_scalars |= scalar_reads(op) - {op[1].dst}
        needed |= _op_views(op)
        kept.append(op)
    kept.reverse()
    return kept


def _reads_scalar(group: "Group", name: str) -> bool:
    for loop in group.ops:
        bodies = [loop.body]
        if loop.what == "apply":
            bodies = []
        for body in bodies:
            for s in walk_statements(body):
                for e in N.statement_exprs(s):
                    for n in walk_expr(e):
                        if kind(n) == "ScalarVar" and n.name == name:
                            return True
    return False


MAX_SIDES = 2


def form_groups(ops: list, an: Analysis, windows: bool = True, side_gathers: bool = False) -> list:
    """Greedy left-to-right grouping.  Returns a schedule of
    ('group', Group) | the non-loop ops unchanged.  `windows`: also merge across
    neighbour dependencies when a halo-recompute plan exists (window_plan)."""
    schedule: list = []
    cur = None  # (Group, trip, access summary)

    def close():
        nonlocal cur
        if cur is not None:
            g = cur[0]
            if windows and not g.windowed:
                # the window generator is also the one that keeps rank-2 rows in register columns and
                # serves neighbour reads of read-only Views from a window instead of repeated loads
                wp = window_plan(g.ops, an)
                if wp is not None and wp.needed:
                    g.windowed = True
            schedule.append(("group", g))
            cur = None

    def summary(loop: LoopOp):
        """view -> (pointwise_only, written, atomic_direct)"""
        out: dict = {}
        accs = loop.accesses()
        if loop.what == "apply":
            view, group, producer = loop.apply_of
            accs = [Access(view, (N.Counter(K),), True), Access(view, (N.Counter(K),), False)]
            for st in group:
                accs.append(Access(f"__stage{st.index}@{id(producer)}", (N.IntLiteral(0),), False))
        if loop.what == "kernel":
            for st in loop.sites:
                if st.mode == "gather":
                    accs.append(Access(f"__stage{st.index}@{id(loop)}", (N.Counter(loop.counter),), True))
        staged_views = {st.view for st in loop.sites if st.mode == "gather"}
        for a in accs:
            if a.atomic and a.view in staged_views:
                continue  # staged: the write goes to the staging column, not to the view
            pw = _is_pointwise(a, loop.counter)
            e = out.setdefault(a.view, [True, False, False])
            e[0] = e[0] and pw
            e[1] = e[1] or a.write
            e[2] = e[2] or (a.atomic)
        return out

    for op in ops:
        if op[0] != "loop":
            if op[0] == "gather" and cur is not None:
                g, trip, acc = cur
                stmt = op[1]
                src = stmt.src
                try:
                    src_trip = an.trip(N.Extent(src, 0))
                except (TypeError, ValueError):
                    src_trip = None
                info = acc.get(src)
                fusable = (src_trip == trip and all(o.shift == 0 for o in g.ops)
                           and (info is None or (info[0] and not info[2])))
                if fusable and an.rank.get(src) == 2:
                    # flat reduction of a rank-2 View: every column must be in registers, i.e. the group
                    # touches exactly the columns 0..C-1 (the host checks extent(src, 1) == C)
                    fusable = windows and info is not None and 1 <= len(group_columns(g.ops, src)) <= MAX_GATHER_COLS \
                        and group_columns(g.ops, src) == set(range(len(group_columns(g.ops, src))))
                elif an.rank.get(src) != 1:
                    fusable = False
                if fusable and side_gathers and an.rank.get(src) == 1 and stmt.dst not in an.live_scalars \
                        and len(g.sides) < MAX_SIDES:
                    g.sides.append((stmt, op[2], len(g.ops)))  # the group stays open
                    continue
                if fusable:
                    g.gather = (stmt, op[2])
                    close()
                    continue
            if op[0] == "declview":
                # creates a new (lazy, zero) View: nothing in the open group can refer to it, so
                # it is scheduled ahead of the group, which stays open
                schedule.append(op)
                continue
            if op[0] == "hostscalar" and cur is not None and not _reads_scalar(cur[0], op[1].name):
                schedule.append(op)  # host bookkeeping the open group does not depend on
                continue
            close()
            schedule.append(op)
            continue
        loop = op[1]
        try:
            trip = an.trip(loop.upper)
        except (TypeError, ValueError):
            close()
            cur = (Group([loop]), None, {})
            close()
            continue
        acc = summary(loop)
        if cur is not None:
            g, gtrip, gacc = cur
            if gtrip != trip and loop.what in ("deepcopy", "suminto") and isinstance(loop.origin.src, str):
                # `dst op= src` over whole Views raises unless their extents are equal (runtime.py:632-635,
                # 658-660; the host checks it before launching), so the loop may as well be counted
                # over the source's extent when that is the open group's range
                try:
                    alt = an.trip(N.Extent(loop.origin.src, 0))
                except (TypeError, ValueError):
                    alt = None
                if alt == gtrip:
                    loop.upper, trip = N.Extent(loop.origin.src, 0), alt
            ok = gtrip == trip
            # one staging buffer per kernel: a group holds at most one producer of staged
            # contributions, and never a producer together with an apply loop
            producer = loop.what == "kernel" and any(st.mode == "gather" for st in loop.sites)
            has_producer = any(o.what == "kernel" and any(st.mode == "gather" for st in o.sites) for o in g.ops)
            has_apply = any(o.what == "apply" for o in g.ops)
            classic = ok and not g.windowed
            if (producer and (has_producer or has_apply)) or (loop.what == "apply" and (has_producer or has_apply)):
                classic = False
            if classic and any(not acc.get(sstmt.src, (True,))[0] for sstmt, _, _ in g.sides):
                # a side reduction (check_finite plans) reads its source from the registers of a pointwise
                # View; this loop reads that View at i + c: no tile kernel (a window kernel may still do)
                classic = False
            if classic:
                for v, (pw, wr, at) in acc.items():
                    if v in gacc:
                        gpw, gwr, gat = gacc[v]
                        if at or gat:
                            classic = False
                        elif (wr or gwr) and not (pw and gpw):
                            classic = False
                    if not classic:
                        break
            merged = classic
            if ok and not classic and windows:
                # halo recompute: the contributions of a producer reach their apply loop through
                # warp-private windows, so the pair may share a kernel; still one producer per group,
                # and an apply loop only next to its own producer
                allowed = not (producer and (has_producer or has_apply))
                if loop.what == "apply" and (has_producer or has_apply):
                    allowed = any(o is loop.apply_of[2] for o in g.ops)
                if allowed and window_plan(g.ops + [loop], an) is not None:
                    merged = True
                    g.windowed = True
            if merged:
                g.ops.append(loop)
                for v, (pw, wr, at) in acc.items():
                    e = gacc.setdefault(v, [True, False, False])
                    e[0], e[1], e[2] = e[0] and pw, e[1] or wr, e[2] or at
                continue
            close()
        cur = (Group([loop]), trip, {v: list(t) for v, t in acc.items()})
    close()
    return schedule
