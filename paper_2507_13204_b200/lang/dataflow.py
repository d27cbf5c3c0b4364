"""Static analyses that gate and shape the reverse sweep.

Behaviour follows the reference's ``krn.analysis``
(/root/reference/pkg/src/krn/analysis.py):

* ``activity``            (reference :98-190)  forward fixed point from ``wrt``
* ``normalize_index``     (reference :204-248) canonical affine index form
* ``race_analysis``       (reference :271-303) rules 1/2/3 -> atomic shadow sets
* ``taping_feasibility``  (reference :400-488) no in-kernel tape: a value the
  reverse sweep re-reads must not be overwritten later in the forward sweep

The GPU executor consumes ``normalize_index`` again (schedule.py) to decide
*how* a flagged accumulation is executed: affine offsets are turned into a
conflict-free gather in the reference's canonical order, indirect targets go
through hardware atomics.
"""

from __future__ import annotations

import dataclasses as _dc

from . import derivative
from .nodes import SourceSpan, desugar_function, free_counters, kind, walk_expr, walk_statements
from .syntax import index_text


class UnknownParameter(ValueError):
    pass


# ---------------------------------------------------------------------------
# activity


@_dc.dataclass(frozen=True)
class ActivityResult:
    fn: object
    wrt: frozenset
    active_views: frozenset
    active_scalars: frozenset
    _flags: dict = _dc.field(compare=False, repr=False, default_factory=dict)

    def is_active(self, name: str) -> bool:
        return name in self.active_views or name in self.active_scalars

    def stmt_active(self, stmt) -> bool:
        return self._flags.get(id(stmt), False)


def value_reads(e) -> set:
    """Names read in value position.  An access contributes its view name
    only: indices (including indirect ones) never carry activity."""
    out: set = set()
    todo = [e]
    while todo:
        n = todo.pop()
        k = kind(n)
        if k == "ScalarVar":
            out.add(n.name)
        elif k == "ViewAccess":
            out.add(n.view)
        elif k in ("Binary", "IdxBinary"):
            todo += [n.lhs, n.rhs]
        elif k == "Neg":
            todo.append(n.operand)
    return out


def _written_name(stmt):
    """(name written, expression or view name feeding it) for dataflow."""
    k = kind(stmt)
    if k == "DeclScalar":
        return stmt.name, stmt.init
    if k == "AssignScalar":
        return stmt.name, stmt.rhs
    if k == "AssignView":
        return stmt.target.view, stmt.rhs
    if k == "AtomicAdd":
        return stmt.target.view, stmt.value
    if k in ("DeepCopy", "ParallelSum", "ParallelSumInto"):
        return stmt.dst, stmt.src
    return None, None


def activity(fn, wrt) -> ActivityResult:
    wrt = frozenset(wrt)
    unknown = wrt - {p.name for p in fn.params}
    if unknown:
        raise UnknownParameter(f"not parameters of '{fn.name}': {', '.join(sorted(unknown))}")

    live = set(wrt)
    writers = [
        (dst, src) for dst, src in map(_written_name, walk_statements(fn.body)) if dst is not None
    ]

    def feeds(src) -> bool:
        if isinstance(src, str):
            return src in live
        return bool(value_reads(src) & live)

    grew = True
    while grew:
        grew = False
        for dst, src in writers:
            if dst not in live and feeds(src):
                live.add(dst)
                grew = True

    views, scalars = set(), set()
    for p in fn.params:
        if p.name in live:
            (views if p.is_view else scalars).add(p.name)
    for s in walk_statements(fn.body):
        k = kind(s)
        if k == "DeclView" and s.name in live:
            views.add(s.name)
        elif k == "DeclScalar" and s.name in live:
            scalars.add(s.name)
        elif k == "ParallelSum" and s.dst in live:
            scalars.add(s.dst)

    flags: dict = {}

    def mark(body) -> bool:
        hit = False
        for s in body:
            k = kind(s)
            if k in ("If", "ParallelFor"):
                on = mark(s.body)
            elif k == "Return":
                on = feeds(s.value)
            elif k == "DeclView":
                on = s.name in live
            else:
                dst, _ = _written_name(s)
                on = dst is not None and dst in live
            flags[id(s)] = on
            hit = hit or on
        return hit

    mark(fn.body)
    return ActivityResult(fn, wrt, frozenset(views), frozenset(scalars), flags)


# ---------------------------------------------------------------------------
# canonical affine indices


def _linear(e):
    """index expression -> (constant, {atom: coefficient})."""
    k = kind(e)
    if k == "IntLiteral":
        return e.value, {}
    if k == "Counter":
        return 0, {("counter", e.name): 1}
    if k == "Extent":
        return 0, {("extent", e.view, e.dim): 1}
    if k == "ViewAccess":
        return 0, {("view", e.view, tuple(normalize_index(i) for i in e.indices)): 1}
    if k == "IdxBinary":
        (lc, lt), (rc, rt) = _linear(e.lhs), _linear(e.rhs)
        if e.op in ("+", "-"):
            sg = 1 if e.op == "+" else -1
            terms = dict(lt)
            for a, c in rt.items():
                terms[a] = terms.get(a, 0) + sg * c
            return lc + sg * rc, terms
        if e.op == "*":
            if not lt:
                return lc * rc, {a: lc * c for a, c in rt.items()}
            if not rt:
                return lc * rc, {a: rc * c for a, c in lt.items()}
            raise ValueError("index multiplication needs an integer literal factor")
    raise TypeError(f"not an index expression: {k}")


def normalize_index(e):
    """Hashable canonical form ``(constant, ((atom, coeff), ...))`` so that
    ``j + 1`` and ``1 + j`` compare equal."""
    const, terms = _linear(e)
    return const, tuple(sorted((a, c) for a, c in terms.items() if c != 0))


# ---------------------------------------------------------------------------
# race flags


@_dc.dataclass(frozen=True)
class RaceFlag:
    kernel: int
    view: str
    rule: int  # 1 indirect, 2 differing counter indices, 3 counter-free index
    indices: tuple


@_dc.dataclass(frozen=True)
class RaceResult:
    flags: tuple

    def flagged(self, kernel: int) -> frozenset:
        return frozenset(f.view for f in self.flags if f.kernel == kernel)


def _index_subnodes(e):
    for n in walk_expr(e):
        yield n


def kernel_accesses(kernel) -> list:
    """Every view access of a kernel body (targets, operands and the accesses
    nested in indirect indices), as records the rules below filter."""
    ctr = kernel.counter
    found: list = []

    def note(acc):
        nested = [n for i in acc.indices for n in _index_subnodes(i) if kind(n) == "ViewAccess"]
        found.append(
            dict(
                view=acc.view,
                norm=tuple(normalize_index(i) for i in acc.indices),
                text="(" + ", ".join(index_text(i) for i in acc.indices) + ")",
                has_counter=any(ctr in free_counters(i) for i in acc.indices),
                indirect=bool(nested),
            )
        )
        # immediate children only: deeper ones are reached recursively
        for i in acc.indices:
            for n in _direct_accesses(i):
                note(n)

    def _direct_accesses(i):
        k = kind(i)
        if k == "ViewAccess":
            yield i
        elif k == "IdxBinary":
            yield from _direct_accesses(i.lhs)
            yield from _direct_accesses(i.rhs)

    def scan_value(e):
        k = kind(e)
        if k == "ViewAccess":
            note(e)
        elif k == "Binary":
            scan_value(e.lhs)
            scan_value(e.rhs)
        elif k == "Neg":
            scan_value(e.operand)

    def scan(body):
        for s in body:
            k = kind(s)
            if k == "AssignView":
                note(s.target)
                scan_value(s.rhs)
            elif k == "AtomicAdd":
                note(s.target)
                scan_value(s.value)
            elif k == "DeclScalar":
                scan_value(s.init)
            elif k == "AssignScalar":
                scan_value(s.rhs)
            elif k == "If":
                scan(s.body)

    scan(kernel.body)
    return found


def race_analysis(fn) -> RaceResult:
    fn = desugar_function(fn)
    out: list = []
    kernels = [s for s in walk_statements(fn.body) if kind(s) == "ParallelFor"]
    for kid, kernel in enumerate(kernels):
        per_view: dict = {}
        for a in kernel_accesses(kernel):
            per_view.setdefault(a["view"], []).append(a)
        for view in sorted(per_view):
            accs = per_view[view]
            indirect = {a["text"] for a in accs if a["indirect"]}
            if indirect:
                out.append(RaceFlag(kid, view, 1, tuple(sorted(indirect))))
            distinct = {a["norm"]: a["text"] for a in accs if a["has_counter"]}
            if len(distinct) >= 2:
                out.append(RaceFlag(kid, view, 2, tuple(sorted(set(distinct.values())))))
            fixed = {a["text"] for a in accs if not a["has_counter"]}
            if fixed:
                out.append(RaceFlag(kid, view, 3, tuple(sorted(fixed))))
    return RaceResult(tuple(out))


# ---------------------------------------------------------------------------
# taping feasibility


@_dc.dataclass(frozen=True)
class TapingViolation:
    span: SourceSpan
    name: str
    overwrite_span: SourceSpan
    # the statement whose reversal needs the value (not part of the reference's record; used by
    # lang/tape.py to snapshot the value instead of rejecting the function)
    stmt: object = _dc.field(default=None, compare=False, repr=False)


@_dc.dataclass(frozen=True)
class TapingVerdict:
    ok: bool
    violations: tuple


def _index_views(e, only_if_view_in=None) -> set:
    """Views read inside the index positions of the accesses in ``e``."""
    out: set = set()

    def from_access(acc):
        for i in acc.indices:
            for n in walk_expr(i):
                if kind(n) == "ViewAccess":
                    out.add(n.view)

    def go(n):
        k = kind(n)
        if k == "ViewAccess":
            if only_if_view_in is None or n.view in only_if_view_in:
                from_access(n)
        elif k == "Binary":
            go(n.lhs)
            go(n.rhs)
        elif k == "Neg":
            go(n.operand)

    go(e)
    return out


def taping_feasibility(fn, act: ActivityResult) -> TapingVerdict:
    fn = desugar_function(fn)
    active = set(act.active_views) | set(act.active_scalars)

    def occurrence_active(occ) -> bool:
        return (occ.view if kind(occ) == "ViewAccess" else occ.name) in active

    needs: list = []  # (position, names, span)
    writes: list = []  # (position, name, span)
    loop_locals: dict = {}
    pos = 0

    def need(rhs, target, span, lhs_name):
        if lhs_name not in active:
            return
        names = derivative.needed_primal_names(rhs, occurrence_active)
        if target is not None:
            names |= _index_views(target)
        names |= _index_views(rhs, only_if_view_in=active)
        if names:
            needs.append((pos, frozenset(names), span, current[0]))

    current = [None]

    def visit(body, in_kernel):
        nonlocal pos
        for s in body:
            pos += 1
            current[0] = s
            k = kind(s)
            if k == "AssignView":
                need(s.rhs, s.target, s.span, s.target.view)
                writes.append((pos, s.target.view, s.span))
            elif k == "AssignScalar":
                need(s.rhs, None, s.span, s.name)
                writes.append((pos, s.name, s.span))
            elif k == "DeclScalar":
                need(s.init, None, s.span, s.name)
                writes.append((pos, s.name, s.span))
                if in_kernel:
                    loop_locals[s.name] = s.span
            elif k == "AtomicAdd":
                writes.append((pos, s.target.view, s.span))
            elif k in ("DeepCopy", "ParallelSum", "ParallelSumInto"):
                writes.append((pos, s.dst, s.span))
            elif k == "If":
                visit(s.body, in_kernel)
            elif k == "ParallelFor":
                visit(s.body, True)

    visit(fn.body, False)

    bad: list = []
    for npos, names, nspan, nstmt in needs:
        for name in sorted(names):
            if name in loop_locals:  # dies with its kernel; cannot be replayed
                bad.append(TapingViolation(nspan, name, loop_locals[name], nstmt))
                continue
            clobber = next((w for w in writes if w[0] >= npos and w[1] == name), None)
            if clobber is not None:
                bad.append(TapingViolation(nspan, name, clobber[2], nstmt))
    return TapingVerdict(not bad, tuple(bad))
