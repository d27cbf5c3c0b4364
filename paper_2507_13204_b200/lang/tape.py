"""Store-instead-of-reject for the reverse sweep (PAPER.md:838-839
lists it as future work; BASELINE.json's north star: "recompute-or-store of overwritten values").

The reference's transform never tapes: when the reversal of a statement would re-read a
value that is overwritten later - or a kernel-local scalar, which dies with its kernel - it
refuses the whole function (``NotFeasible``, adjoint.py:165-168 / analysis.py:400-488).
``differentiate(..., tape=True)`` accepts such functions by rewriting the *primal* first:

    right before the statement N whose reversal needs the value, the value is copied into a
    fresh local View (a snapshot), and N reads the snapshot instead

        x(i) = x(i) * x(i);          ->     _tape_x(i) = x(i);
                                            x(i) = _tape_x(i) * _tape_x(i);

        let t: f64 = a(i) + 1.0;     ->     let t: f64 = a(i) + 1.0;
        y(i) = t * t;                       _tape_t(i) = t;
                                            y(i) = _tape_t(i) * _tape_t(i);

The snapshot is never written again, so the ordinary transform applies unchanged: the copy
is one more assignment whose reversal routes the adjoint back (``_d_x(i) += _d__tape_x(i)``),
race flags and atomics follow from the same analyses, and - unlike a save/restore tape - the
caller still finds the forward results in the parameter Views after ``<fn>_grad``.  The
rewrite preserves the primal bit for bit (a copy does not round).

On the GPU a snapshot is an ordinary pointwise local: when the statements that write and
read it end up in the same fused kernel it lives in a register ("recompute" costs nothing);
otherwise it is the stored tape.

Supported: Views read at index-only positions (any ``v(i + c)``, ``v(i, 2)``) inside a
kernel, kernel-local scalars, function-scope scalars and View elements.  Anything else
(a needed value read through an indirect index that is itself overwritten, ...) still raises
``NotFeasible``.
"""

from __future__ import annotations

import dataclasses as _dc

from .dataflow import activity, taping_feasibility
from .nodes import (
    AssignView,
    DeclScalar,
    DeclView,
    Extent,
    FunctionDef,
    If,
    ParallelFor,
    ScalarVar,
    ViewAccess,
    ViewDescriptor,
    desugar_function,
    kind,
    walk_expr,
    walk_statements,
)

MAX_ROUNDS = 16


def _map_expr(e, f):
    """Bottom-up rebuild of an expression tree; ``f(node)`` may return a replacement."""
    if _dc.is_dataclass(e) and not isinstance(e, type):
        changes = {}
        for fld in _dc.fields(e):
            if fld.name == "span":
                continue
            v = getattr(e, fld.name)
            if _dc.is_dataclass(v) and not isinstance(v, type):
                nv = _map_expr(v, f)
                if nv is not v:
                    changes[fld.name] = nv
            elif isinstance(v, tuple) and v and all(_dc.is_dataclass(x) for x in v):
                nv = tuple(_map_expr(x, f) for x in v)
                if any(a is not b for a, b in zip(nv, v)):
                    changes[fld.name] = nv
        if changes:
            e = _dc.replace(e, **changes)
    r = f(e)
    return e if r is None else r


def _index_only(indices) -> bool:
    return not any(kind(n) == "ViewAccess" for i in indices for n in walk_expr(i))


class _Unsupported(Exception):
    pass


def _rewrite(fn, low, verdict, claim):
    """One round: snapshot what the reported statements need."""
    wanted: dict = {}  # id(needing statement) -> set of names
    for v in verdict.violations:
        if v.stmt is None:
            raise _Unsupported
        wanted.setdefault(id(v.stmt), set()).add(v.name)
    rank = {p.name: p.type.rank for p in fn.params if p.is_view}
    declared: dict = {}  # local View -> its declaration (a snapshot is declared with the same extents)
    for s in walk_statements(low.body):
        if kind(s) == "DeclView":
            rank[s.name] = s.descriptor.rank
            declared[s.name] = s

    def like(view, name):
        """`let name = view(...)` with the extents of `view`: a local's own extent expressions (the
        shadow of the snapshot is declared at the top of <fn>_grad, before the local exists), a
        parameter's extent(view, d)."""
        d = declared.get(view)
        if d is not None:
            return DeclView(_dc.replace(d.descriptor, name=name), d.dyn_args, label=name)
        r = rank[view]
        return DeclView(ViewDescriptor(name, rank=r), tuple(Extent(view, k) for k in range(r)), label=name)

    scalars_fn_scope = {p.name for p in fn.params if not p.is_view}
    decls_before_loop: dict = {}  # id(loop) -> [DeclView]

    def snapshot_in_kernel(stmt, names, loop):
        """(statements to put before stmt, rewritten stmt)"""
        pre: list = []
        tapes: dict = {}  # (name, index text) -> ViewAccess of the snapshot

        def tape_for_view(acc):
            if not _index_only(acc.indices):
                raise _Unsupported
            key = (acc.view, repr(acc.indices))
            if key not in tapes:
                name = claim("_tape_" + acc.view)
                decls_before_loop.setdefault(id(loop), []).append(like(acc.view, name))
                snap = ViewAccess(name, acc.indices)
                pre.append(AssignView(snap, "=", ViewAccess(acc.view, acc.indices), span=stmt.span))
                tapes[key] = snap
            return tapes[key]

        def tape_for_local(name):
            key = (name, "")
            if key not in tapes:
                tname = claim("_tape_" + name)
                decls_before_loop.setdefault(id(loop), []).append(
                    DeclView(ViewDescriptor(tname, rank=1), (loop.upper,), label=tname))
                from .nodes import Counter

                snap = ViewAccess(tname, (Counter(loop.counter),))
                pre.append(AssignView(snap, "=", ScalarVar(name), span=stmt.span))
                tapes[key] = snap
            return tapes[key]

        def redirect(n):
            k = kind(n)
            if k == "ViewAccess" and n.view in names:
                return tape_for_view(n)
            if k == "ScalarVar" and n.name in names:
                if n.name in scalars_fn_scope:
                    raise _Unsupported  # function-scope scalar needed inside a kernel: snapshot it outside
                return tape_for_local(n.name)
            return None

        k = kind(stmt)
        if k == "AssignView":
            new_target = ViewAccess(stmt.target.view, tuple(_map_expr(i, redirect) for i in stmt.target.indices))
            new = _dc.replace(stmt, target=new_target, rhs=_map_expr(stmt.rhs, redirect))
        elif k == "AssignScalar":
            new = _dc.replace(stmt, rhs=_map_expr(stmt.rhs, redirect))
        elif k == "DeclScalar":
            new = _dc.replace(stmt, init=_map_expr(stmt.init, redirect))
        else:
            raise _Unsupported
        if not pre:
            raise _Unsupported  # nothing could be redirected: the analysis asks for something else
        return pre, new

    def snapshot_at_function_scope(stmt, names):
        pre: list = []
        tapes: dict = {}

        def redirect(n):
            k = kind(n)
            hit = (k == "ViewAccess" and n.view in names and _index_only(n.indices)) or \
                  (k == "ScalarVar" and n.name in names)
            if not hit:
                if k == "ViewAccess" and n.view in names:
                    raise _Unsupported
                return None
            key = repr(n)
            if key not in tapes:
                tname = claim("_tape_" + (n.view if k == "ViewAccess" else n.name))
                pre.append(DeclScalar(tname, n, span=stmt.span))
                tapes[key] = ScalarVar(tname)
            return tapes[key]

        k = kind(stmt)
        if k == "AssignScalar":
            new = _dc.replace(stmt, rhs=_map_expr(stmt.rhs, redirect))
        elif k == "DeclScalar":
            new = _dc.replace(stmt, init=_map_expr(stmt.init, redirect))
        elif k == "AssignView":
            new = _dc.replace(stmt, rhs=_map_expr(stmt.rhs, redirect))
        else:
            raise _Unsupported
        if not pre:
            raise _Unsupported
        return pre, new

    def walk(body, loop):
        out: list = []
        for s in body:
            k = kind(s)
            if k == "If":
                out.append(If(s.cond, tuple(walk(s.body, loop)), span=s.span))
            elif k == "ParallelFor":
                inner = tuple(walk(s.body, s))
                out.extend(decls_before_loop.pop(id(s), []))
                out.append(ParallelFor(s.counter, s.upper, inner, span=s.span))
            elif id(s) in wanted:
                names = wanted[id(s)]
                pre, new = (snapshot_in_kernel(s, names, loop) if loop is not None
                            else snapshot_at_function_scope(s, names))
                out.extend(pre)
                out.append(new)
            else:
                out.append(s)
        return out

    return FunctionDef(fn.name, fn.params, tuple(walk(low.body, None)), fn.returns, span=fn.span)


def make_feasible(fn, wrt, claim):
    """``fn`` rewritten (desugared, snapshots inserted) so that the reverse-mode transform's
    taping check passes; raises the caller's NotFeasible material (the last verdict) when a
    needed value cannot be snapshotted.  Returns (function, number of snapshots)."""
    count = 0
    verdict = None
    for _ in range(MAX_ROUNDS):
        low = desugar_function(fn)
        act = activity(low, wrt)
        verdict = taping_feasibility(low, act)
        if verdict.ok:
            return fn, count, None
        try:
            before = sum(1 for s in walk_statements(low.body) if kind(s) == "DeclView")
            fn = _rewrite(fn, low, verdict, claim)
            count += sum(1 for s in walk_statements(fn.body) if kind(s) == "DeclView") - before
        except _Unsupported:
            return fn, count, verdict
    return fn, count, verdict
