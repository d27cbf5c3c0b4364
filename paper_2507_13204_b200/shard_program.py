"""Sharded execution of ANY row-wise function over several GPUs (SURVEY.md section 8e:
"everything else in the corpus is elementwise -> partition only").

The headline objective has its own sharded kernels (sharded.py: halo rows, bit-identical
reduction).  This module covers the rest: functions whose kernels touch every View only at
the running row - all of the reference's corpus except the two stencils and the indirect
gather, and their generated gradients.  One process per GPU owns the rows [lo, hi) of every
View (rank-2: whole rows); nothing but scalars ever crosses a rank:

* the function is cut into *segments* at its ``s = parallel_sum(v)`` statements.  A segment
  is an ordinary function of the same language (built here, executed by ``execute`` under any
  policy - normally one fused kernel); it ends with the gather and returns the rank's partial
  sum, which is all-reduced (one double) and handed to the following segments as an ``f64``
  parameter;
* function-scope scalar statements are literal / parameter / gathered-scalar arithmetic and
  are evaluated on the host, identically on every rank;
* index-dependent code is *localised*: in guards and ``float(i)`` the counter becomes
  ``i + lo`` and ``extent(v, 0)`` the global row count, while memory accesses and trip counts
  stay local.

Views come out bit-identical to a single-device run wherever they do not depend on a gathered
scalar; a gathered scalar is the sum of the ranks' partial trees, i.e. exact up to
reassociation (the 1e-12 relative tolerance of BASELINE.json).

Views reached through another row (``x(idx(i))``, ``q(idx(i), 2)``) are *replicated*: every rank
holds all of them.  They may be read freely; written only by ``atomic_add`` (the generated adjoint
of an indirect read): every rank then accumulates its own contributions (rank 0 on top of the
caller's values, the others on zeros) and the copies are all-reduced once at the end - the one
bandwidth-carrying collective of this module (N doubles), as SURVEY.md section 8e prescribes.
Functions with neighbour reads are refused (``NotShardable``): their halos are future work (the
headline stencil has its own sharded kernels).
"""

from __future__ import annotations

import dataclasses as _dc

import numpy as np

from .lang import nodes as N
from .lang.nodes import kind, walk_expr, walk_statements
from .lang.tape import _map_expr


class NotShardable(ValueError):
    pass


_execute_override = None  # tests only: a stand-in for runtime.execute (see tests/test_shard_program_cpu.py)


# ---------------------------------------------------------------------------
# analysis


def classify(fn) -> tuple:
    """(replicated Views, replicated Views that are scatter targets); raises NotShardable.

    A View accessed at the running row is *sharded* (a rank holds its own rows).  A View reached
    through another row - `x(idx(i))`, `q(idx(i), 2)`, `v(0)` - is *replicated*: every rank holds
    all of it.  Replicated Views may be read freely; they may be written only by `atomic_add`
    (the generated adjoint of an indirect read), and then every rank accumulates its own
    contributions and the copies are summed across ranks at the end (SURVEY.md section 8e:
    "replicate _d_x per GPU and allreduce it")."""
    row_use, other_use, scattered, plainly_written = set(), set(), set(), set()
    trip_views = set()
    for s in fn.body:
        k = kind(s)
        if k == "ParallelFor":
            if not (kind(s.upper) == "Extent" and s.upper.dim == 0):
                raise NotShardable(f"kernel range is not extent(view, 0): {kind(s.upper)}")
            trip_views.add(s.upper.view)

            def note(acc, write, atomic, counter=s.counter):
                row = acc.indices[0]
                if kind(row) == "Counter" and row.name == counter:
                    row_use.add(acc.view)
                elif any(kind(m) == "Counter" for m in walk_expr(row)) and not any(
                        kind(m) == "ViewAccess" for m in walk_expr(row)):
                    raise NotShardable(f"view '{acc.view}' is read at a neighbouring row (needs halos)")
                else:
                    other_use.add(acc.view)
                    if write:
                        (scattered if atomic else plainly_written).add(acc.view)
                for other in acc.indices[1:]:
                    if any(kind(m) in ("Counter", "ViewAccess") for m in walk_expr(other)):
                        raise NotShardable(f"view '{acc.view}': column index depends on the row")
                for i in acc.indices:  # accesses inside index positions: idx(i)
                    for m in walk_expr(i):
                        if kind(m) == "ViewAccess":
                            note(m, False, False)

            for inner in walk_statements(s.body):
                kk = kind(inner)
                if kk in ("AssignView", "AtomicAdd"):
                    note(inner.target, True, kk == "AtomicAdd")
                    if kk == "AssignView" and inner.op != "=":
                        pass  # the read of the target is the same access
                for e in N.statement_exprs(inner):
                    if kk in ("AssignView", "AtomicAdd") and e is inner.target:
                        continue
                    for n in walk_expr(e):
                        if kind(n) == "ViewAccess" and not _inside_index(e, n):
                            note(n, False, False)
        elif k == "DeclView":
            if not s.dyn_args or not (kind(s.dyn_args[0]) == "Extent" and s.dyn_args[0].dim == 0):
                raise NotShardable(f"local view '{s.name}' is not declared with extent(view, 0) rows")
        elif k in ("DeclScalar", "AssignScalar"):
            rhs = s.init if k == "DeclScalar" else s.rhs
            if any(kind(n) in ("ViewAccess", "IndexVar") for n in walk_expr(rhs)):
                raise NotShardable("function-scope scalar reads a view element")
        elif k in ("If", "AtomicAdd", "AssignView"):
            raise NotShardable(f"function-scope {k} is not supported")
    both = row_use & other_use
    if both:
        raise NotShardable(f"views accessed both at the running row and elsewhere: {sorted(both)}")
    if plainly_written:
        raise NotShardable(f"replicated views written without atomic_add: {sorted(plainly_written)}")
    replicated = set(other_use)
    if trip_views & replicated:
        raise NotShardable("a kernel ranges over a replicated view")
    for s in fn.body:  # bulk statements and declarations must not involve replicated Views
        k = kind(s)
        names = set()
        if k in ("DeepCopy", "ParallelSumInto"):
            names = {s.dst} | ({s.src} if isinstance(s.src, str) else set())
        elif k == "ParallelSum":
            names = {s.src}
        elif k == "DeclView":
            names = {s.name} | {n.view for a in s.dyn_args for n in walk_expr(a) if kind(n) == "Extent"}
        if names & replicated:
            raise NotShardable(f"bulk statement / declaration on a replicated view: {sorted(names & replicated)}")
    return frozenset(replicated), frozenset(scattered)


def _inside_index(root, node) -> bool:
    """True when `node` occurs inside the index positions of an access of `root` (those are
    visited through their owner)."""
    for n in walk_expr(root):
        if kind(n) == "ViewAccess" and n is not node:
            for i in n.indices:
                if any(m is node for m in walk_expr(i)):
                    return True
    return False


def check_shardable(fn) -> None:
    classify(fn)


def localize(stmt, lo: int, n_global: int, replicated=frozenset()):
    """The statement as rank `lo`'s rows see it: guards and float(i) use the global row; the
    extent of a sharded View is the global row count (a replicated View is whole already)."""

    def in_condition(e):
        def f(n):
            if kind(n) == "Counter":
                return N.IdxBinary("+", n, N.IntLiteral(lo)) if lo else None
            if kind(n) == "Extent" and n.dim == 0 and n.view not in replicated:
                return N.IntLiteral(n_global)
            return None

        return _map_expr(e, f)

    def in_value(e):
        def f(n):
            if kind(n) == "IndexVar":
                return N.Binary("+", n, N.Literal(float(lo))) if lo else None
            if kind(n) == "Extent" and n.dim == 0 and n.view not in replicated:
                return N.Literal(float(n_global))
            return None

        # accesses keep their (local) indices: only whole value subtrees outside index positions change
        def g(n):
            if kind(n) == "ViewAccess":
                return n
            return f(n)

        return _map_value(e, g)

    def go(s):
        k = kind(s)
        if k == "If":
            return N.If(in_condition(s.cond), tuple(go(x) for x in s.body), span=s.span)
        if k == "AssignView":
            return _dc.replace(s, rhs=in_value(s.rhs))
        if k == "AssignScalar":
            return _dc.replace(s, rhs=in_value(s.rhs))
        if k == "DeclScalar":
            return _dc.replace(s, init=in_value(s.init))
        if k == "ParallelFor":
            return N.ParallelFor(s.counter, s.upper, tuple(go(x) for x in s.body), span=s.span)
        return s

    return go(stmt)


def _map_value(e, f):
    """Like tape._map_expr but does not descend into ViewAccess indices."""
    k = kind(e)
    if k == "ViewAccess":
        return e
    if k == "Binary":
        e2 = N.Binary(e.op, _map_value(e.lhs, f), _map_value(e.rhs, f), span=e.span)
    elif k == "Neg":
        e2 = N.Neg(_map_value(e.operand, f), span=e.span)
    else:
        e2 = e
    r = f(e2)
    return e2 if r is None else r


# ---------------------------------------------------------------------------
# segmentation


@_dc.dataclass
class Step:
    what: str                 # "host" (scalar statement) | "decl" (local view) | "segment" | "return"
    stmt: object = None
    fn: object = None         # segment: FunctionDef
    views: tuple = ()         # segment: view parameter names
    scalars: tuple = ()       # segment: f64 parameter names
    gather: object = None     # segment: (dst scalar, accumulate?) when it ends with a gather


def _names_in(stmts):
    views, scalars = set(), set()
    for s in stmts:  # top level: kernels bring their own local scalars
        k = kind(s)
        if k in ("DeepCopy", "ParallelSumInto"):
            views.add(s.dst)
            if isinstance(s.src, str):
                views.add(s.src)
        elif k == "ParallelSum":
            views.add(s.src)
        locals_ = {x.name for x in walk_statements([s]) if kind(x) == "DeclScalar"} if k == "ParallelFor" else set()
        for inner in walk_statements([s]):
            for e in N.statement_exprs(inner):
                for n in walk_expr(e):
                    if kind(n) in ("ViewAccess", "Extent"):
                        views.add(n.view)
                    elif kind(n) == "ScalarVar" and n.name not in locals_:
                        scalars.add(n.name)
    return views, scalars


def plan_steps(fn, ranks: dict) -> list:
    """Cut `fn` into host steps, local-view declarations and segments."""
    check_shardable(fn)
    steps: list = []
    pending: list = []
    bound: set = {p.name for p in fn.params if not p.is_view}
    counter = [0]

    def close(gather_stmt=None):
        if not pending and gather_stmt is None:
            return
        body = list(pending)
        pending.clear()
        gather = None
        returns = None
        if gather_stmt is not None:
            body.append(N.ParallelSum("__part", gather_stmt.src))
            body.append(N.Return(N.ScalarVar("__part")))
            returns = "f64"
            gather = (gather_stmt.dst, gather_stmt.dst in bound)
            bound.add(gather_stmt.dst)
        views, scalars = _names_in(body)
        scalars.discard("__part")
        params = tuple(N.Param(v, N.ViewDescriptor(v, rank=ranks[v])) for v in sorted(views)) + \
            tuple(N.Param(s_, "f64") for s_ in sorted(scalars))
        name = f"{fn.name}__seg{counter[0]}"
        counter[0] += 1
        steps.append(Step("segment", fn=N.FunctionDef(name, params, tuple(body), returns),
                          views=tuple(sorted(views)), scalars=tuple(sorted(scalars)), gather=gather))

    for s in fn.body:
        k = kind(s)
        if k in ("DeclScalar", "AssignScalar"):
            close()
            steps.append(Step("host", stmt=s))
            bound.add(s.name)
        elif k == "DeclView":
            close()
            steps.append(Step("decl", stmt=s))
        elif k == "ParallelSum":
            close(s)
        elif k == "Return":
            close()
            steps.append(Step("return", stmt=s))
        else:
            pending.append(s)
    close()
    return steps


# ---------------------------------------------------------------------------
# execution


class TorchComm:
    """all-reduce(SUM) of a few doubles over torch.distributed (NCCL: through a device tensor)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist, self.group = dist, group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1

    def allreduce_sum(self, value: float) -> float:
        if self.world == 1:
            return value
        import torch

        device = "cuda" if self.dist.get_backend(self.group) == "nccl" else "cpu"
        t = torch.tensor([value], dtype=torch.float64, device=device)
        self.dist.all_reduce(t, group=self.group)
        return float(t.item())

    def allreduce_array(self, arr: np.ndarray) -> None:
        """In-place sum of a replicated View's copies (host array; NCCL: staged through the device)."""
        if self.world == 1:
            return
        import torch

        if self.dist.get_backend(self.group) == "nccl":
            t = torch.from_numpy(arr).cuda()
            self.dist.all_reduce(t, group=self.group)
            arr[...] = t.cpu().numpy()
        else:
            t = torch.from_numpy(arr)
            self.dist.all_reduce(t, group=self.group)


class ShardedProgram:
    """One rank's executor of `fn_name` over rows [lo, lo + local rows) of a problem of
    `n_global` rows.  `run(inputs)` takes this rank's slices (ViewStorage or arrays; rank-2:
    whole rows) and the scalar parameters; Views are updated in place like ``execute`` does."""

    def __init__(self, program, fn_name: str, n_global: int, lo: int, comm=None):
        fn = program.function(fn_name)
        if fn is None:
            raise KeyError(f"no function named '{fn_name}'")
        self.fn, self.n_global, self.lo = fn, int(n_global), int(lo)
        self.comm = comm if comm is not None else TorchComm()
        self.ranks = {p.name: p.type.rank for p in fn.params if p.is_view}
        for s in walk_statements(fn.body):
            if kind(s) == "DeclView":
                self.ranks[s.name] = s.descriptor.rank
        self.replicated, self.scattered = classify(fn)
        self.steps = plan_steps(fn, self.ranks)
        # localised segment programs (one Program per segment: `execute` caches its plan per function)
        self.programs = {}
        for st in self.steps:
            if st.what == "segment":
                body = tuple(localize(s, self.lo, self.n_global, self.replicated) for s in st.fn.body)
                st.fn = N.FunctionDef(st.fn.name, st.fn.params, body, st.fn.returns)
                self.programs[st.fn.name] = N.Program((st.fn,))

    def run(self, inputs: dict, cfg=None):
        from .compiled import host_eval
        from .runtime import ExecutionConfig, ViewStorage, _index_value, execute

        if _execute_override is not None:  # CPU tests of the transform plug the oracle in here
            execute = _execute_override
        cfg = cfg or ExecutionConfig()
        views, H = {}, {}
        for p in self.fn.params:
            v = inputs[p.name]
            if p.is_view:
                if not isinstance(v, ViewStorage):
                    v = ViewStorage.from_values(p.name, v)
                    inputs[p.name] = v
                views[p.name] = v
            else:
                H[p.name] = np.float64(v)

        # scatter targets are replicated: rank 0 keeps the caller's values, the others start from zero,
        # every rank adds its own contributions, the copies are summed at the end
        for name in self.scattered:
            if self.lo > 0:
                views[name].buffer[...] = 0.0

        class _Global:  # host_eval asks Views for extents: rows are the GLOBAL count
            def __init__(self, v, n):
                self.extents = (n,) + tuple(v.extents[1:])


        value = None
        for st in self.steps:
            if st.what == "decl":
                s = st.stmt
                args = iter(s.dyn_args)
                dims = [e.size if kind(e) == "StaticExtent" else int(_index_value(next(args), views))
                        for e in s.descriptor.extents]
                views[s.name] = ViewStorage.zeros(s.name, dims)
            elif st.what == "host":
                s = st.stmt
                g = {k: (v if k in self.replicated else _Global(v, self.n_global)) for k, v in views.items()}
                rhs = host_eval(s.init if kind(s) == "DeclScalar" else s.rhs, H, g)
                if kind(s) == "DeclScalar" or s.op == "=":
                    H[s.name] = rhs
                else:
                    H[s.name] = H[s.name] + rhs if s.op == "+=" else H[s.name] - rhs
            elif st.what == "segment":
                call = {v: views[v] for v in st.views}
                call.update({s_: float(H[s_]) for s_ in st.scalars})
                part = execute(self.programs[st.fn.name], st.fn.name, call, cfg).value
                if st.gather is not None:
                    dst, accumulate = st.gather
                    total = np.float64(self.comm.allreduce_sum(float(part)))
                    # reference: scalars[dst] = scalars.get(dst, 0.0) + total (runtime.py:649-651)
                    H[dst] = (H[dst] if accumulate else np.float64(0.0)) + total
            elif st.what == "return":
                g = {k: (v if k in self.replicated else _Global(v, self.n_global)) for k, v in views.items()}
                value = float(host_eval(st.stmt.value, H, g))
        for name in sorted(self.scattered):
            self.comm.allreduce_array(views[name].buffer)
        return value
