"""Sharded execution of ANY function of the language over several GPUs.

The headline objective has its own sharded kernels (sharded.py: six halo values, bit-identical
reduction, everything resident on the device).  This module is the general mechanism: one process
per GPU owns the rows [lo, hi) of every View (rank-2: whole rows) and runs the SAME generated
kernels as a single device would, on programs derived from the tree:

* the function is cut into *segments* at its ``s = parallel_sum(v)`` statements.  A segment
  is an ordinary function of the same language (built here, executed by ``execute`` under any
  policy - normally one fused kernel); it ends with the gather and returns the rank's partial
  sum, which is all-reduced (one double) and handed to the following segments as an ``f64``
  parameter;
* function-scope scalar statements are literal / parameter / gathered-scalar arithmetic and
  are evaluated on the host, identically on every rank;
* index-dependent code is *localised*: in guards and ``float(i)`` the counter becomes
  ``i + lo`` and ``extent(v, 0)`` the global row count, while memory accesses and trip counts
  stay local;
* **neighbour accesses** (stencil reads ``v(i + c)``, writes / atomic adds to ``v(i + c)``) are
  served by *ghost rows*, the rank-level twin of the window kernels' halo recompute: every rank
  extends its Views by ``ghost`` rows of each neighbour (one all-gather of 2 x ghost rows per
  View at the start), runs the whole function on the extended rows - re-running its neighbours'
  edge iterations - and keeps its own rows.  ``ghost`` is the sum over the kernels of (farthest
  neighbour read + farthest neighbour write); statements that would reach outside the rows held
  are fenced off (their results lie in the discarded band); gathers sum a copy masked to the own
  rows.  No adjoint crosses a rank and the order of every accumulation is the single-device one;
* Views reached through **another row** (``x(idx(i))``, ``q(idx(i), 2)``) are *replicated*: every
  rank holds all of them.  They may be read freely; written only by ``atomic_add`` (the generated
  adjoint of an indirect read): every rank accumulates its own contributions (rank 0 on top of the
  caller's values, the others on zeros) and the copies are all-reduced once at the end - the one
  bandwidth-carrying collective (N doubles), as SURVEY.md section 8e prescribes.

Views come out bit-identical to a single-device run wherever they do not depend on a gathered
scalar or on the order of hardware atomics; a gathered scalar is the sum of the ranks' partial
trees, i.e. exact up to reassociation (the 1e-12 relative tolerance of BASELINE.json).  All 11
corpus programs and their gradients run this way.  Extended Views are assembled in HBM (own rows
device to device; only the 2 x ghost edge rows and the gathered scalars touch the host); under NCCL
replicated shadows are all-reduced in place in HBM.  Refused (``NotShardable``): non-unit strides, rank-2 Views at a
neighbouring row, kernel-local scalars initialised from a neighbouring row.
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


def classify(fn):
    """Classification(replicated Views, scatter targets among them, ghost width); raises NotShardable.

    A View accessed at the running row is *sharded* (a rank holds its own rows).  A View reached
    through another row - `x(idx(i))`, `q(idx(i), 2)`, `v(0)` - is *replicated*: every rank holds
    all of it.  Replicated Views may be read freely; they may be written only by `atomic_add`
    (the generated adjoint of an indirect read), and then every rank accumulates its own
    contributions and the copies are summed across ranks at the end (SURVEY.md section 8e:
    "replicate _d_x per GPU and allreduce it")."""
    row_use, other_use, scattered, plainly_written = set(), set(), set(), set()
    trip_views = set()
    ghost = 0
    reach: dict = {}  # id(kernel) -> (lowest, highest) neighbour offset it touches
    for s in fn.body:
        k = kind(s)
        if k == "ParallelFor":
            if not (kind(s.upper) == "Extent" and s.upper.dim == 0):
                raise NotShardable(f"kernel range is not extent(view, 0): {kind(s.upper)}")
            trip_views.add(s.upper.view)
            rd, wr = [0, 0], [0, 0]

            def note(acc, write, atomic, counter=s.counter, rd=rd, wr=wr):
                from .codegen import _unit_affine

                row = acc.indices[0]
                c = _unit_affine(row, counter)
                if kind(row) == "Counter" and row.name == counter:
                    row_use.add(acc.view)
                elif c is not None:
                    # a neighbouring row: served by ghost rows - the rank re-runs its neighbours' edge
                    # iterations, so a row it owns also receives what iteration k - c writes or adds to it
                    if len(acc.indices) != 1:
                        raise NotShardable(f"rank-2 view '{acc.view}' is accessed at a neighbouring row")
                    row_use.add(acc.view)
                    box = wr if write else rd
                    box[0], box[1] = min(box[0], c), max(box[1], c)
                elif any(kind(m) == "Counter" for m in walk_expr(row)) and not any(
                        kind(m) == "ViewAccess" for m in walk_expr(row)):
                    raise NotShardable(f"view '{acc.view}' is accessed at a non-unit stride")
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
                if kk == "DeclScalar":
                    from .codegen import _unit_affine as _ua

                    for n in walk_expr(inner.init):
                        if kind(n) == "ViewAccess" and _ua(n.indices[0], s.counter) not in (None, 0):
                            raise NotShardable("a kernel-local scalar is initialised from a neighbouring row")
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
            # every kernel shrinks the band of ghost rows that still hold correct values by what it
            # reads from its neighbours plus how far it scatters
            ghost += max(-rd[0], rd[1]) + max(-wr[0], wr[1])
            reach[id(s)] = (min(rd[0], wr[0]), max(rd[1], wr[1]))
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
    if ghost:
        for s in fn.body:
            if kind(s) == "ParallelSum" and _rank_of(fn, s.src) != 1:
                raise NotShardable("gather over a rank-2 view in a function with neighbour reads")
    return Classification(frozenset(replicated), frozenset(scattered), ghost, reach)


def _rank_of(fn, view) -> int:
    p = fn.param(view)
    if p is not None:
        return p.type.rank
    for s in walk_statements(fn.body):
        if kind(s) == "DeclView" and s.name == view:
            return s.descriptor.rank
    return 1


@_dc.dataclass(frozen=True)
class Classification:
    replicated: frozenset   # Views every rank holds whole (reached through another row)
    scattered: frozenset    # replicated Views written by atomic_add: summed across ranks at the end
    ghost: int              # rows of its neighbours a rank keeps (and recomputes) on either side
    reach: dict = _dc.field(default_factory=dict, compare=False)

    def __iter__(self):     # (replicated, scattered) for callers that only need the sets
        return iter((self.replicated, self.scattered))

    def __getitem__(self, i):
        return (self.replicated, self.scattered)[i]


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
    from .codegen import carries_across_iterations

    for s in walk_statements(fn.body):
        if kind(s) == "ParallelFor" and carries_across_iterations(s):
            # its result is defined by ONE sweep over the whole range in iteration order
            # (runtime._Run.do_kernel): rows cannot be cut across ranks
            raise NotShardable(f"line {getattr(s.span, 'line', 0)}: iterations of this kernel may meet at a plainly "
                               "written location; its result depends on their order")
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
        if k == "AtomicAdd":
            return _dc.replace(s, value=in_value(s.value))
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
    mask: object = None       # segment with ghost rows: (masked copy, gathered view) - see ShardedProgram._build


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


def plan_steps(fn, ranks: dict, ghost: int = 0) -> list:
    """Cut `fn` into host steps, local-view declarations and segments.  With ghost rows a gather
    must only count the rank's own rows: it sums a masked copy (`__own<k>`, zero on ghost rows; the
    bounds GLO_ / GHI_ are filled in per rank by ShardedProgram)."""
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
        mask = None
        if gather_stmt is not None:
            src = gather_stmt.src
            mask = None
            if ghost:
                own = f"__own{counter[0]}"
                ranks[own] = 1
                steps.append(Step("decl", stmt=N.DeclView(N.ViewDescriptor(own, rank=1), (N.Extent(src, 0),), label=own)))
                mask, src = (own, src), own
            body.append(N.ParallelSum("__part", src))
            body.append(N.Return(N.ScalarVar("__part")))
            returns = "f64"
            gather = (gather_stmt.dst, gather_stmt.dst in bound)
            bound.add(gather_stmt.dst)
        views, scalars = _names_in(body)
        if gather_stmt is not None and mask is not None:
            views |= {mask[0], mask[1]}
        scalars.discard("__part")
        params = tuple(N.Param(v, N.ViewDescriptor(v, rank=ranks[v])) for v in sorted(views)) + \
            tuple(N.Param(s_, "f64") for s_ in sorted(scalars))
        name = f"{fn.name}__seg{counter[0]}"
        counter[0] += 1
        steps.append(Step("segment", fn=N.FunctionDef(name, params, tuple(body), returns),
                          views=tuple(sorted(views)), scalars=tuple(sorted(scalars)), gather=gather,
                          mask=mask if gather_stmt is not None else None))

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


def _edge_rows(v, start: int, count: int) -> np.ndarray:
    """`count` rows of a View from row `start`, fetched from wherever the View lives."""
    if v._dev_ok and not v._host_ok:
        dev = v._dev.dev
        cols = v.size // max(v.extents[0], 1)
        out = np.empty((count,) + tuple(v.extents[1:]), dtype=np.float64)
        dev.download(out, v._dev.ptr + 8 * start * cols)
        return out
    return np.array(v.peek()[start:start + count])


def _put_rows(dev, dst_ptr: int, rows) -> None:
    """ghost rows into an extended View: device to device when they arrived as a CUDA tensor (the
    all-gather's output), from the host otherwise"""
    if hasattr(rows, "data_ptr"):
        dev.copy(dst_ptr, rows.data_ptr(), rows.numel())
    else:
        dev.upload(dst_ptr, np.ascontiguousarray(rows))


def _streams(dev):
    """(torch's current stream, the library context's stream as a torch stream) or (None, None)
    when they are one and the same timeline"""
    import ctypes as C

    import torch

    cur = torch.cuda.current_stream(dev.ordinal)
    sp = C.c_void_p()
    dev.lib.krn_ctx_stream(dev.h, C.byref(sp))
    if (sp.value or 0) == cur.cuda_stream:
        return None, None
    return cur, torch.cuda.ExternalStream(sp.value, device=torch.device("cuda", dev.ordinal))


def torch_after_library(dev) -> None:
    cur, ext = _streams(dev)
    if ext is not None:
        cur.wait_stream(ext)


def library_after_torch(dev) -> None:
    cur, ext = _streams(dev)
    if ext is not None:
        ext.wait_stream(cur)


def _extended_on_device(v, below, above):
    """A new View = [ghost rows from below | v | ghost rows from above], assembled in HBM: the own
    rows are copied device to device, and so are the ghost rows when the exchange delivered them
    as device tensors (TorchComm.exchange_rows_device)."""
    from .runtime import Device, ViewStorage, _DeviceBuffer

    dev = v._dev.dev if (v._dev is not None and v._dev_ok) else Device.get()
    cols = v.size // max(v.extents[0], 1)
    glo = 0 if below is None else below.shape[0]
    ghi = 0 if above is None else above.shape[0]
    rows = glo + v.extents[0] + ghi
    ext = ViewStorage._blank(v.name, (rows,) + tuple(v.extents[1:]))
    ext._dev = _DeviceBuffer(dev, 8 * rows * cols)
    if glo:
        _put_rows(dev, ext._dev.ptr, below)
    dev.copy(ext._dev.ptr + 8 * glo * cols, v.device_ptr(dev, write=False), v.size)
    if ghi:
        _put_rows(dev, ext._dev.ptr + 8 * (glo + v.extents[0]) * cols, above)
    ext._dev_ok, ext._host_ok, ext._zero = True, False, False
    return ext


def _copy_rows_on_device(dst, src, start: int, count: int) -> None:
    """dst[:] = src[start : start + count] without leaving the device."""
    dev = src._dev.dev
    cols = dst.size // max(dst.extents[0], 1)
    dev.copy(dst.device_ptr(dev, discard=True), src.device_ptr(dev, write=False) + 8 * start * cols, count * cols)


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

    def exchange_rows(self, first: np.ndarray, last: np.ndarray):
        """(last rows of the rank below, first rows of the rank above); None at the ends."""
        if self.world == 1:
            return None, None
        import torch

        device = "cuda" if self.dist.get_backend(self.group) == "nccl" else "cpu"
        mine = torch.from_numpy(np.concatenate([first.reshape(-1), last.reshape(-1)])).to(device)
        everyone = torch.empty(self.world * mine.numel(), dtype=mine.dtype, device=device)
        self.dist.all_gather_into_tensor(everyone, mine, group=self.group)
        everyone = everyone.cpu().numpy().reshape(self.world, 2, *first.shape)
        below = everyone[self.rank - 1, 1] if self.rank > 0 else None
        above = everyone[self.rank + 1, 0] if self.rank < self.world - 1 else None
        return below, above

    def exchange_rows_device(self, view, dev, ghost: int):
        """Device-resident twin of exchange_rows: the first / last `ghost` rows of `view` are
        sliced out of its HBM buffer (a torch tensor aliasing it), all-gathered on the device
        (NCCL over NVLink; gloo moves CUDA tensors too) and returned as CUDA tensors - nothing
        passes through the host.  Stream order: torch's stream waits for the library's before the
        slices are read; the caller lets the library wait for torch before it copies the rows."""
        if self.world == 1:
            return None, None
        import torch

        t = device_tensor(view, dev, write=False).reshape(view.extents[0], -1)
        torch_after_library(dev)
        rows = t.shape[0]
        mine = torch.cat([t[:ghost].reshape(-1), t[rows - ghost:].reshape(-1)])
        everyone = torch.empty(self.world * mine.numel(), dtype=mine.dtype, device=mine.device)
        self.dist.all_gather_into_tensor(everyone, mine, group=self.group)
        everyone = everyone.view(self.world, 2, -1)
        below = everyone[self.rank - 1, 1] if self.rank > 0 else None
        above = everyone[self.rank + 1, 0] if self.rank < self.world - 1 else None
        return below, above

    def allreduce_array(self, arr: np.ndarray) -> None:
        """In-place sum of a replicated View's copies, given as a host array (gloo)."""
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

    def allreduce_view(self, view) -> None:
        """In-place sum of a replicated View's copies.  NCCL: directly on the View's HBM buffer (a
        torch tensor aliasing it through __cuda_array_interface__) - N doubles over NVLink, nothing
        through the host; gloo: through the host array."""
        if self.world == 1:
            return
        if self.dist.get_backend(self.group) == "nccl":
            dev = view._dev.dev if (view._dev is not None and view._dev_ok) else None
            if dev is None:
                from .runtime import Device

                dev = Device.get()
            t = device_tensor(view, dev)
            torch_after_library(dev)  # the library's stream and torch's are different timelines:
            self.dist.all_reduce(t, group=self.group)
            library_after_torch(dev)  # ordered by events, no host synchronisation
        else:
            self.allreduce_array(view.buffer)


class _CudaArray:
    """Minimal __cuda_array_interface__ carrier for a device pointer."""

    def __init__(self, ptr: int, shape: tuple):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": "<f8", "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def device_tensor(view, dev, write: bool = True):
    """A torch CUDA tensor that ALIASES the View's device buffer (no copy); with `write` the View's
    host copy is marked stale because the tensor may be written through."""
    import torch

    ptr = view.device_ptr(dev, write=write)
    return torch.as_tensor(_CudaArray(ptr, view.extents), device=torch.device("cuda", dev.ordinal))


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
        self.cls = classify(fn)
        self.replicated, self.scattered, self.ghost = self.cls.replicated, self.cls.scattered, self.cls.ghost
        self.steps = plan_steps(fn, self.ranks, self.ghost)
        self._built: dict = {}  # (ghost rows below, own rows, ghost rows above) -> {segment name: Program}

    def _build(self, glo: int, own: int, ghi: int) -> dict:
        """The segment programs as this rank runs them: guards / float(i) / extents localised to the
        first row it holds (lo - glo); with ghost rows, kernels skip the edge iterations whose
        neighbours lie outside the rows held (their results are in the discarded band anyway) and
        gathers sum a copy masked to the rank's own rows."""
        key = (glo, own, ghi)
        hit = self._built.get(key)
        if hit is not None:
            return hit
        from .codegen import _unit_affine

        def reach(stmt, counter):
            lo_c = hi_c = 0
            for e in N.statement_exprs(stmt):
                for n in walk_expr(e):
                    if kind(n) == "ViewAccess" and n.view not in self.replicated:
                        c = _unit_affine(n.indices[0], counter)
                        if c is not None:
                            lo_c, hi_c = min(lo_c, c), max(hi_c, c)
            return lo_c, hi_c

        def fence(stmts, kernel):
            """every statement that touches a neighbouring row runs only where that row is held"""
            out_ = []
            i = N.Counter(kernel.counter)
            for x in stmts:
                if kind(x) == "If":
                    out_.append(N.If(x.cond, tuple(fence(x.body, kernel)), span=x.span))
                    continue
                cmin, cmax = reach(x, kernel.counter)
                if ghi and cmax > 0:
                    x = N.If(N.Compare("<", i, N.IdxBinary("-", kernel.upper, N.IntLiteral(cmax))), (x,))
                if glo and cmin < 0:
                    x = N.If(N.Compare(">=", i, N.IntLiteral(-cmin)), (x,))
                out_.append(x)
            return out_

        out = {}
        for st in self.steps:
            if st.what != "segment":
                continue
            body = []
            for s in st.fn.body:
                s = localize(s, self.lo - glo, self.n_global, self.replicated)
                if kind(s) == "ParallelFor" and self.ghost:
                    s = N.ParallelFor(s.counter, s.upper, tuple(fence(s.body, s)), span=s.span)
                if kind(s) == "ParallelSum" and st.mask is not None:
                    own_view, src = st.mask
                    i = N.Counter("__i")
                    copy = N.AssignView(N.ViewAccess(own_view, (i,)), "=", N.ViewAccess(src, (i,)))
                    body.append(N.ParallelFor("__i", N.Extent(src, 0), (
                        N.If(N.Compare(">=", i, N.IntLiteral(glo)), (
                            N.If(N.Compare("<", i, N.IntLiteral(glo + own)), (copy,)),)),)))
                body.append(s)
            fn = N.FunctionDef(st.fn.name, st.fn.params, tuple(body), st.fn.returns)
            out[fn.name] = N.Program((fn,))
        self._built[key] = out
        return out

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

        # ghost rows: every sharded parameter is extended by the neighbours' edge rows (one all-gather of
        # 2 x ghost rows per View); the function then runs on the extended rows and the own rows are
        # written back at the end
        sharded = [p.name for p in self.fn.params if p.is_view and p.name not in self.replicated]
        own = views[sharded[0]].extents[0] if sharded else 0
        glo = ghi = 0
        originals: dict = {}
        if self.ghost and sharded:
            G = self.ghost
            if own < G:
                raise NotShardable(f"a rank needs at least {G} rows of its own, got {own}")
            on_device = _execute_override is None
            resident = on_device and hasattr(self.comm, "exchange_rows_device")
            if resident:
                from .runtime import Device

                dev = Device.get(cfg.device)
            keep = []  # gathered tensors stay alive until the library's copies of their rows are ordered
            for name in sharded:
                v = views[name]
                if resident:
                    # edge rows sliced, gathered and copied inside HBM
                    below, above = self.comm.exchange_rows_device(v, dev, G)
                    keep.append((below, above))
                    library_after_torch(dev)
                else:
                    first, last = (_edge_rows(v, 0, G), _edge_rows(v, own - G, G)) if on_device else \
                        (v.buffer[:G].copy(), v.buffer[own - G:].copy())
                    below, above = self.comm.exchange_rows(first, last)
                glo, ghi = (G if below is not None else 0), (G if above is not None else 0)
                originals[name] = v
                views[name] = _extended_on_device(v, below, above) if on_device else ViewStorage.from_values(
                    name, np.concatenate(([below] if below is not None else []) + [v.buffer] +
                                         ([above] if above is not None else [])))
            if resident and keep:
                torch_after_library(dev)  # torch may recycle the gathered buffers only after the copies
                del keep
        programs = self._build(glo, own, ghi)

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
                part = execute(programs[st.fn.name], st.fn.name, call, cfg).value
                if st.gather is not None:
                    dst, accumulate = st.gather
                    total = np.float64(self.comm.allreduce_sum(float(part)))
                    # reference: scalars[dst] = scalars.get(dst, 0.0) + total (runtime.py:649-651)
                    H[dst] = (H[dst] if accumulate else np.float64(0.0)) + total
            elif st.what == "return":
                g = {k: (v if k in self.replicated else _Global(v, self.n_global)) for k, v in views.items()}
                value = float(host_eval(st.stmt.value, H, g))
        for name, original in originals.items():
            if _execute_override is None:
                _copy_rows_on_device(original, views[name], glo, own)
            else:
                original.buffer[...] = views[name].buffer[glo:glo + own]
        for name in sorted(self.scattered):
            if hasattr(self.comm, "allreduce_view") and _execute_override is None:
                self.comm.allreduce_view(views[name])
            else:
                self.comm.allreduce_array(views[name].buffer)
        return value
