"""Execution of a function through the fusion pass (policy "fused" for anything
that is not the hand-written headline, and policy "compiled" for everything).

Plan = schedule of fused groups (tile kernels, tilegen.py) interleaved with the
statements the pass leaves alone (library builtins, unfused generated kernels).
Before anything is launched the run is checked *dry* on the host - all extents are
host data - and if a fused group could not honour the reference's error semantics
(an access that would be out of bounds, mismatching extents of a bulk statement)
the whole call is handed to the statement path, which raises exactly where the
reference does.
"""

from __future__ import annotations

import ctypes as C
import os
import struct

import numpy as np

from . import _cabi, codegen, fusion, tilegen
from .lang import nodes as N
from .lang.nodes import kind, walk_expr, walk_statements


def _views_in_stmts(stmts) -> set:
    out = set()
    for s in walk_statements(stmts):
        k = kind(s)
        if k in ("DeepCopy", "ParallelSumInto"):
            out.add(s.dst)
            if isinstance(s.src, str):
                out.add(s.src)
        elif k == "ParallelSum":
            out.add(s.src)
        for e in N.statement_exprs(s):
            for n in walk_expr(e):
                if kind(n) in ("ViewAccess", "Extent"):
                    out.add(n.view)
    return out


def _views_of(item) -> set:
    tag = item[0]
    if tag == "group":
        g = item[1]
        out = set()
        for loop in g.ops:
            if loop.what == "apply":
                out.add(loop.apply_of[0])
            else:
                out |= _views_in_stmts(loop.body)
        if g.gather is not None:
            out.add(g.gather[0].src)
        return out
    if tag == "gather":
        return {item[1].src}
    if tag == "scalars":
        return _views_in_stmts(item[1])
    if tag == "raw":
        return _views_in_stmts([item[1]])
    if tag == "return":
        return {n.view for n in walk_expr(item[1]) if kind(n) in ("ViewAccess", "Extent")}
    return set()


def _host_evaluable(e, host_scalars) -> bool:
    for n in walk_expr(e):
        k = kind(n)
        if k == "ViewAccess" or k == "IndexVar" or (k == "ScalarVar" and n.name not in host_scalars):
            return False
    return True


class CompiledPlan:
    def __init__(self, fn, windows: bool = True, track: bool = False):
        """`track`: a check_finite plan - nothing dead is dropped, every fused kernel tests the values its
        statements leave behind and records them per (statement, View) (`checkpoints`, finite_replay);
        raises tilegen.Untrackable when a statement cannot be watched from inside its kernel."""
        self.fn = fn
        self.track = track
        an = self.an = fusion.Analysis(fn)
        self.schedule = fusion.form_groups(fusion.build_ops(fn, an, windows, keep_dead=track), an, windows,
                                           side_gathers=track)
        self.windowed = any(item[0] == "group" and item[1].windowed for item in self.schedule)
        b = self.builder = codegen.ModuleBuilder(fn, host_scalars=an.host_scalars)
        self.checkpoints: list = []
        if track:
            # checkpoint numbers in statement order (0 = the Views as they come in): the reference checks
            # every View after each kernel / bulk statement and the scalar after each gather
            # (runtime.py:624, 641, 651, 665)
            b.track = {}
            for item in self.schedule:
                if item[0] == "raw":
                    raise tilegen.Untrackable("a statement outside the fused kernels")
                if item[0] == "group":
                    for loop in item[1].ops:
                        if id(loop.origin) not in b.track:
                            b.track[id(loop.origin)] = len(b.track) + 1
        params = {p.name for p in fn.params if p.is_view}
        self.steps: list = []
        bound = set()
        fresh: set = set()  # local Views declared so far that no statement has touched: all +0.0
        for idx, item in enumerate(self.schedule):
            tag = item[0]
            if track:
                self._note_checkpoints(item)
            if tag == "declview":
                fresh.add(item[1].name)
            elif tag != "group":
                fresh -= _views_of(item)
            if tag == "group":
                later = set(params)
                for nxt in self.schedule[idx + 1:]:
                    later |= _views_of(nxt)
                item[1].fresh = frozenset(fresh)
                fresh -= _views_of(item)
                touched_now = _views_of(item)
                for stmt, _, _ in item[1].sides:
                    b.slot(stmt.dst)
                if item[1].windowed:
                    plan = tilegen.plan_window_group(b, item[1], an, later)
                    self.steps.append(("group", item[1], tilegen.window_kernel(b, item[1], f"g{idx}", plan, an)))
                else:
                    plan = tilegen.plan_group(b, item[1], an, later)
                    self.steps.append(("group", item[1], tilegen.tile_kernel(b, item[1], f"g{idx}", plan, an)))
                b.touched_before |= touched_now
            elif tag == "raw":
                s = item[1]
                if kind(s) == "ParallelFor":
                    self.steps.append(("kernel", s, b.kernel(s, f"k{idx}")))
                else:
                    self.steps.append(("deepcopy" if kind(s) == "DeepCopy" else "suminto", s))
            elif tag == "gather":
                b.slot(item[1].dst)
                self.steps.append(("gather", item[1], item[2]))
            elif tag == "scalars":
                self.steps.append(("scalars", b.scalar_block(item[1], f"s{idx}"), _views_of(item)))
            elif tag == "return":
                if _host_evaluable(item[1], an.host_scalars):
                    self.steps.append(("hostreturn", item[1]))
                elif kind(item[1]) == "ScalarVar":
                    self.steps.append(("slotreturn", b.slot(item[1].name)))  # read the slot, no kernel
                else:
                    self.steps.append(("return", b.return_block(item[1], f"r{idx}"), _views_of(item)))
            else:
                self.steps.append(item)  # declview, hostscalar
        self.source = b.source()
        self.nslots = max(len(b.slots), 1) + 1
        self.launch_count = sum(1 for s in self.steps if s[0] in ("group", "kernel", "scalars", "return", "gather"))


    def _note_checkpoints(self, item):
        b, tag = self.builder, item[0]
        if tag == "declview":
            self.checkpoints.append(("decl", item[1].name))
        elif tag == "gather":
            self.checkpoints.append(("scalar", item[1].dst))
        elif tag == "group":
            g = item[1]
            seen = []  # [checkpoint, Views] runs and side-gather scalars, in statement order
            for k, loop in enumerate(g.ops):
                for stmt, _, pos in g.sides:
                    if pos == k:
                        seen.append(("scalar", stmt.dst))
                cp = b.track[id(loop.origin)]
                written = [loop.apply_of[0]] if loop.what == "apply" else \
                    sorted({a.view for a in loop.accesses() if a.write and not a.atomic})
                if seen and seen[-1][0] == cp:
                    seen[-1][1].update(written)
                else:
                    seen.append((cp, set(written)))
            for stmt, _, pos in g.sides:
                if pos == len(g.ops):
                    seen.append(("scalar", stmt.dst))
            for first, second in seen:
                self.checkpoints.append(("scalar", second) if first == "scalar" else ("views", first, sorted(second)))
            if g.gather is not None:
                self.checkpoints.append(("scalar", g.gather[0].dst))


_plans: dict = {}


RETUNE_MIN_ELEMENTS = 1 << 20


def retuned_module(dev, plan: CompiledPlan):
    """The plan's module with the occupancy bound of its fused kernels set one block per SM above
    what the compiler chose on its own.  These kernels are latency bound at 2-5 resident blocks
    (8 warps each) per SM, and the compiler's register allocation usually sits just above a step of
    the occupancy staircase.  Measured on B200 at 134 M rows (tools/corpus_bench.py): generated
    headline gradient 80 registers -> 64: 0.861 -> 0.798 ms; headline primal 58 -> 48: 0.530 ->
    0.509 ms; stencil_smooth gradient 64 -> 48: 0.387 -> 0.373 ms; safe_divide primal / gradient
    0.260 -> 0.231 / 0.414 -> 0.358 ms; the others unchanged within 1 %.  A bound BELOW what the
    compiler chose is never set (it then spends the extra registers and loses occupancy), and a
    kernel that would spill more than a few values keeps its own allocation.  First use compiles the
    module twice; both images land in the on-disk cache.  KRN_RETUNE=0 switches this off."""
    key = id(dev)
    hit = plan.__dict__.setdefault("_tuned", {}).get(key)
    if hit is not None:
        return dev.module(hit)
    base = dev.module(plan.source)
    # kernels that scatter with hardware atomics are bound by random sector traffic, not by latency:
    # more resident blocks only add contention (gather_rows_rank2 gradient 13.4 -> 14.0 ms)
    names = [st[2]["name"] for st in plan.steps if st[0] == "group" and not st[2].get("atomic_views")]
    want: dict = {}
    before: dict = {}
    if os.environ.get("KRN_RETUNE", "1") != "0":
        for name in names:
            regs, local, _ = before[name] = dev.kernel_info(base, name)
            blocks = 65536 // (((regs + 7) // 8 * 8) * 256)  # registers are allocated in units of 8 per thread
            if regs > 40 and blocks < 6:
                want[name] = blocks + 1
    source, module = plan.source, base
    while want:
        source = "".join(f"#define KRN_MINB_{n} , {k}\n" for n, k in sorted(want.items())) + plan.source
        module = dev.module(source)
        spilled = [n for n in want if dev.kernel_info(module, n)[1] > before[n][1] + 64]
        if not spilled:
            break
        for n in spilled:
            del want[n]
        source, module = plan.source, base
    plan._tuned[key] = source
    return module


def plan_for(fn, windows: bool = True, track: bool = False):
    """Plan of `fn`; with `windows` the halo-recompute fusion is tried first (the plan's
    `.windowed` says whether any group uses it).  `track`: the check_finite variant, or None when
    some statement of `fn` cannot be watched from inside a fused kernel."""
    key = (id(fn), bool(windows), bool(track))
    hit = _plans.get(key)
    if hit is not None and hit[0] is fn:
        return hit[1]
    plan = None
    if windows:
        try:
            plan = CompiledPlan(fn, True, track)
        except ValueError:
            plan = None  # shape outside the window kernel: plain tile kernels
    if plan is None:
        try:
            plan = CompiledPlan(fn, False, track)
        except tilegen.Untrackable:
            plan = None
    _plans[key] = (fn, plan)
    return plan


def host_eval(e, H: dict, views: dict):
    k = kind(e)
    if k == "Literal":
        return np.float64(e.value)
    if k == "ScalarVar":
        return H[e.name]
    if k == "Extent":
        return np.float64(views[e.view].extents[e.dim])
    if k == "Neg":
        return -host_eval(e.operand, H, views)
    if k == "Binary":
        a, b = host_eval(e.lhs, H, views), host_eval(e.rhs, H, views)
        with np.errstate(all="ignore"):
            return a + b if e.op == "+" else a - b if e.op == "-" else a * b if e.op == "*" else a / b
    raise TypeError(f"not host-evaluable: {k}")


def run(dev, fn, views: dict, scalars: dict, cfg):
    """Execute `fn`; falls back to the statement path when the dry check says a fused
    group cannot preserve the reference's error behaviour."""
    from .runtime import _Run, _plan_for

    track = bool(cfg.check_finite)
    plan = plan_for(fn, cfg.fuse_neighbours, track)
    if plan is None:  # check_finite and a statement no fused kernel can watch
        return _Run(dev, _plan_for(fn), views, scalars, cfg).go()
    r = _CompiledRun(dev, plan, views, scalars, cfg)
    if not r.dry_check() and plan.windowed:
        alt = plan_for(fn, False, track)
        if alt is not None:
            r = _CompiledRun(dev, alt, views, scalars, cfg)
            if r.dry_check():
                return r.go()
        return _Run(dev, _plan_for(fn), views, scalars, cfg).go()
    if not r.dry_check():
        return _Run(dev, _plan_for(fn), views, scalars, cfg).go()
    return r.go()


class _Borrowed:
    """A device pointer owned by someone else (the context's scalar slots)."""

    __slots__ = ("ptr",)

    def __init__(self, ptr: int):
        self.ptr = ptr


class _CompiledRun:
    def __init__(self, dev, plan: CompiledPlan, views, scalars, cfg):
        self.dev, self.plan, self.views, self.cfg = dev, plan, views, cfg
        self.b = plan.builder
        self.H = {k: np.float64(v) for k, v in scalars.items()}
        self.stage: dict = {}
        self.ret_slot = None
        self.host_value = None

    # ---- host-only rehearsal ----------------------------------------------------------
    def dry_check(self) -> bool:
        """Memoised per plan on the extents of the bound Views (the check depends on nothing else,
        apart from aliasing, which is looked at every time)."""
        objs = [id(v) for v in self.views.values()]
        if len(set(objs)) != len(objs):
            return False  # one storage object bound to two names: registers/windows would hide the aliasing
        key = tuple((k, v.extents) for k, v in self.views.items())
        memo = self.plan.__dict__.setdefault("_dry_memo", {})
        hit = memo.get(key)
        if hit is None:
            if len(memo) > 256:
                memo.clear()
            hit = memo[key] = self._dry_check()
        return hit

    def _dry_check(self) -> bool:
        from .runtime import _index_value

        ext = {k: v.extents for k, v in self.views.items()}

        class _V:  # extents-only stand-in for _index_value
            def __init__(self, e):
                self.extents = e

        def trip(e):
            return int(_index_value(e, {k: _V(v) for k, v in ext.items()}))

        try:
            for step in self.plan.steps:
                tag = step[0]
                if tag == "declview":
                    s = step[1]
                    args = iter(s.dyn_args)
                    dims = tuple(e.size if kind(e) == "StaticExtent" else trip(next(args)) for e in s.descriptor.extents)
                    if any(d < 0 for d in dims):
                        return False
                    ext[s.name] = dims
                elif tag == "group":
                    g, recipe = step[1], step[2]
                    n = trip(g.ops[0].upper)
                    if n < 0:
                        return False
                    promoted = {p["view"] for p in recipe["promoted"]}
                    for loop in g.ops:
                        if loop.what == "apply":
                            continue
                        if trip(loop.upper) != n:
                            return False
                        if loop.what in ("deepcopy", "suminto"):
                            st = loop.origin
                            if isinstance(st.src, str) and ext[st.dst] != ext[st.src]:
                                return False
                        for v in fusion_views(loop) & promoted:
                            if n > ext[v][0]:
                                return False  # would be OutOfBounds: let the statement path report it
                        for v, ncols in loop.need_cols.items():
                            if ext[v][1] != ncols:
                                return False  # a bulk statement unrolled over the columns the function names
                    for p in recipe["promoted"]:
                        if "cols" in p and p["cols"] and max(p["cols"]) >= ext[p["view"]][1]:
                            return False  # a literal column outside the View: the statement path reports it
                    if g.gather is not None and ext[g.gather[0].src][0] != n:
                        return False
                    if recipe.get("gather_cols") and ext[g.gather[0].src][1] != recipe["gather_cols"]:
                        return False  # the fused flat reduction was laid out for exactly these columns
                    for v in recipe["elided_views"]:
                        if n > ext[v][0]:
                            return False  # the elided checks assumed extent >= range
                    if self.plan.track and any(ext[p["view"]][0] != n for p in recipe["promoted"]):
                        return False  # check_finite: rows the kernel does not visit would go untested
                    for v in recipe.get("alt", ()):
                        if ext[v][0] > n + recipe["max_shift"]:
                            return False  # rows the kernel does not cover would be lost in the buffer swap
        except (TypeError, KeyError):
            return False
        return True

    # ---- launching -----------------------------------------------------------------------
    def env(self, ptrs: dict, needed=None, atomic=(0, 0, 0, 0, 0, 0)) -> bytes:
        """Kernel argument block.  `ptrs`: explicit device pointers (promoted Views);
        `needed`: the other Views the kernel touches - only those are materialised on the
        device (None = every View of the function, for kernels that are not analysed)."""
        b = self.b
        nv, nh = max(len(b.views), 1), max(len(b.hslots), 1)
        p, e0, e1 = [0] * nv, [0] * nv, [0] * nv
        for i, name in enumerate(b.views):
            v = self.views.get(name)
            if v is None:
                continue
            e0[i] = v.extents[0]
            e1[i] = v.extents[1] if len(v.extents) == 2 else 1
            if name in ptrs:
                p[i] = ptrs[name]
            elif needed is None or name in needed:
                p[i] = v.device_ptr(self.dev)
        h = [0.0] * nh
        for name, slot in b.hslots.items():
            h[slot] = float(self.H.get(name, 0.0))
        self._shared = 8 * atomic[0] if atomic[1] == 2 else 0
        from .runtime import ENV_TAIL

        fin = self.fin.ptr if getattr(self, "fin", None) is not None else 0
        return struct.pack(f"{nv}Q{nv}q{nv}qQQ{nh}d" + ENV_TAIL, *p, *e0, *e1, self.S.ptr, self.dev.status_ptr, *h,
                           *atomic, fin)

    def launch_raw(self, name, grid_items, env_bytes, extra):
        env = C.create_string_buffer(env_bytes)
        holders, args = [env], [C.addressof(env)]
        for x in extra:
            h = C.c_longlong(x) if isinstance(x, int) else x
            holders.append(h)
            args.append(C.addressof(h))
        arr = (C.c_void_p * len(args))(*args)
        _cabi.check(self.dev.lib.krn_module_launch(self.dev.h, self.mod, name.encode(), grid_items,
                                                   getattr(self, "_shared", 0), arr))

    def go(self):
        from .runtime import _DeviceBuffer

        dev = self.dev
        # small problems are launch-latency bound: the compiler's own allocation, one compilation
        big = any(v.size >= RETUNE_MIN_ELEMENTS for v in self.views.values())
        self.mod = retuned_module(dev, self.plan) if big else dev.module(self.plan.source)
        # status word and scalar slots live side by side in the context: one memset starts the run
        slots, cap = C.c_void_p(), C.c_size_t()
        _cabi.check(dev.lib.krn_run_begin(dev.h, C.byref(slots), C.byref(cap)))
        if self.plan.nslots <= cap.value:
            self.S = _Borrowed(slots.value)
        else:
            self.S = _DeviceBuffer(dev, 8 * self.plan.nslots)
            dev.fill(self.S.ptr, self.plan.nslots, 0.0)
        self.fin = None
        self.block = None  # (capacity in slots) when status word, scalar slots and flags are one block
        if self.plan.track:
            self.start_tracking(slots.value, cap.value)
        # scalar parameters the function redefines with device data (a gather into the parameter,
        # arithmetic on View elements) live in the slot array: start them at the caller's value
        for p in self.plan.fn.params:
            if not p.is_view and p.name not in self.plan.an.host_scalars:
                dev.fill(self.S.ptr + 8 * self.b.slot(p.name), 1, float(self.H[p.name]))
        for step in self.plan.steps:
            getattr(self, "do_" + step[0])(*step[1:])
        return self.finish()

    # ---- check_finite inside the fused kernels ---------------------------------------------------
    def start_tracking(self, slots: int, cap: int):
        """fin[checkpoint][view]: one int per (statement, View), set by the kernels when the statement
        leaves a non-finite value in the View.  Row 0 is the state the Views come in with: parameter
        Views that no kernel tests when it loads them are probed here (krn_check_finite), unless the
        first statement overwrites them before the reference's first check.  The flags live behind the
        scalar slots of the context's status block when they fit (krn_run_begin has cleared it): no
        memset of their own, and status word, scalars and flags come back with ONE copy (finish)."""
        from .runtime import _DeviceBuffer

        dev, b = self.dev, self.b
        nv = max(len(b.views), 1)
        rows = len(b.track) + 1
        if isinstance(self.S, _Borrowed) and 8 * self.plan.nslots + 4 * rows * nv <= 8 * cap:
            self.fin = _Borrowed(slots + 8 * self.plan.nslots)
            self.block = cap
        else:
            self.fin = _DeviceBuffer(dev, 4 * rows * nv)
            _cabi.check(dev.lib.krn_memset(dev.h, C.c_void_p(self.fin.ptr), 0, 4 * rows * nv))
        first = next((c for c in self.plan.checkpoints if c[0] == "views"), None)
        for p in self.plan.fn.params:
            if not p.is_view or p.name in b.init_tested:
                continue
            v = self.views[p.name]
            if v.size == 0 or v._zero or (first is not None and p.name in first[2]):
                continue
            dev.check_finite(v.device_ptr(dev, write=False), v.size, self.fin.ptr + 4 * b.vid(p.name))

    def finite_replay(self):
        """The reference's checks, replayed on the host from the recorded flags: after every kernel /
        bulk statement the first View (parameters in order, then locals as declared) holding a
        non-finite value raises; after every gather its scalar (runtime.py:624-676)."""
        from .runtime import NonFiniteDetected

        dev, b = self.dev, self.b
        nv = max(len(b.views), 1)
        rows = len(b.track) + 1
        if self.block is not None:  # already on the host: finish() fetched the whole block
            slots = dev.staging[64 : 64 + 8 * self.plan.nslots].view(np.float64)
            first = 64 + 8 * self.plan.nslots
            flags = dev.staging[first : first + 4 * rows * nv].view(np.int32).reshape(rows, nv)
        else:
            flags = np.zeros((rows, nv), dtype=np.int32)
            dev.download(flags, self.fin.ptr)
            slots = np.zeros(self.plan.nslots)
            dev.download(slots, self.S.ptr)
        order = [p.name for p in self.plan.fn.params if p.is_view]
        bad = {name: bool(flags[0, b.vid(name)]) for name in order}
        for cpt in self.plan.checkpoints:
            if cpt[0] == "decl":
                order.append(cpt[1])
                bad[cpt[1]] = False
            elif cpt[0] == "views":
                for name in cpt[2]:
                    bad[name] = bool(flags[cpt[1], b.vid(name)])
                for name in order:
                    if bad[name]:
                        raise NonFiniteDetected(f"non-finite value in view '{name}'")
            elif cpt[0] == "scalar":
                value = float(slots[b.slot(cpt[1])]) if cpt[1] not in self.plan.an.host_scalars else float(self.H[cpt[1]])
                if not np.isfinite(value):
                    raise NonFiniteDetected(f"non-finite scalar {value!r}")

    def do_declview(self, s):
        from .runtime import ViewStorage, _index_value

        args = iter(s.dyn_args)
        dims = [e.size if kind(e) == "StaticExtent" else int(_index_value(next(args), self.views))
                for e in s.descriptor.extents]
        self.views[s.name] = ViewStorage.zeros(s.name, dims)

    def do_hostscalar(self, s):
        v = host_eval(s.init if kind(s) == "DeclScalar" else s.rhs, self.H, self.views)
        if kind(s) == "DeclScalar" or s.op == "=":
            self.H[s.name] = v
        elif s.op == "+=":
            self.H[s.name] = self.H[s.name] + v
        else:
            self.H[s.name] = self.H[s.name] - v

    def do_group(self, g, recipe):
        from .runtime import _DeviceBuffer, _index_value

        dev = self.dev
        n = int(_index_value(g.ops[0].upper, self.views))
        n_launch = n + recipe["max_shift"]
        if n_launch <= 0:
            if g.gather is not None:
                self.do_gather(*g.gather)
            return
        ptrs, zero_mask, n_safe = {}, 0, n
        alt_bufs: dict = {}
        alt_views = set(recipe.get("alt", ()))
        for k_, p in enumerate(recipe["promoted"]):
            v = self.views[p["view"]]
            rows = v.extents[0]
            n_safe = min(n_safe, rows)
            zero = bool(v._zero)
            if p["view"] in alt_views:
                # out of place: the kernel reads the old buffer (neighbouring warps included) and
                # writes a fresh one, which the View adopts afterwards
                alt_bufs[p["view"]] = _DeviceBuffer(dev, v.nbytes)
                if zero:
                    zero_mask |= 1 << k_
                    ptrs[p["view"]] = 0
                else:
                    ptrs[p["view"]] = v.device_ptr(dev, write=False)
                continue
            if zero and p["store"] and rows > n_launch:
                zero = False  # rows the kernel does not cover must really hold zeros
            if zero:
                zero_mask |= 1 << k_
            if p["store"]:
                # rank-2 register columns: only the written columns are stored, so the others must
                # really hold their zeros (the kernel still skips the loads)
                partial = "cols" in p and {c for c in p["cols"] if p["col_store"][c]} != set(range(v.extents[1]))
                ptrs[p["view"]] = v.device_ptr(dev, discard=zero and not partial)
            elif zero and not p.get("nbr"):
                ptrs[p["view"]] = 0
            else:
                # (neighbour registers: the first and last steps of the range read the View through
                # bounds-checked loads, so a lazily zero one needs its buffer all the same)
                ptrs[p["view"]] = v.device_ptr(dev, write=False)
        ld = ((n_launch + 3) // 4) * 4 + tilegen.STRIDE_PAD
        stage_ptr = 0
        if recipe["stage_cols"]:
            producer = recipe["stage_cols"][0][0]
            ncols = max(idx for _, idx in recipe["stage_cols"]) + 1
            buf = _DeviceBuffer(dev, 8 * ncols * ld)
            self.stage[producer] = (buf, ld)
            stage_ptr = buf.ptr
        for loop in g.ops:
            if loop.what == "apply" and id(loop.apply_of[2]) in self.stage:
                buf, ld = self.stage[id(loop.apply_of[2])]  # contributions staged by an earlier launch
                stage_ptr = buf.ptr
        blocks_items = n_launch
        red_out, acc, partials, scratch, ticket = 0, 0, 0, 0, 0
        if g.gather is not None:
            stmt, accumulate = g.gather
            red_out, acc = self.S.ptr + 8 * self.b.slot(stmt.dst), int(accumulate)
        needed = recipe.get("_needed")
        if needed is None:  # Views the kernel touches (walks the tree: once per plan, not per call)
            needed = set()
            for loop in g.ops:
                if loop.what == "apply":
                    needed.add(loop.apply_of[0])
                    continue
                staged = {st.view for st in loop.sites if st.mode == "gather"}
                needed |= {a.view for a in loop.accesses() if not (a.atomic and a.view in staged)}
            recipe["_needed"] = needed
        from .runtime import atomic_choice

        choice, ordered = atomic_choice(dev, self.cfg, recipe, self.views, self.b, n, recipe.get("static_smem", 0))
        env = self.env(ptrs, needed - set(ptrs), choice)
        extra = [n, n_launch, n_safe, C.c_uint(zero_mask), C.c_void_p(stage_ptr), ld]
        # steps per warp (a power of two: a block is a node of the reduction tree).  Measured on B200 at
        # 134 M rows (tools/corpus_bench.py): kernels that end in a fused reduction pay a block-level
        # tree, a ticket and a partial per block and run best with 8 (4: -4%, 1: -50%); kernels without
        # one run best with 2 (8: -2..4%, 1: -2..5%).  Small problems are latency bound: as many
        # blocks as possible.
        reduces = g.gather is not None or bool(g.sides)
        steps = 1 if n_launch <= (1 << 20) else (8 if reduces else 2)
        nblocks = (n_launch + 1024 * steps - 1) // (1024 * steps)
        side_args = [C.c_void_p(0), C.c_int(0)] * fusion.MAX_SIDES
        if reduces:
            # the context's reduction workspace: no allocation inside the launch sequence; one run of
            # nblocks partials for the fused gather, one more per side gather
            pa, sc, tk = C.c_void_p(), C.c_void_p(), C.c_void_p()
            _cabi.check(dev.lib.krn_reduce_workspace(
                dev.h, nblocks * (max(1, recipe.get("gather_cols", 0)) + len(g.sides)), C.byref(pa), C.byref(sc),
                C.byref(tk)))
            extra += [pa, sc, tk, C.c_void_p(red_out), C.c_int(acc)]
            for j, (stmt, accumulate, _) in enumerate(g.sides):
                side_args[2 * j] = C.c_void_p(self.S.ptr + 8 * self.b.slot(stmt.dst))
                side_args[2 * j + 1] = C.c_int(int(accumulate))
        else:
            extra += [C.c_void_p(0), C.c_void_p(0), C.c_void_p(0), C.c_void_p(0), C.c_int(0)]
        extra.append(C.c_int(steps))
        if recipe.get("window"):
            order = list(recipe["alt"]) + [None] * (fusion.MAX_ALT - len(recipe["alt"]))
            extra += [C.c_void_p(alt_bufs[v].ptr if v is not None else 0) for v in order]
        extra += side_args
        self.launch_tile(recipe["name"], nblocks, env, extra)
        for name, buf in alt_bufs.items():
            self.views[name]._adopt(buf)
        if ordered is not None:
            ordered.apply()

    def launch_tile(self, name, nblocks, env_bytes, extra):
        # krn_module_launch sizes a grid-stride grid; tile kernels need exactly ceil(threads/256) blocks
        env = C.create_string_buffer(env_bytes)
        holders, args = [env], [C.addressof(env)]
        for x in extra:
            h = C.c_longlong(x) if isinstance(x, int) else x
            holders.append(h)
            args.append(C.addressof(h))
        arr = (C.c_void_p * len(args))(*args)
        _cabi.check(self.dev.lib.krn_module_launch_exact(self.dev.h, self.mod, name.encode(), nblocks, 256,
                                                         getattr(self, "_shared", 0), arr))

    def do_kernel(self, loop, recipe):
        from .runtime import _DeviceBuffer, _index_value

        n = int(_index_value(loop.upper, self.views))
        stage = ostage = None
        extra = [max(n, 0), C.c_void_p(0), C.c_void_p(0)]
        if recipe["n_staged"] and n > 0:
            stage = _DeviceBuffer(self.dev, 8 * recipe["n_staged"] * n)
            extra[1] = C.c_void_p(stage.ptr)
            if recipe["needs_offsets"]:
                ostage = _DeviceBuffer(self.dev, 8 * recipe["n_staged"] * n)
                extra[2] = C.c_void_p(ostage.ptr)
        if n > 0:
            from .runtime import atomic_choice

            needed = _views_in_stmts([loop])
            choice, ordered = atomic_choice(self.dev, self.cfg, recipe, self.views, self.b, n)
            self.launch_raw(recipe["name"], n, self.env({}, needed, choice), extra)
            for ap in recipe["apply"]:
                if ordered is not None and ap["over"] == "iterations":
                    continue  # the staged contributions went to the ordered queue instead
                count = self.views[ap["view"]].extents[0] if ap["over"] == "rows" else n
                if count > 0:
                    self.launch_raw(ap["name"], count, self.env({}, needed), extra)
            if ordered is not None:
                ordered.apply()

    def do_deepcopy(self, s):
        from .runtime import ShapeMismatch

        d = self.views[s.dst]
        if isinstance(s.src, str):
            src = self.views[s.src]
            if d.extents != src.extents:
                raise ShapeMismatch(f"deep_copy: {s.dst}{d.extents} vs {s.src}{src.extents}")
            self.dev.copy(d.device_ptr(self.dev, discard=True), src.device_ptr(self.dev, write=False), d.size)
        else:
            value, dptr = self.scalar_operand(s.src)
            self.dev.fill(d.device_ptr(self.dev, discard=True), d.size, value, dptr)

    def do_suminto(self, s):
        from .runtime import ShapeMismatch

        d = self.views[s.dst]
        if isinstance(s.src, str):
            src = self.views[s.src]
            if d.extents != src.extents:
                raise ShapeMismatch(f"parallel_sum: {s.dst}{d.extents} vs {s.src}{src.extents}")
            self.dev.add_view(d.device_ptr(self.dev), src.device_ptr(self.dev, write=False), d.size)
        else:
            value, dptr = self.scalar_operand(s.src)
            self.dev.add_scalar(d.device_ptr(self.dev), d.size, value, dptr)

    def scalar_operand(self, src):
        if kind(src) == "Literal":
            return float(src.value), 0
        if src.name in self.H and src.name in self.plan.an.host_scalars:
            return float(self.H[src.name]), 0
        return 0.0, self.S.ptr + 8 * self.b.slot(src.name)

    def do_gather(self, s, accumulate):
        src = self.views[s.src]
        out = self.S.ptr + 8 * self.b.slot(s.dst)
        self.dev.reduce_pairwise(src.device_ptr(self.dev, write=False), src.size, out, accumulate)

    def do_scalars(self, recipe, needed):
        self.launch_raw(recipe["name"], 1, self.env({}, needed), [])

    def do_return(self, recipe, needed):
        self.launch_raw(recipe["name"], 1, self.env({}, needed), [])
        self.ret_slot = recipe["slot"]

    def do_slotreturn(self, slot):
        self.ret_slot = slot

    def do_hostreturn(self, expr):
        self.host_value = float(host_eval(expr, self.H, self.views))

    def finish(self):
        from .runtime import _Run

        dev = self.dev
        if not self.cfg.synchronous:
            return None
        st = dev.staging[:64].view(np.int64)
        if self.block is not None:
            # check_finite: status word, every scalar slot and the flags in one copy
            dev.download(dev.staging[: 64 + 8 * self.block], dev.status_ptr)
            out = dev.staging[64 + 8 * (self.ret_slot or 0) :][:8].view(np.float64)
        else:
            out = dev.staging[64:72].view(np.float64)
            if self.ret_slot is not None:
                dev.download_async(out, self.S.ptr + 8 * self.ret_slot)
            dev.download(st, dev.status_ptr)
        if st[0] != 0:
            helper = _Run.__new__(_Run)
            helper.b, helper.views = self.b, self.views
            raise helper.error_from(st.copy())
        value = float(out[0]) if self.ret_slot is not None else self.host_value
        if self.plan.track:
            from .runtime import NonFiniteDetected

            self.finite_replay()
            if value is not None and not np.isfinite(value):
                raise NonFiniteDetected(f"non-finite scalar {value!r}")
        return value


def fusion_views(loop) -> set:
    return {a.view for a in loop.accesses()}
