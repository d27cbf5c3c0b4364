"""Well-formedness rules for kernel-language programs.

``validate(program)`` returns a list of ``Diagnostic`` (empty = well
formed).  The rule set is the reference's
(/root/reference/pkg/src/krn/validate.py:109-397); the GPU executor leans on
three of them to reason about launches statically:

* iteration spaces are ``0..bound`` with ``bound`` free of view data, so a
  launch shape is known before any kernel runs;
* ``if`` conditions compare index expressions only, so guards are uniform
  functions of the iteration number;
* kernel bodies contain only element assignments, loop-local scalars,
  guards and atomic accumulates - no nested parallelism or bulk operations.
"""

from __future__ import annotations

import dataclasses as _dc
import re

from .nodes import SourceSpan, kind

RESERVED = frozenset(
    "fn let if in return parallel_for parallel_sum deep_copy atomic_add view extent f64".split()
)

_NAME = re.compile(r"[A-Za-z_][A-Za-z0-9_]*\Z")
_ASSIGN_OPS = ("=", "+=", "-=")
_CMP_OPS = ("==", "!=", "<", "<=", ">", ">=")
_NOT_IN_KERNEL = ("DeclView", "DeepCopy", "ParallelSum", "ParallelSumInto", "Return")


@_dc.dataclass(frozen=True)
class Diagnostic:
    span: SourceSpan
    message: str

    def __str__(self) -> str:
        return f"{self.span.line}:{self.span.col}: {self.message}" if self.span.line else self.message


def _span(node) -> SourceSpan:
    return getattr(node, "span", None) or SourceSpan()


class _Pass:
    def __init__(self):
        self.out: list = []
        self.fn_names: dict = {}
        self.loop_names: dict = {}

    def fail(self, where, msg):
        self.out.append(Diagnostic(_span(where) if not isinstance(where, SourceSpan) else where, msg))

    # symbol table ------------------------------------------------------------

    def sym(self, name):
        return self.loop_names.get(name, self.fn_names.get(name))

    def good_name(self, name, where, what):
        if not _NAME.match(name or ""):
            self.fail(where, f"invalid {what} name {name!r}")
        elif name in RESERVED:
            self.fail(where, f"{what} name '{name}' is a reserved word")

    def bind(self, name, what, where, loop_local=False):
        self.good_name(name, where, "variable")
        if name in self.fn_names or name in self.loop_names:
            self.fail(where, f"'{name}' shadows an existing declaration")
            return
        (self.loop_names if loop_local else self.fn_names)[name] = what

    # program / function ---------------------------------------------------------

    def program(self, prog):
        seen = set()
        for fn in prog.functions:
            if fn.name in seen:
                self.fail(fn, f"duplicate function name '{fn.name}'")
            seen.add(fn.name)
            self.function(fn)

    def function(self, fn):
        self.good_name(fn.name, fn, "function")
        self.fn_names, self.loop_names = {}, {}
        for p in fn.params:
            self.good_name(p.name, p, "parameter")
            if p.name in self.fn_names:
                self.fail(p, f"duplicate parameter '{p.name}'")
            elif p.is_view:
                self.shape(p.type, p)
                self.fn_names[p.name] = ("view", p.type.rank)
            elif p.type == "f64":
                self.fn_names[p.name] = "scalar"
            else:
                self.fail(p, f"parameter '{p.name}' has unknown type {p.type!r}")
        last = len(fn.body) - 1
        for i, s in enumerate(fn.body):
            self.stmt(s, False, i == last)
        ends_in_return = bool(fn.body) and kind(fn.body[-1]) == "Return"
        if fn.returns == "f64" and not ends_in_return:
            self.fail(fn, f"function '{fn.name}' declares -> f64 but has no return")
        if fn.returns is None and ends_in_return:
            self.fail(fn.body[-1], f"void function '{fn.name}' returns a value")

    def shape(self, d, where):
        if d.rank not in (1, 2):
            self.fail(where, f"view '{d.name}' has rank {d.rank}; only 1 and 2 are supported")
        if len(d.extents) != d.rank:
            self.fail(where, f"view '{d.name}' has {len(d.extents)} extents for rank {d.rank}")
        for e in d.extents:
            if kind(e) == "StaticExtent" and e.size < 1:
                self.fail(where, f"view '{d.name}' has non-positive static extent {e.size}")

    # statements ------------------------------------------------------------------

    def stmt(self, s, in_kernel, last_of_fn=False):
        k = kind(s)
        fn = getattr(self, "s_" + k, None)
        if fn is None:
            self.fail(s, f"unknown statement {k}")
            return
        fn(s, in_kernel, last_of_fn)

    def s_DeclView(self, s, in_kernel, _):
        if in_kernel:
            self.fail(s, "view declarations are not allowed inside parallel_for")
            return
        self.bind(s.name, ("view", s.descriptor.rank), s)
        self.shape(s.descriptor, s)
        want = s.descriptor.dynamic_count()
        if len(s.dyn_args) != want:
            self.fail(s, f"view '{s.name}' needs {want} extent arguments, got {len(s.dyn_args)}")
        for a in s.dyn_args:
            self.index(a, False, "view extent")

    def s_DeclScalar(self, s, in_kernel, _):
        self.bind(s.name, "scalar", s, loop_local=in_kernel)
        self.value(s.init)

    def s_AssignView(self, s, in_kernel, _):
        self.access(s.target)
        if s.op not in _ASSIGN_OPS:
            self.fail(s, f"unknown assignment operator {s.op!r}")
        self.value(s.rhs)

    def s_AssignScalar(self, s, in_kernel, _):
        what = self.sym(s.name)
        if what is None:
            self.fail(s, f"unknown scalar '{s.name}'")
        elif what != "scalar":
            self.fail(s, f"'{s.name}' is not a scalar")
        elif in_kernel and s.name not in self.loop_names:
            self.fail(
                s,
                f"assignment to '{s.name}' inside parallel_for; only loop-local scalars "
                "may be assigned in a kernel",
            )
        if s.op not in _ASSIGN_OPS:
            self.fail(s, f"unknown assignment operator {s.op!r}")
        self.value(s.rhs)

    def s_If(self, s, in_kernel, _):
        c = s.cond
        if kind(c) != "Compare":
            self.fail(c, "if condition must be an index comparison")
        else:
            if c.op not in _CMP_OPS:
                self.fail(c, f"unknown comparison operator {c.op!r}")
            self.index(c.lhs, False, "condition")
            self.index(c.rhs, False, "condition")
        for inner in s.body:
            if kind(inner) == "Return":
                self.fail(inner, "return must be the final statement of a function")
            self.stmt(inner, in_kernel)

    def s_ParallelFor(self, s, in_kernel, _):
        if in_kernel:
            self.fail(s, "nested parallel_for is not allowed")
            return
        self.index(s.upper, False, "parallel_for bound")
        self.bind(s.counter, "counter", s, loop_local=True)
        for inner in s.body:
            if kind(inner) in _NOT_IN_KERNEL:
                self.fail(inner, f"{kind(inner)} is not allowed inside parallel_for")
            else:
                self.stmt(inner, True)
        self.loop_names = {}

    def _bulk(self, s, what):
        dst = self.sym(s.dst)
        if not isinstance(dst, tuple):
            self.fail(s, f"{what} destination '{s.dst}' is not a view")
            dst = None
        src = s.src
        if isinstance(src, str):
            sk = self.sym(src)
            if not isinstance(sk, tuple):
                self.fail(s, f"{what} source '{src}' is not a view")
            elif dst is not None and sk[1] != dst[1]:
                self.fail(
                    s,
                    f"{what} rank mismatch: '{s.dst}' is rank {dst[1]}, '{src}' is rank {sk[1]}",
                )
        elif kind(src) == "ScalarVar":
            if self.sym(src.name) != "scalar":
                self.fail(s, f"{what} source '{src.name}' is not a scalar")
        elif kind(src) != "Literal":
            self.fail(s, f"{what} source must be a view, a scalar variable, or a literal")

    def s_DeepCopy(self, s, in_kernel, _):
        if in_kernel:
            self.fail(s, "deep_copy is not allowed inside parallel_for")
            return
        self._bulk(s, "deep_copy")

    def s_ParallelSumInto(self, s, in_kernel, _):
        self._bulk(s, "parallel_sum")

    def s_ParallelSum(self, s, in_kernel, _):
        if not isinstance(self.sym(s.src), tuple):
            self.fail(s, f"parallel_sum source '{s.src}' is not a view")
        what = self.sym(s.dst)
        if what is None:  # a gather binds an unbound destination
            self.good_name(s.dst, s, "scalar")
            self.fn_names[s.dst] = "scalar"
        elif what != "scalar":
            self.fail(s, f"parallel_sum destination '{s.dst}' is not a scalar")

    def s_AtomicAdd(self, s, in_kernel, _):
        self.access(s.target)
        self.value(s.value)

    def s_Return(self, s, in_kernel, last_of_fn):
        if not last_of_fn:
            self.fail(s, "return must be the final statement of a function")
        self.value(s.value)

    # expressions -------------------------------------------------------------------

    def access(self, e):
        what = self.sym(e.view)
        if not isinstance(what, tuple):
            self.fail(e, f"unknown view '{e.view}'")
        elif len(e.indices) != what[1]:
            self.fail(
                e,
                f"view '{e.view}' has rank {what[1]} but is accessed with {len(e.indices)} indices",
            )
        for i in e.indices:
            self.index(i, True, "index")

    def extent(self, e):
        what = self.sym(e.view)
        if not isinstance(what, tuple):
            self.fail(e, f"unknown view '{e.view}' in extent")
        elif not 0 <= e.dim < what[1]:
            self.fail(e, f"extent dimension {e.dim} out of range for rank {what[1]}")

    def value(self, e):
        k = kind(e)
        if k == "Literal":
            return
        if k == "ScalarVar":
            what = self.sym(e.name)
            if what is None:
                self.fail(e, f"unknown scalar '{e.name}'")
            elif what == "counter":
                self.fail(e, f"'{e.name}' is a loop counter, not a scalar")
            elif what != "scalar":
                self.fail(e, f"'{e.name}' is a view; views are read with indices")
        elif k == "IndexVar":
            if self.sym(e.name) != "counter":
                self.fail(e, f"'{e.name}' is not a loop counter")
        elif k == "ViewAccess":
            self.access(e)
        elif k == "Extent":
            self.extent(e)
        elif k == "Binary":
            if e.op not in ("+", "-", "*", "/"):
                self.fail(e, f"unknown operator {e.op!r}")
            self.value(e.lhs)
            self.value(e.rhs)
        elif k == "Neg":
            self.value(e.operand)
        else:
            self.fail(e, f"{k} is not a value expression")

    def index(self, e, views_ok, where):
        k = kind(e)
        if k == "IntLiteral":
            return
        if k == "Counter":
            what = self.sym(e.name)
            if what is None:
                self.fail(e, f"unknown identifier '{e.name}' in {where}")
            elif what != "counter":
                self.fail(
                    e,
                    f"'{e.name}' is not a loop counter; index expressions hold counters, "
                    "integers, and extents",
                )
        elif k == "Extent":
            self.extent(e)
        elif k == "IdxBinary":
            if e.op not in ("+", "-", "*"):
                self.fail(e, f"unknown index operator {e.op!r}")
            if e.op == "*" and "IntLiteral" not in (kind(e.lhs), kind(e.rhs)):
                self.fail(e, "index multiplication needs an integer literal factor")
            self.index(e.lhs, views_ok, where)
            self.index(e.rhs, views_ok, where)
        elif k == "ViewAccess":
            if not views_ok:
                if where == "condition":
                    self.fail(
                        e,
                        "active condition unsupported: view values may not appear in if conditions",
                    )
                else:
                    self.fail(e, f"view access is not allowed in a {where}")
            self.access(e)
        else:
            self.fail(e, f"{k} is not an index expression")


def validate(program) -> list:
    p = _Pass()
    p.program(program)
    return p.out
