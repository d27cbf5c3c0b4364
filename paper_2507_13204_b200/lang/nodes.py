"""Tree vocabulary of the kernel language (``.krn``).

Node names and field names mirror the reference's ``krn.ast``
(/root/reference/pkg/src/krn/ast.py:94-343) on purpose: the GPU executor
dispatches on ``type(node).__name__`` and attribute names only, so a tree
built by the reference package can be handed to this package's ``execute``
unchanged, and the other way round.  Everything else in this file (how
nodes are declared, the traversal helpers) is this package's own.

Two sub-languages share the vocabulary:

* value expressions (f64): Literal, ScalarVar, IndexVar, ViewAccess,
  Extent, Binary, Neg
* index expressions (integers): Counter, IntLiteral, Extent, IdxBinary and
  ViewAccess (indirect indexing)

All nodes are immutable, hashable, and compare structurally with the
source location ignored.
"""

from __future__ import annotations

import dataclasses as _dc
from typing import Iterator, Union


@_dc.dataclass(frozen=True)
class SourceSpan:
    start: int = 0
    end: int = 0
    line: int = 0
    col: int = 0


NO_SPAN = SourceSpan()


class Node:
    """Common base of every tree node (the reference's ``krn.ast.Node``, ast.py:35): lets callers
    write ``isinstance(x, Node)``.  Carries nothing; ``_node`` adds the ``span`` field."""

    __slots__ = ()


def _node(cls):
    """Class decorator: frozen dataclass + keyword-only ``span`` excluded
    from equality, list-valued fields coerced to tuples."""
    ann = dict(cls.__dict__.get("__annotations__", {}))
    ann["span"] = SourceSpan
    cls.__annotations__ = ann
    cls.span = _dc.field(default=NO_SPAN, compare=False, repr=False, kw_only=True)
    user_post = cls.__dict__.get("__post_init__")

    def __post_init__(self):
        for f in _dc.fields(self):
            v = getattr(self, f.name)
            if isinstance(v, list):
                object.__setattr__(self, f.name, tuple(v))
        if user_post is not None:
            user_post(self)

    cls.__post_init__ = __post_init__
    return _dc.dataclass(frozen=True)(cls)


# ---- view shapes -----------------------------------------------------------


@_dc.dataclass(frozen=True)
class StaticExtent:
    size: int


@_dc.dataclass(frozen=True)
class DynamicExtent:
    pass


@_dc.dataclass(frozen=True)
class ViewDescriptor:
    """f64, rank 1 or 2, row-major; ``extents`` defaults to all-dynamic."""

    name: str
    rank: int
    extents: tuple = ()
    element: str = "f64"

    def __post_init__(self):
        ext = tuple(self.extents) or tuple(DynamicExtent() for _ in range(self.rank))
        object.__setattr__(self, "extents", ext)

    def dynamic_count(self) -> int:
        return sum(isinstance(e, DynamicExtent) for e in self.extents)


# ---- expressions -----------------------------------------------------------


@_node
class Literal(Node):
    value: float


@_node
class ScalarVar(Node):
    name: str


@_node
class IndexVar(Node):
    name: str


@_node
class ViewAccess(Node):
    view: str
    indices: tuple


@_node
class Extent(Node):
    view: str
    dim: int


@_node
class Binary(Node):
    op: str
    lhs: object
    rhs: object


@_node
class Neg(Node):
    operand: object


@_node
class Counter(Node):
    name: str


@_node
class IntLiteral(Node):
    value: int


@_node
class IdxBinary(Node):
    op: str
    lhs: object
    rhs: object


@_node
class Compare(Node):
    op: str
    lhs: object
    rhs: object


# ---- statements ------------------------------------------------------------


@_node
class DeclView(Node):
    descriptor: ViewDescriptor
    dyn_args: tuple = ()
    label: str = ""

    def __post_init__(self):
        if not self.label:
            object.__setattr__(self, "label", self.descriptor.name)

    @property
    def name(self) -> str:
        return self.descriptor.name


@_node
class DeclScalar(Node):
    name: str
    init: object


@_node
class AssignView(Node):
    target: ViewAccess
    op: str
    rhs: object


@_node
class AssignScalar(Node):
    name: str
    op: str
    rhs: object


@_node
class If(Node):
    cond: Compare
    body: tuple


@_node
class ParallelFor(Node):
    counter: str
    upper: object
    body: tuple


@_node
class DeepCopy(Node):
    dst: str
    src: object  # view name (str) or scalar expression


@_node
class ParallelSum(Node):
    dst: str
    src: str


@_node
class ParallelSumInto(Node):
    dst: str
    src: object  # view name (str) or scalar expression


@_node
class AtomicAdd(Node):
    target: ViewAccess
    value: object


@_node
class Return(Node):
    value: object


@_node
class Param(Node):
    name: str
    type: object  # ViewDescriptor or "f64"

    @property
    def is_view(self) -> bool:
        return kind(self.type) == "ViewDescriptor"


@_node
class FunctionDef(Node):
    name: str
    params: tuple
    body: tuple
    returns: Union[str, None] = None

    def param(self, name: str):
        return next((p for p in self.params if p.name == name), None)


@_node
class Program(Node):
    functions: tuple = ()

    def function(self, name: str):
        return next((f for f in self.functions if f.name == name), None)


# ---- duck-typed helpers ----------------------------------------------------


def kind(node) -> str:
    """Class name of a node; the only thing consumers dispatch on, so trees
    from the reference package are accepted as they are."""
    return type(node).__name__


_BLOCKS = ("If", "ParallelFor")


def walk_statements(body) -> Iterator:
    """Pre-order over statements, entering If / ParallelFor bodies."""
    stack = list(reversed(tuple(body)))
    while stack:
        s = stack.pop()
        yield s
        if kind(s) in _BLOCKS:
            stack.extend(reversed(tuple(s.body)))


def walk_expr(e) -> Iterator:
    """Pre-order over an expression of either sub-language."""
    stack = [e]
    while stack:
        n = stack.pop()
        yield n
        k = kind(n)
        if k in ("Binary", "IdxBinary", "Compare"):
            stack.append(n.rhs)
            stack.append(n.lhs)
        elif k == "Neg":
            stack.append(n.operand)
        elif k == "ViewAccess":
            stack.extend(reversed(tuple(n.indices)))


def free_counters(e) -> set:
    return {n.name for n in walk_expr(e) if kind(n) in ("Counter", "IndexVar")}


def statement_exprs(stmt) -> Iterator:
    """Expressions directly owned by one statement (not its nested block)."""
    k = kind(stmt)
    if k == "DeclView":
        yield from stmt.dyn_args
    elif k == "DeclScalar":
        yield stmt.init
    elif k == "AssignView":
        yield stmt.target
        yield stmt.rhs
    elif k == "AssignScalar":
        yield stmt.rhs
    elif k == "If":
        yield stmt.cond
    elif k == "ParallelFor":
        yield stmt.upper
    elif k in ("DeepCopy", "ParallelSumInto"):
        if not isinstance(stmt.src, str):
            yield stmt.src
    elif k == "AtomicAdd":
        yield stmt.target
        yield stmt.value
    elif k == "Return":
        yield stmt.value


def walk_all_exprs(fn) -> Iterator:
    for stmt in walk_statements(fn.body):
        for e in statement_exprs(stmt):
            yield from walk_expr(e)


def all_identifiers(fn) -> set:
    names = {p.name for p in fn.params}
    for s in walk_statements(fn.body):
        k = kind(s)
        if k in ("DeclView", "DeclScalar"):
            names.add(s.name)
        elif k in ("ParallelSum", "ParallelSumInto", "DeepCopy"):
            names.add(s.dst)
            if isinstance(s.src, str):
                names.add(s.src)
        elif k == "ParallelFor":
            names.add(s.counter)
    for e in walk_all_exprs(fn):
        k = kind(e)
        if k in ("ScalarVar", "IndexVar", "Counter"):
            names.add(e.name)
        elif k in ("ViewAccess", "Extent"):
            names.add(e.view)
    return names


def lhs_as_expr(stmt):
    if kind(stmt) == "AssignView":
        return stmt.target
    if kind(stmt) == "AssignScalar":
        return ScalarVar(stmt.name)
    raise TypeError(f"not an assignment: {kind(stmt)}")


_COMPOUND = {"+=": "+", "-=": "-"}


def desugar_statement(stmt):
    """``a op= e`` becomes ``a = a op e`` (reference: ast.py:398-418)."""
    k = kind(stmt)
    if k == "AssignView" and stmt.op in _COMPOUND:
        return AssignView(
            stmt.target, "=", Binary(_COMPOUND[stmt.op], stmt.target, stmt.rhs), span=stmt.span
        )
    if k == "AssignScalar" and stmt.op in _COMPOUND:
        return AssignScalar(
            stmt.name,
            "=",
            Binary(_COMPOUND[stmt.op], ScalarVar(stmt.name), stmt.rhs),
            span=stmt.span,
        )
    if k == "If":
        return If(stmt.cond, tuple(map(desugar_statement, stmt.body)), span=stmt.span)
    if k == "ParallelFor":
        return ParallelFor(
            stmt.counter, stmt.upper, tuple(map(desugar_statement, stmt.body)), span=stmt.span
        )
    return stmt


def desugar_function(fn):
    return FunctionDef(
        fn.name, fn.params, tuple(map(desugar_statement, fn.body)), fn.returns, span=fn.span
    )


def fresh_name(base: str, taken) -> str:
    """``base`` if free, else ``base2``, ``base3``, ..."""
    if base not in taken:
        return base
    k = 2
    while f"{base}{k}" in taken:
        k += 1
    return f"{base}{k}"
