"""Symbolic vector-Jacobian factors of a right-hand side.

For an assignment ``lhs = rhs`` with incoming adjoint ``adj`` the reverse
sweep adds, for every differentiable leaf occurrence ``o`` of ``rhs``
(scalar variable or view access, left to right), ``adj * d rhs / d o`` into
the shadow of ``o``.  ``contributions`` returns those products as
expression trees.  The *shape* of each product is part of the contract with
the reference (/root/reference/pkg/src/krn/partials.py:34-69): the adjoint
factor sits where the occurrence sat (``u*v`` gives ``adj*v`` and ``u*adj``),
which fixes the floating-point evaluation order of every generated kernel
and therefore the bits the GPU kernels must reproduce.
"""

from __future__ import annotations

from .nodes import Binary, Neg, ScalarVar, kind, walk_expr


class NonDifferentiableOp(Exception):
    pass


def contributions(rhs, adj) -> list:
    """[(occurrence node, contribution expression)] in left-to-right order."""
    out: list = []
    # explicit stack of (sub-expression, adjoint flowing into it); children are
    # pushed right-first so leaves pop in source order
    todo = [(rhs, adj)]
    while todo:
        e, a = todo.pop()
        k = kind(e)
        if k in ("Literal", "IndexVar", "Extent"):
            continue
        if k in ("ScalarVar", "ViewAccess"):
            out.append((e, a))
        elif k == "Neg":
            todo.append((e.operand, Neg(a)))
        elif k == "Binary":
            u, v = e.lhs, e.rhs
            if e.op == "+":
                pair = (a, a)
            elif e.op == "-":
                pair = (a, Neg(a))
            elif e.op == "*":
                pair = (Binary("*", a, v), Binary("*", u, a))
            elif e.op == "/":
                pair = (
                    Binary("/", a, v),
                    Neg(Binary("/", Binary("*", u, a), Binary("*", v, v))),
                )
            else:
                raise NonDifferentiableOp(f"no derivative rule for operator {e.op!r}")
            todo.append((v, pair[1]))
            todo.append((u, pair[0]))
        else:
            raise NonDifferentiableOp(f"no derivative rule for {k}")
    return out


_ADJ = "__adj__"


def needed_primal_names(rhs, occ_is_active) -> set:
    """Views/scalars whose forward values the reversal of ``rhs`` re-reads
    (empty for an rhs affine in its active leaves)."""
    names: set = set()
    for occ, expr in contributions(rhs, ScalarVar(_ADJ)):
        if not occ_is_active(occ):
            continue
        for n in walk_expr(expr):
            k = kind(n)
            if k == "ScalarVar" and n.name != _ADJ:
                names.add(n.name)
            elif k == "ViewAccess":
                names.add(n.view)
    return names
