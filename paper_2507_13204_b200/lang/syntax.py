"""Concrete syntax of ``.krn`` files: text -> tree (``parse``) and
tree -> canonical text (``emit``).

Grammar and canonical form follow the reference front-end
(/root/reference/pkg/src/krn/parser.py:115-576 for what is accepted,
/root/reference/pkg/src/krn/printer.py:47-158 for the printed form), so a
program text is interchangeable between the two packages and
``emit(differentiate(...))`` can be compared byte for byte
(tests/golden/grad_text/*.krn).  The implementation is this package's own:
a single-pass scanner feeding a precedence-climbing parser that keeps a
symbol table (declaration before use decides whether ``name`` is a scalar,
a loop counter or a view).
"""

from __future__ import annotations

import re

from . import nodes as N
from .nodes import SourceSpan, kind

MAX_NESTING = 200

KEYWORDS = frozenset(
    "fn let if in return parallel_for parallel_sum deep_copy atomic_add view extent f64".split()
)


class ParseError(Exception):
    def __init__(self, message: str, span: SourceSpan = SourceSpan()):
        self.message = message
        self.span = span
        super().__init__(f"{span.line}:{span.col}: {message}" if span.line else message)


class ValidationError(Exception):
    def __init__(self, diagnostics):
        self.diagnostics = list(diagnostics)
        super().__init__("; ".join(str(d) for d in self.diagnostics))


# ---------------------------------------------------------------------------
# scanner

_SCAN = re.compile(
    r"(?P<skip>\s+|//[^\n]*)"
    r"|(?P<FLOAT>\d+\.\d+(?:[eE][+-]?\d+)?|\d+[eE][+-]?\d+)"
    r"|(?P<INT>\d+)"
    r"|(?P<NAME>[A-Za-z_][A-Za-z0-9_]*)"
    r'|(?P<STRING>"[^"\n]*")'
    r"|(?P<OP>->|\.\.|\+=|-=|==|!=|<=|>=|[-+*/(){}<>=,;:])"
    r"|(?P<BAD>.)",
    re.DOTALL,
)


class _Tok:
    __slots__ = ("kind", "text", "span")

    def __init__(self, kind_, text, span):
        self.kind, self.text, self.span = kind_, text, span


def _scan(text: str) -> list:
    toks = []
    line, line_start = 1, 0
    for m in _SCAN.finditer(text):
        grp, s, e = m.lastgroup, m.start(), m.end()
        span = SourceSpan(s, e, line, s - line_start + 1)
        if grp == "BAD":
            raise ParseError(f"unexpected character {m.group()!r}", span)
        if grp != "skip":
            toks.append(_Tok(m.group() if grp == "OP" else grp, m.group(), span))
        nl = text.count("\n", s, e)
        if nl:
            line += nl
            line_start = text.rfind("\n", s, e) + 1
    toks.append(_Tok("EOF", "", SourceSpan(len(text), len(text), line, len(text) - line_start + 1)))
    return toks


# ---------------------------------------------------------------------------
# parser

_ADD = ("+", "-")
_MUL = ("*", "/")
_CMP = ("==", "!=", "<", "<=", ">", ">=")


class _Reader:
    """Token cursor + symbol table for one translation unit."""

    def __init__(self, text: str):
        self.toks = _scan(text)
        self.i = 0
        self.nest = 0
        self.fn_scope: dict = {}  # name -> ("view", rank) | "scalar"
        self.kernel_scope: dict = {}  # counter / loop-local scalars

    # -- cursor ---------------------------------------------------------------

    def tok(self, ahead: int = 0) -> _Tok:
        return self.toks[min(self.i + ahead, len(self.toks) - 1)]

    def take(self, kind_):
        t = self.tok()
        if t.kind == kind_:
            self.i += 1
            return t
        return None

    def need(self, kind_, what=None) -> _Tok:
        t = self.take(kind_)
        if t is None:
            got = self.tok()
            raise ParseError(
                f"expected {what or repr(kind_)}, found {got.text or 'end of input'!r}", got.span
            )
        return t

    def word(self, literal: str) -> _Tok:
        t = self.need("NAME", f"'{literal}'")
        if t.text != literal:
            raise ParseError(f"expected '{literal}', found {t.text!r}", t.span)
        return t

    def name(self, what="identifier") -> _Tok:
        t = self.need("NAME", what)
        if t.text in KEYWORDS:
            raise ParseError(f"'{t.text}' is a reserved word", t.span)
        return t

    def sym(self, name: str):
        return self.kernel_scope.get(name, self.fn_scope.get(name))

    def view_name(self, what="view") -> _Tok:
        t = self.name(what)
        if not isinstance(self.sym(t.text), tuple):
            raise ParseError(f"unknown view '{t.text}'", t.span)
        return t

    # -- declarations ---------------------------------------------------------

    def unit(self) -> N.Program:
        fns = []
        while self.tok().kind != "EOF":
            fns.append(self.function())
        return N.Program(tuple(fns))

    def function(self) -> N.FunctionDef:
        head = self.word("fn")
        fname = self.name("function name")
        self.fn_scope, self.kernel_scope = {}, {}
        self.need("(")
        params = []
        while self.tok().kind != ")":
            if params:
                self.need(",")
            pname = self.name("parameter name")
            self.need(":")
            ty = self.type_(pname.text)
            self.fn_scope[pname.text] = "scalar" if ty == "f64" else ("view", ty.rank)
            params.append(N.Param(pname.text, ty, span=pname.span))
        self.need(")")
        returns = None
        if self.take("->"):
            t = self.need("NAME", "'f64'")
            if t.text != "f64":
                raise ParseError("only f64 returns are supported", t.span)
            returns = "f64"
        body = self.block(False)
        return N.FunctionDef(fname.text, tuple(params), tuple(body), returns, span=head.span)

    def type_(self, owner: str):
        t = self.need("NAME", "type")
        if t.text == "f64":
            return "f64"
        if t.text != "view":
            raise ParseError(f"expected 'f64' or 'view<f64,R>', found {t.text!r}", t.span)
        self.need("<")
        el = self.need("NAME", "'f64'")
        if el.text != "f64":
            raise ParseError("views hold f64 elements only", el.span)
        self.need(",")
        r = self.need("INT", "rank")
        if int(r.text) not in (1, 2):
            raise ParseError(f"rank must be 1 or 2, got {int(r.text)}", r.span)
        self.need(">")
        return N.ViewDescriptor(owner, int(r.text))

    # -- statements -----------------------------------------------------------

    def block(self, in_kernel: bool) -> list:
        self.need("{")
        out = []
        while self.tok().kind != "}":
            if self.tok().kind == "EOF":
                raise ParseError("unexpected end of input inside block", self.tok().span)
            out.extend(self.statement(in_kernel))
        self.need("}")
        return out

    def statement(self, in_kernel: bool) -> list:
        t = self.tok()
        if t.kind != "NAME":
            raise ParseError(f"expected a statement, found {t.text!r}", t.span)
        handler = {
            "let": self.st_let,
            "if": self.st_if,
            "parallel_for": self.st_pfor,
            "deep_copy": self.st_bulk,
            "parallel_sum": self.st_bulk,
            "atomic_add": self.st_atomic,
            "return": self.st_return,
        }.get(t.text, self.st_assign)
        return handler(in_kernel)

    def st_let(self, in_kernel):
        head = self.need("NAME")
        nm = self.name("variable name")
        self.need(":")
        ty = self.type_(nm.text)
        self.need("=")
        if ty == "f64":
            init = self.value()
            self.need(";")
            (self.kernel_scope if in_kernel else self.fn_scope)[nm.text] = "scalar"
            return [N.DeclScalar(nm.text, init, span=head.span)]
        ctor = self.need("NAME", "'view'")
        if ctor.text != "view":
            raise ParseError("view declarations are initialized with view(...)", ctor.span)
        self.need("(")
        label = self.need("STRING", "view label")
        dims = []
        while self.take(","):
            dims.append(self.index())
        self.need(")")
        self.need(";")
        self.fn_scope[nm.text] = ("view", ty.rank)
        return [N.DeclView(ty, tuple(dims), label.text[1:-1], span=head.span)]

    def st_if(self, in_kernel):
        head = self.need("NAME")
        self.need("(")
        lhs = self.index()
        op = self.tok()
        if op.kind not in _CMP:
            raise ParseError("expected a comparison operator", op.span)
        self.i += 1
        rhs = self.index()
        self.need(")")
        cond = N.Compare(op.kind, lhs, rhs, span=op.span)
        return [N.If(cond, tuple(self.block(in_kernel)), span=head.span)]

    def st_pfor(self, in_kernel):
        head = self.need("NAME")
        if in_kernel:
            raise ParseError("nested parallel_for is not allowed", head.span)
        ctr = self.name("loop counter")
        self.word("in")
        zero = self.need("INT", "'0'")
        if zero.text != "0":
            raise ParseError("iteration spaces start at 0", zero.span)
        self.need("..")
        upper = self.index()
        self.kernel_scope = {ctr.text: "counter"}
        body = self.block(True)
        self.kernel_scope = {}
        return [N.ParallelFor(ctr.text, upper, tuple(body), span=head.span)]

    def st_bulk(self, in_kernel):
        """``deep_copy(dst, src);`` and the accumulate form
        ``parallel_sum(dst, src);`` share their operand rules."""
        head = self.need("NAME")
        self.need("(")
        dst = self.name("destination view")
        self.need(",")
        t = self.tok()
        if t.kind == "NAME" and self.tok(1).kind == ")":
            s = self.sym(t.text)
            if isinstance(s, tuple):
                src = t.text
            elif s == "scalar":
                src = N.ScalarVar(t.text, span=t.span)
            else:
                raise ParseError(f"unknown identifier '{t.text}'", t.span)
            self.i += 1
        else:
            src = self.value()
            if kind(src) not in ("Literal", "ScalarVar"):
                raise ParseError(
                    f"{head.text} source must be a view, a scalar variable, or a literal", t.span
                )
        self.need(")")
        self.need(";")
        make = N.DeepCopy if head.text == "deep_copy" else N.ParallelSumInto
        return [make(dst.text, src, span=head.span)]

    def st_atomic(self, in_kernel):
        head = self.need("NAME")
        self.need("(")
        target = self.access(self.view_name())
        self.need(",")
        val = self.value()
        self.need(")")
        self.need(";")
        return [N.AtomicAdd(target, val, span=head.span)]

    def gather_tail(self) -> str:
        """After ``parallel_sum`` has been seen: ``( view ) ;`` -> view name."""
        self.i += 1
        self.need("(")
        src = self.view_name()
        self.need(")")
        self.need(";")
        return src.text

    def at_gather(self) -> bool:
        return self.tok().text == "parallel_sum" and self.tok(1).kind == "("

    def st_return(self, in_kernel):
        head = self.need("NAME")
        if self.at_gather():
            # `return parallel_sum(v);` gathers into a fresh scalar first
            src = self.gather_tail()
            dst = N.fresh_name("_sum", set(self.fn_scope) | set(self.kernel_scope))
            self.fn_scope[dst] = "scalar"
            return [
                N.ParallelSum(dst, src, span=head.span),
                N.Return(N.ScalarVar(dst, span=head.span), span=head.span),
            ]
        val = self.value()
        self.need(";")
        return [N.Return(val, span=head.span)]

    def assign_op(self) -> str:
        for op in ("=", "+=", "-="):
            if self.take(op):
                return op
        raise ParseError("expected '=', '+=', or '-='", self.tok().span)

    def st_assign(self, in_kernel):
        nm = self.name()
        if self.tok().kind == "(":
            target = self.access(nm)
            op = self.assign_op()
            rhs = self.value()
            self.need(";")
            return [N.AssignView(target, op, rhs, span=nm.span)]
        op = self.assign_op()
        s = self.sym(nm.text)
        if op == "=" and self.at_gather():
            src = self.gather_tail()
            if s is None:
                self.fn_scope[nm.text] = "scalar"
            elif s != "scalar":
                raise ParseError(
                    f"parallel_sum destination '{nm.text}' is not a scalar", nm.span
                )
            return [N.ParallelSum(nm.text, src, span=nm.span)]
        if s is None:
            raise ParseError(f"unknown identifier '{nm.text}'", nm.span)
        if s != "scalar":
            raise ParseError(f"'{nm.text}' is not a scalar", nm.span)
        rhs = self.value()
        self.need(";")
        return [N.AssignScalar(nm.text, op, rhs, span=nm.span)]

    # -- expressions ----------------------------------------------------------

    def access(self, name_tok) -> N.ViewAccess:
        if not isinstance(self.sym(name_tok.text), tuple):
            raise ParseError(f"unknown view '{name_tok.text}'", name_tok.span)
        self.need("(")
        idx = [self.index()]
        while self.take(","):
            idx.append(self.index())
        self.need(")")
        return N.ViewAccess(name_tok.text, tuple(idx), span=name_tok.span)

    def extent(self) -> N.Extent:
        head = self.need("NAME")
        self.need("(")
        v = self.name("view")
        if not isinstance(self.sym(v.text), tuple):
            raise ParseError(f"unknown view '{v.text}' in extent", v.span)
        self.need(",")
        d = self.need("INT", "dimension")
        self.need(")")
        return N.Extent(v.text, int(d.text), span=head.span)

    def _enter(self, what):
        self.nest += 1
        if self.nest > MAX_NESTING:
            raise ParseError(f"{what} too deeply nested", self.tok().span)

    def value(self, level: int = 0):
        """Precedence climbing: level 0 = additive, 1 = multiplicative."""
        if level == 2:
            return self.value_atom()
        if level == 0:
            self._enter("expression")
        try:
            ops = _ADD if level == 0 else _MUL
            e = self.value(level + 1)
            while self.tok().kind in ops:
                op = self.tok()
                self.i += 1
                e = N.Binary(op.kind, e, self.value(level + 1), span=op.span)
            return e
        finally:
            if level == 0:
                self.nest -= 1

    def value_atom(self):
        t = self.tok()
        if t.kind in ("FLOAT", "INT"):
            self.i += 1
            return N.Literal(float(t.text), span=t.span)
        if t.kind == "-":
            self.i += 1
            inner = self.value_atom()
            if kind(inner) == "Literal":  # -<literal> folds
                return N.Literal(-inner.value, span=t.span)
            return N.Neg(inner, span=t.span)
        if t.kind == "(":
            self.i += 1
            e = self.value()
            self.need(")")
            return e
        if t.kind == "NAME":
            if t.text == "extent":
                return self.extent()
            nm = self.name()
            if self.tok().kind == "(":
                return self.access(nm)
            s = self.sym(nm.text)
            if s == "scalar":
                return N.ScalarVar(nm.text, span=nm.span)
            if s == "counter":
                return N.IndexVar(nm.text, span=nm.span)
            if isinstance(s, tuple):
                raise ParseError(f"view '{nm.text}' is read with indices", nm.span)
            raise ParseError(f"unknown identifier '{nm.text}'", nm.span)
        raise ParseError(f"expected an expression, found {t.text or 'end of input'!r}", t.span)

    def index(self, level: int = 0):
        if level == 2:
            return self.index_atom()
        if level == 0:
            self._enter("index expression")
        try:
            ops = _ADD if level == 0 else ("*",)
            e = self.index(level + 1)
            while self.tok().kind in ops:
                op = self.tok()
                self.i += 1
                e = N.IdxBinary(op.kind, e, self.index(level + 1), span=op.span)
            return e
        finally:
            if level == 0:
                self.nest -= 1

    def index_atom(self):
        t = self.tok()
        if t.kind == "INT":
            self.i += 1
            return N.IntLiteral(int(t.text), span=t.span)
        if t.kind == "-":
            self.i += 1
            inner = self.index_atom()
            if kind(inner) == "IntLiteral" and inner.span.start == t.span.end:
                return N.IntLiteral(-inner.value, span=t.span)
            return N.IdxBinary("*", N.IntLiteral(-1, span=t.span), inner, span=t.span)
        if t.kind == "(":
            self.i += 1
            e = self.index()
            self.need(")")
            return e
        if t.kind == "NAME":
            if t.text == "extent":
                return self.extent()
            nm = self.name()
            if self.tok().kind == "(":
                return self.access(nm)
            s = self.sym(nm.text)
            if s == "counter":
                return N.Counter(nm.text, span=nm.span)
            if s == "scalar":
                raise ParseError(
                    f"scalar '{nm.text}' is not allowed in an index expression", nm.span
                )
            if isinstance(s, tuple):
                raise ParseError(f"view '{nm.text}' is read with indices", nm.span)
            raise ParseError(f"unknown identifier '{nm.text}'", nm.span)
        if t.kind == "FLOAT":
            raise ParseError("index expressions are integral; no float literals", t.span)
        raise ParseError(
            f"expected an index expression, found {t.text or 'end of input'!r}", t.span
        )


def parse(text: str, *, check: bool = True) -> N.Program:
    """Text -> validated Program.  ParseError for syntax problems,
    ValidationError for well-formedness problems."""
    from .checks import validate

    try:
        program = _Reader(text).unit()
    except RecursionError:  # pathological nesting outside expressions
        raise ParseError("input too deeply nested") from None
    if check:
        diags = validate(program)
        if diags:
            raise ValidationError(diags)
    return program


# ---------------------------------------------------------------------------
# printer

_LEVEL = {"+": 1, "-": 1, "*": 2, "/": 2}


def _infix(e, env: int, is_right: bool, leaf) -> str:
    lvl = _LEVEL[e.op]
    s = f"{leaf(e.lhs, lvl, False)} {e.op} {leaf(e.rhs, lvl, True)}"
    return f"({s})" if lvl < env or (lvl == env and is_right) else s


def index_text(e, env: int = 0, is_right: bool = False) -> str:
    k = kind(e)
    if k == "IntLiteral":
        return str(e.value)
    if k == "Counter":
        return e.name
    if k == "Extent":
        return f"extent({e.view}, {e.dim})"
    if k == "ViewAccess":
        return f"{e.view}({', '.join(index_text(i) for i in e.indices)})"
    if k == "IdxBinary":
        return _infix(e, env, is_right, index_text)
    raise TypeError(f"cannot print index expression {k}")


def value_text(e, env: int = 0, is_right: bool = False) -> str:
    k = kind(e)
    if k == "Literal":
        return repr(e.value)
    if k in ("ScalarVar", "IndexVar"):
        return e.name
    if k == "ViewAccess":
        return index_text(e)
    if k == "Extent":
        return f"extent({e.view}, {e.dim})"
    if k == "Neg":
        return "-" + value_text(e.operand, 3)
    if k == "Binary":
        return _infix(e, env, is_right, value_text)
    raise TypeError(f"cannot print expression {k}")


def _src_text(src) -> str:
    return src if isinstance(src, str) else value_text(src)


def statement_lines(stmt, depth: int = 0) -> list:
    pad = "    " * depth
    k = kind(stmt)

    def nested(header):
        out = [pad + header + " {"]
        for s in stmt.body:
            out.extend(statement_lines(s, depth + 1))
        out.append(pad + "}")
        return out

    if k == "DeclView":
        if any(kind(x) == "StaticExtent" for x in stmt.descriptor.extents):
            raise ValueError(
                f"view '{stmt.name}' uses a static extent, which has no concrete syntax; "
                "use a dynamic extent argument"
            )
        dims = "".join(", " + index_text(a) for a in stmt.dyn_args)
        return [
            f'{pad}let {stmt.name}: view<f64,{stmt.descriptor.rank}> = view("{stmt.label}"{dims});'
        ]
    if k == "DeclScalar":
        return [f"{pad}let {stmt.name}: f64 = {value_text(stmt.init)};"]
    if k == "AssignView":
        return [f"{pad}{value_text(stmt.target)} {stmt.op} {value_text(stmt.rhs)};"]
    if k == "AssignScalar":
        return [f"{pad}{stmt.name} {stmt.op} {value_text(stmt.rhs)};"]
    if k == "If":
        c = stmt.cond
        return nested(f"if ({index_text(c.lhs)} {c.op} {index_text(c.rhs)})")
    if k == "ParallelFor":
        return nested(f"parallel_for {stmt.counter} in 0..{index_text(stmt.upper)}")
    if k == "DeepCopy":
        return [f"{pad}deep_copy({stmt.dst}, {_src_text(stmt.src)});"]
    if k == "ParallelSum":
        return [f"{pad}{stmt.dst} = parallel_sum({stmt.src});"]
    if k == "ParallelSumInto":
        return [f"{pad}parallel_sum({stmt.dst}, {_src_text(stmt.src)});"]
    if k == "AtomicAdd":
        return [f"{pad}atomic_add({value_text(stmt.target)}, {value_text(stmt.value)});"]
    if k == "Return":
        return [f"{pad}return {value_text(stmt.value)};"]
    raise TypeError(f"cannot print statement {k}")


def _function_text(fn) -> str:
    ps = ", ".join(
        f"{p.name}: view<f64,{p.type.rank}>" if p.is_view else f"{p.name}: f64" for p in fn.params
    )
    out = [f"fn {fn.name}({ps}){' -> f64' if fn.returns == 'f64' else ''} {{"]
    for s in fn.body:
        out.extend(statement_lines(s, 1))
    out += ["}", ""]
    return "\n".join(out)


def emit(program) -> str:
    """Canonical text of a Program (or one FunctionDef); '' when empty."""
    if kind(program) == "FunctionDef":
        return _function_text(program)
    return "\n".join(_function_text(f) for f in program.functions)
