"""Name-compatible alias of the reference's ``krn.ast`` (tree vocabulary)."""
from .lang.nodes import *  # noqa: F401,F403
from .lang.nodes import NO_SPAN, all_identifiers, desugar_function, desugar_statement, fresh_name, free_counters, lhs_as_expr, statement_exprs, walk_all_exprs, walk_expr, walk_statements  # noqa: F401
