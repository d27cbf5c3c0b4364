"""Name-compatible alias of the reference's ``krn.printer`` (the private helpers its own tests
reach for included: ``_statement(stmt, depth) -> lines``, printer.py:71)."""
from .lang.syntax import emit, index_text as _index, statement_lines as _statement, value_text as _expr  # noqa: F401
