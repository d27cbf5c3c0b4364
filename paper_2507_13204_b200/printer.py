"""Name-compatible alias of the reference's ``krn.printer``."""
from .lang.syntax import emit, index_text as _index, value_text as _expr  # noqa: F401
