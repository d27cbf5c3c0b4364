"""Name-compatible alias of the reference's ``krn.parser``."""
from .lang.syntax import ParseError, ValidationError, parse  # noqa: F401
