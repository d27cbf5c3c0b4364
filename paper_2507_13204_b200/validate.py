"""Name-compatible alias of the reference's ``krn.validate``."""
from .lang.checks import Diagnostic, validate  # noqa: F401
