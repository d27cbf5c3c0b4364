"""Name-compatible alias of the reference's ``krn.partials``."""
from .lang.derivative import NonDifferentiableOp, contributions, needed_primal_names  # noqa: F401
