"""Name-compatible alias of the reference's ``krn.adjoint``."""
from .lang.reverse import *  # noqa: F401,F403
from .lang.reverse import GradientPlan, differentiate, reverse_deep_copy, reverse_parallel_for, reverse_parallel_sum, reverse_statement  # noqa: F401
