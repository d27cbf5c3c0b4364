"""Name-compatible alias of the reference's ``krn.analysis``."""
from .lang.dataflow import *  # noqa: F401,F403
from .lang.dataflow import normalize_index  # noqa: F401
