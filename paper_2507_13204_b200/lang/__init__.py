"""Front-end of the kernel language: tree vocabulary, concrete syntax,
well-formedness checks, the analyses and the reverse-mode transform.  Pure
Python and value-free - nothing here touches array data; the data path is
``paper_2507_13204_b200.runtime`` (CUDA)."""

from .checks import RESERVED, Diagnostic, validate
from .dataflow import (
    ActivityResult,
    RaceFlag,
    RaceResult,
    TapingVerdict,
    TapingViolation,
    UnknownParameter,
    activity,
    normalize_index,
    race_analysis,
    taping_feasibility,
)
from .derivative import NonDifferentiableOp, contributions
from .reverse import GradientPlan, InactiveReturn, NotFeasible, UnknownFunction, differentiate
from .syntax import ParseError, ValidationError, emit, parse
