"""krn on B200: the reference package's API (``krn``) with the data path on
the GPU.

The names below are the reference's flat export list
(/root/reference/pkg/src/krn/__init__.py:9-96).  Front-end functions
(``parse``, ``emit``, ``differentiate``, the analyses) are value-free Python;
``execute`` and everything built on it (``ad_gradient``, ``bench_ratio``,
``finite_difference_gradient``) run CUDA kernels through libkrn_b200.so and
fail loudly when the library or a device is missing - there is no CPU
execution path in this package.
"""

from .lang import (
    ActivityResult,
    GradientPlan,
    InactiveReturn,
    NonDifferentiableOp,
    NotFeasible,
    ParseError,
    RaceFlag,
    RaceResult,
    TapingVerdict,
    TapingViolation,
    UnknownFunction,
    UnknownParameter,
    ValidationError,
    activity,
    differentiate,
    emit,
    parse,
    race_analysis,
    taping_feasibility,
    validate,
)
from .runtime import (
    ConflictRecord,
    ConflictReport,
    Device,
    ExecResult,
    ExecutionConfig,
    NonFiniteDetected,
    OutOfBounds,
    ShapeMismatch,
    ViewStorage,
    detect_conflicts,
    execute,
    load_tensor,
    pairwise_sum,
    save_tensor,
)
from .verify import (
    BenchResult,
    GradientReport,
    ad_gradient,
    bench_ratio,
    check_gradient,
    finite_difference_gradient,
    laplacian_oracle,
)

from .shard_program import NotShardable, ShardedProgram  # noqa: E402  (multi-GPU, beyond the reference)

__version__ = "0.1.0"

import os as _os

PROGRAMS_DIR = _os.path.join(_os.path.dirname(_os.path.abspath(__file__)), "programs")


def load_program(stem: str):
    """Parse one of the shipped programs: the reference's corpus (``programs/<stem>.krn``) or
    an additional one (``extra_programs/<stem>.krn``, see the README there)."""
    path = _os.path.join(PROGRAMS_DIR, stem + ".krn")
    if not _os.path.exists(path):
        path = _os.path.join(_os.path.dirname(PROGRAMS_DIR), "extra_programs", stem + ".krn")
    with open(path, encoding="utf-8") as f:
        return parse(f.read())
