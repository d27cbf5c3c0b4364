"""Differential run against the REFERENCE ITSELF (build container only: imports /root/reference/pkg/src
as `krn`; nothing under tests/, bench.py or the package imports this file).  Random well-formed programs
(the generator of tests/test_gpu_random_programs.py) through both frontends: printed program text,
generated gradient text for three wrt sets (or the same exception class and message), race-analysis
flags - all must be identical.

    python oracle/diff_frontend_vs_reference.py <seed> <programs>

Round 2: 8 seeds x 1500 programs, 36 000 differentiate calls, no difference."""
import sys, warnings, os
_ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, _ROOT); sys.path.insert(0, os.path.join(_ROOT, "tests")); sys.path.insert(0, "/root/reference/pkg/src")
import krn as ref
import paper_2507_13204_b200 as mine
from hypothesis import given, settings, HealthCheck, strategies as st, seed
from test_gpu_random_programs import programs
import numpy as np
stats = {"n": 0, "grad": 0, "infeasible": 0}
def both(f_ref, f_mine):
    try:
        a = ("ok", f_ref())
    except Exception as e:
        a = ("err", type(e).__name__, str(e))
    try:
        b = ("ok", f_mine())
    except Exception as e:
        b = ("err", type(e).__name__, str(e))
    return a, b
@seed(int(sys.argv[1]))
@settings(max_examples=int(sys.argv[2]), deadline=None, suppress_health_check=list(HealthCheck), database=None)
@given(programs())
def run(prog):
    text, use_idx, use_c, use_m = prog
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        a, b = both(lambda: ref.emit(ref.parse(text)),
                    lambda: mine.emit(mine.parse(text)))
        assert a == b, ("print", text, a, b)
        if a[0] != "ok":
            return
        stats["n"] += 1
        wrt = ("a", "b") + (("m",) if use_m else ())
        for w in (wrt, ("a",), ("b",)):
            a, b = both(lambda: ref.emit(ref.differentiate(ref.parse(text), "f", w)),
                        lambda: mine.emit(mine.differentiate(mine.parse(text), "f", w)))
            assert a == b, ("grad", w, text, a, b)
            stats["grad" if a[0] == "ok" else "infeasible"] += 1
        a, b = both(lambda: [(type(f).__name__, str(f)) for f in ref.race_analysis(ref.parse(text).functions[0]).flags],
                    lambda: [(type(f).__name__, str(f)) for f in mine.race_analysis(mine.parse(text).functions[0]).flags])
        assert a == b, ("race", text, a, b)
run()
print(stats)
