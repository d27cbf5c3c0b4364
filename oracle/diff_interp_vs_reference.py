"""Differential run of the oracle interpreter (oracle/interp.py) against the REFERENCE ITSELF (build
container only: imports /root/reference/pkg/src as `krn`; test infrastructure, nothing under the package
imports this file).  Random well-formed programs and their generated gradients, n = 1 ... 130, the
reference with threads = 1 and 3, check_finite on and off: returned value and every View bit-identical,
or the same exception class and message.

    python oracle/diff_interp_vs_reference.py <seed> <programs>

Round 2: 8 seeds x 800 programs (6 400 primal + 5 739 gradient executions), no difference."""
import sys, warnings, os
_ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, _ROOT); sys.path.insert(0, os.path.join(_ROOT, "tests")); sys.path.insert(0, "/root/reference/pkg/src")
import krn as ref
import paper_2507_13204_b200 as mine
from oracle import interp
from hypothesis import given, settings, HealthCheck, strategies as st, seed
from test_gpu_random_programs import programs, _inputs
import numpy as np
stats = {"n": 0, "grad": 0, "err": 0}
def run_ref(program, name, arrays, check, threads):
    cfg = ref.ExecutionConfig(threads=threads, deterministic_reduction=True, check_finite=check)
    call = {k: ref.ViewStorage.from_values(k, v) if isinstance(v, np.ndarray) else v for k, v in arrays.items()}
    try:
        with np.errstate(all="ignore"):
            value = ref.execute(program, name, call, cfg).value
        return ("ok", value, {k: v.buffer.copy() for k, v in call.items() if isinstance(v, ref.ViewStorage)})
    except Exception as e:
        return ("err", type(e).__name__, str(e))
def run_mine(program, name, arrays, check):
    call = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in arrays.items()}
    try:
        with np.errstate(all="ignore"):
            value = interp.run(program, name, call, check_finite=check) if check else interp.run(program, name, call)
        return ("ok", value, {k: v for k, v in call.items() if isinstance(v, np.ndarray)})
    except Exception as e:
        return ("err", type(e).__name__, str(e))
def same(a, b, what):
    assert a[0] == b[0], (what, a[:2] if a[0]=="err" else a[0], b[:2] if b[0]=="err" else b[0])
    if a[0] == "err":
        assert a == b, (what, a, b); stats["err"] += 1; return
    av, bv = a[1], b[1]
    assert (av is None) == (bv is None) and (av is None or np.float64(av).tobytes() == np.float64(bv).tobytes()), (what, av, bv)
    for k in a[2]:
        assert a[2][k].tobytes() == np.asarray(b[2][k]).tobytes(), (what, k)
@seed(int(sys.argv[1]))
@settings(max_examples=int(sys.argv[2]), deadline=None, suppress_health_check=list(HealthCheck), database=None)
@given(programs(), st.sampled_from([1, 2, 5, 33, 130]), st.integers(0, 10**6), st.booleans(), st.sampled_from([1, 3]))
def run(prog, n, sd, check, threads):
    text, use_idx, use_c, use_m = prog
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        try:
            rp = ref.parse(text); mp = mine.parse(text)
        except Exception:
            return
        inputs = _inputs(n, use_idx, use_c, sd, use_m)
        same(run_ref(rp, "f", inputs, check, threads), run_mine(mp, "f", inputs, check), ("primal", text, n, sd, check))
        stats["n"] += 1
        wrt = ("a", "b") + (("m",) if use_m else ())
        try:
            rg = ref.differentiate(rp, "f", wrt); mg = mine.differentiate(mp, "f", wrt)
        except Exception:
            return
        gname = rg.functions[-1].name
        g = dict(inputs)
        rng = np.random.default_rng(sd)
        for p in rg.functions[-1].params[len(rp.functions[0].params):]:
            g[p.name] = rng.normal(size=np.shape(inputs[p.name[3:]]))
        same(run_ref(rg, gname, g, check, threads), run_mine(mg, gname, g, check), ("grad", text, n, sd, check))
        stats["grad"] += 1
run()
print(stats)
