"""Conflict detector (reference: detect_conflicts / _Tracer, runtime.py:198-227, 574-585,
709-726).  tests/golden/conflicts.json holds the reports of the REFERENCE itself
(oracle/make_golden_conflicts.py) for 105 cases: every corpus program and gradient (clean), the
gradients with their atomics stripped (reference tests test_runtime.py:204-221), the reference's
three unit programs (test_runtime.py:224-268) and hand-written mixes.

CPU tier: the oracle's restatement against the golden reports; the traced module of every case
compiles for sm_100a.  GPU tier: the device detector against the golden reports record for record,
against the oracle on fresh random index maps, and at a size only the device handles."""

import json
import os
import shutil
import subprocess

import numpy as np
import pytest

import paper_2507_13204_b200 as krn
from conftest import GOLDEN, ROOT
from oracle import interp

CASES = json.load(open(os.path.join(GOLDEN, "conflicts.json")))
IDS = [c["name"] for c in CASES]


def arrays(case):
    return {k: (np.array(v["data"], dtype=np.float64).reshape(v["shape"]) if isinstance(v, dict) else v)
            for k, v in case["inputs"].items()}


def as_lists(records):
    return [[r.kernel, r.view, r.offset, list(r.iterations), list(r.kinds)] for r in records]


@pytest.mark.parametrize("case", CASES, ids=IDS)
def test_oracle_matches_reference_reports(case):
    got = interp.detect(krn.parse(case["source"]), case["fn"], arrays(case), rng_seed=case["rng_seed"])
    assert [[k, v, o, list(it), list(kd)] for k, v, o, it, kd in got] == case["records"]


def test_golden_covers_the_reference_cases():
    by = {c["name"]: c for c in CASES}
    (ww,) = by["ref_write_write"]["records"]  # test_runtime.py:224-235
    assert ww[1:3] == ["acc", 0] and ww[3] == list(range(8)) and ww[4] == ["write"]
    assert by["ref_shared_reads"]["records"] == [] and by["ref_atomic_contention"]["records"] == []
    stripped = by["laplacian/grad_stripped/n64"]["records"]  # test_runtime.py:212-221
    assert {r[1] for r in stripped} == {"_d_x"} and all(len(set(r[3])) >= 2 for r in stripped)
    assert all(c["records"] == [] for n, c in by.items() if n.split("/")[1:2] in (["primal"], ["grad"]))
    kinds = {tuple(r[4]) for c in CASES for r in c["records"]}
    assert kinds == {("write",), ("read", "write"), ("atomic", "write")}


def test_traced_modules_compile_for_sm100a(tmp_path):
    """Every distinct traced module (dry replay kernels + the Trace prelude) through nvcc."""
    nvcc = shutil.which("nvcc")
    if nvcc is None:
        pytest.skip("nvcc not on PATH")
    from paper_2507_13204_b200.runtime import _plan_for

    seen = {}
    for case in CASES:
        if case["source"] in seen or not (case["name"].endswith("n64") or "/" not in case["name"]):
            continue
        plan = _plan_for(krn.parse(case["source"]).function(case["fn"]), trace=True)
        assert plan.source.count("Trace T") == sum(1 for s in plan.steps if s[0] == "kernel")
        seen[case["source"]] = plan.source
    # one translation unit per module would repeat the prelude 40 times: compile a sample of
    # structurally different ones (stencil guards, rank 2, indirect, locals)
    pick = [s for s in seen.values()][::6]
    for k, src in enumerate(pick):
        path = tmp_path / f"m{k}.cu"
        path.write_text(src)
        r = subprocess.run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "--fmad=false",
                            "-I", os.path.join(ROOT, "paper_2507_13204_b200", "csrc"), "-c", str(path),
                            "-o", str(tmp_path / f"m{k}.o")], capture_output=True, text=True)
        assert r.returncode == 0, r.stderr[-2000:]


# ---------------------------------------------------------------------------------------------
# GPU tier


def device_report(source, fn, inputs, **cfg):
    call = {k: (krn.ViewStorage.from_values(k, v) if isinstance(v, np.ndarray) else v) for k, v in inputs.items()}
    report = krn.detect_conflicts(krn.parse(source), fn, call, krn.ExecutionConfig(**cfg))
    return report, call


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=IDS)
def test_device_report_equals_reference(case):
    report, call = device_report(case["source"], case["fn"], arrays(case), rng_seed=case["rng_seed"])
    assert isinstance(report, krn.ConflictReport)
    assert as_lists(report.records) == case["records"]
    assert bool(report) == bool(case["records"])
    assert report.write_write() == report.records
    # the instrumented run executes the function as well: a clean function is schedule independent,
    # a kernel with conflicts runs in iteration order - either way the values of a plain sequential run
    want = arrays(case)
    interp.run(krn.parse(case["source"]), case["fn"], want)
    for k, v in call.items():
        if isinstance(v, krn.ViewStorage) and not case["name"].startswith("gather_indirect/grad"):
            assert np.array_equal(v.buffer, want[k], equal_nan=True), k


@pytest.mark.gpu
def test_execute_with_conflict_detect_returns_value_and_report():
    case = next(c for c in CASES if c["name"] == "ref_write_write")
    call = {k: krn.ViewStorage.from_values(k, v) for k, v in arrays(case).items()}
    res = krn.execute(krn.parse(case["source"]), "f", call, krn.ExecutionConfig(conflict_detect=True))
    assert res.value == 0.0 and as_lists(res.conflicts.records) == case["records"]
    clean = krn.execute(krn.load_program("laplacian"), "normRes1DLaplacianSQ",
                        {"x": np.ones(3), "b": np.zeros(3)}, krn.ExecutionConfig(conflict_detect=True))
    assert clean.value == 18.0 and not clean.conflicts and clean.conflicts.records == ()
    plain = krn.execute(krn.load_program("laplacian"), "normRes1DLaplacianSQ", {"x": np.ones(3), "b": np.zeros(3)})
    assert plain.conflicts is None


@pytest.mark.gpu
def test_out_of_bounds_surfaces_from_the_replay():
    src = "fn f(v: view<f64,1>) { parallel_for i in 0..extent(v,0) { v(i + 1) = v(i); } }"
    with pytest.raises(krn.OutOfBounds, match=r"line 1: v\(4\) outside extent 4"):
        krn.detect_conflicts(krn.parse(src), "f", {"v": np.zeros(4)})


INDIRECT = """
fn f(v: view<f64, 1>, idx: view<f64, 1>, out: view<f64, 2>) -> f64 {
    parallel_for i in 0..extent(idx, 0) {
        out(idx(i), 1) = v(i);
        atomic_add(out(idx(i), 0), v(i));
        if (i != 0) {
            out(idx(i - 1), 2) += out(idx(i), 0);
        }
    }
    return out(0, 0);
}
"""


@pytest.mark.gpu
@pytest.mark.parametrize("n,rows,seed", [(1, 1, 0), (2, 1, 1), (50, 7, 2), (300, 300, 3), (2000, 40, 4), (5000, 100000, 5)])
def test_random_index_maps_against_oracle(n, rows, seed):
    rng = np.random.default_rng(seed)
    inputs = {"v": rng.normal(size=n), "idx": rng.integers(0, rows, size=n).astype(np.float64),
              "out": np.zeros((rows, 3))}
    want = interp.detect(krn.parse(INDIRECT), "f", {k: v.copy() for k, v in inputs.items()}, rng_seed=seed)
    report, _ = device_report(INDIRECT, "f", inputs, rng_seed=seed)
    assert as_lists(report.records) == [[k, v, o, list(it), list(kd)] for k, v, o, it, kd in want]


@pytest.mark.gpu
def test_more_triples_than_the_first_buffer_holds():
    """Every one of n iterations touches acc(0): one record listing all of them; the first
    collect pass overflows its buffer and is repeated with the exact size."""
    from paper_2507_13204_b200.runtime import _Run

    case = next(c for c in CASES if c["name"] == "hot_location")
    n = 3 * _Run.TRIPLES_FIRST // 2 // 2 + 11  # two accesses per iteration
    report, call = device_report(case["source"], "f", {"v": np.ones(n), "acc": np.zeros(1)})
    (rec,) = report.records
    assert (rec.kernel, rec.view, rec.offset, rec.kinds) == (0, "acc", 0, ("read", "write"))
    assert rec.iterations == tuple(range(n))


@pytest.mark.gpu
def test_large_stripped_gradient():
    """Headline gradient with atomics stripped at 2^18 rows: every row of _d_x is a conflict
    (iterations j-1, j, j+1), found in a few launches."""
    case = next(c for c in CASES if c["name"] == "laplacian/grad_stripped/n64")
    n = 1 << 18
    rng = np.random.default_rng(0)
    report, _ = device_report(case["source"], case["fn"], {
        "x": rng.normal(size=n), "b": rng.normal(size=n), "_d_x": np.zeros(n), "_d_b": np.zeros(n)})
    recs = report.records
    assert len(recs) == n and {r.view for r in recs} == {"_d_x"} and len({r.kernel for r in recs}) == 1
    assert recs[0].iterations == (0, 1) and recs[-1].iterations == (n - 2, n - 1)
    k = n // 3
    assert recs[k].offset == k and recs[k].iterations == (k - 1, k, k + 1)
