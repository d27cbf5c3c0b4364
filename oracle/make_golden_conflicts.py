"""TEST INFRASTRUCTURE - golden conflict reports, produced by running the REFERENCE's
``detect_conflicts`` (imported from /root/reference/pkg/src, which exists only in the build
container).  While generating it asserts that ``oracle.interp.detect`` reproduces every report
record for record (kernel, view, offset, iterations, kinds).

    python -m oracle.make_golden_conflicts        # from the repo root

Writes tests/golden/conflicts.json: a list of cases {name, source, fn, inputs, rng_seed,
records}.  Cases:

* every corpus program and its generated gradient (all clean: the transform's atomics and the
  race analysis exist to guarantee that), reference tests test_runtime.py:204-209
* every corpus gradient with its atomic_adds rewritten into plain ``+=`` (the reference's
  ``strip_atomics`` test helper, test_runtime.py:273-300, done here on the program TEXT so no
  tree of one package is handed to the other), test_runtime.py:212-221
* the reference's own three unit programs (write-write, shared reads, atomic contention),
  test_runtime.py:224-268
* hand-written programs covering what those leave out: read/write and atomic/write mixes,
  rank-2 targets, indirect targets with repeated indices, guards, several kernels in one
  function (kernel numbering), a local View, a hot location touched by every iteration
"""

from __future__ import annotations

import glob
import json
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
PROGRAMS = os.path.join(ROOT, "paper_2507_13204_b200", "programs")
SIZES = (1, 2, 5, 64)


def strip_atomics_text(text: str) -> str:
    """``atomic_add(v(idx...), e);`` -> ``v(idx...) += e;`` on canonical program text."""
    out, pos = [], 0
    key = "atomic_add("
    while True:
        at = text.find(key, pos)
        if at < 0:
            out.append(text[pos:])
            return "".join(out)
        out.append(text[pos:at])
        k = at + len(key)
        start = k
        while text[k] != "(":  # view name
            k += 1
        depth = 0
        while True:  # balanced index list
            depth += text[k] == "("
            depth -= text[k] == ")"
            k += 1
            if depth == 0:
                break
        target = text[start:k]
        assert text[k] == ",", text[at:k + 10]
        k += 1
        depth, vstart = 0, k
        while not (text[k] == ")" and depth == 0):
            depth += text[k] == "("
            depth -= text[k] == ")"
            k += 1
        value = text[vstart:k].strip()
        assert text[k:k + 2] == ");", text[at:k + 10]
        out.append(f"{target} += {value};")
        pos = k + 2


EXTRA = {
    "ref_write_write": ("""
fn f(v: view<f64, 1>, acc: view<f64, 1>) -> f64 {
    parallel_for i in 0..extent(v, 0) {
        acc(0) = v(i);
    }
    return acc(0);
}
""", {"v": np.zeros(8), "acc": np.zeros(1)}),
    "ref_shared_reads": ("""
fn f(v: view<f64, 1>, out: view<f64, 1>) -> f64 {
    parallel_for i in 0..extent(v, 0) {
        out(i) = v(0);
    }
    return out(0);
}
""", {"v": np.array([5.0, 0.0]), "out": np.zeros(2)}),
    "ref_atomic_contention": ("""
fn f(v: view<f64, 1>, acc: view<f64, 1>) -> f64 {
    parallel_for i in 0..extent(v, 0) {
        atomic_add(acc(0), v(i));
    }
    return acc(0);
}
""", {"v": np.array([1.0, 2.0]), "acc": np.zeros(1)}),
    "read_write_neighbour": ("""
fn f(v: view<f64, 1>, out: view<f64, 1>) -> f64 {
    parallel_for i in 0..extent(v, 0) {
        if (i != extent(v, 0) - 1) {
            out(i) = v(i + 1);
        }
        v(i) = 2.0 * out(i);
    }
    return v(0);
}
""", {"v": np.arange(9.0), "out": np.zeros(9)}),
    "atomic_and_write": ("""
fn f(v: view<f64, 1>, acc: view<f64, 1>) -> f64 {
    parallel_for i in 0..extent(v, 0) {
        atomic_add(acc(1), v(i));
        if (i == 3) {
            acc(1) = 7.0;
        }
        if (i >= 5) {
            acc(2) += v(i);
        }
    }
    return acc(1);
}
""", {"v": np.arange(8.0), "acc": np.zeros(4)}),
    "rank2_columns": ("""
fn f(m: view<f64, 2>, r: view<f64, 1>) -> f64 {
    parallel_for i in 0..extent(m, 0) {
        m(i, 0) = r(i);
        if (i != 0) {
            m(i - 1, 1) = m(i, 2);
        }
        m(i, 1) += 1.0;
        m(0, 2) -= r(i);
    }
    return m(0, 0);
}
""", {"m": np.arange(18.0).reshape(6, 3), "r": np.ones(6)}),
    "indirect_scatter": ("""
fn f(v: view<f64, 1>, idx: view<f64, 1>, out: view<f64, 1>) -> f64 {
    parallel_for i in 0..extent(idx, 0) {
        out(idx(i)) = v(i);
    }
    parallel_for i in 0..extent(idx, 0) {
        out(idx(i)) += v(i);
        v(i) = out(i);
    }
    return out(0);
}
""", {"v": np.arange(12.0), "idx": np.array([0, 3, 3, 7, 1, 0, 0, 11, 5, 6, 7, 2], dtype=np.float64),
      "out": np.zeros(12)}),
    "local_view_and_kernel_numbers": ("""
fn f(v: view<f64, 1>) -> f64 {
    let t: view<f64, 1> = view("t", extent(v, 0));
    parallel_for i in 0..extent(v, 0) {
        t(i) = v(i);
    }
    parallel_for i in 0..extent(v, 0) {
        t(0) += v(i);
    }
    _s = parallel_sum(t);
    parallel_for i in 0..extent(v, 0) {
        if (i < 3) {
            v(2) = t(i);
        }
    }
    return _s;
}
""", {"v": np.arange(1.0, 7.0)}),
    "hot_location": ("""
fn f(v: view<f64, 1>, acc: view<f64, 1>) -> f64 {
    parallel_for i in 0..extent(v, 0) {
        let a: f64 = acc(0);
        acc(0) = a + v(i);
    }
    return acc(0);
}
""", {"v": np.ones(700), "acc": np.zeros(1)}),
}


def corpus_inputs(fn, n, rng):
    inputs = {}
    for p in fn.params:
        if not p.is_view:
            inputs[p.name] = float(rng.uniform(0.5, 1.5))
        elif p.name == "idx":
            inputs[p.name] = rng.integers(0, n, size=n).astype(np.float64)
        elif p.type.rank == 2:
            inputs[p.name] = rng.normal(size=(n, 3))
        else:
            inputs[p.name] = rng.normal(size=n)
    wrt = tuple(p.name for p in fn.params if p.is_view and p.name != "idx")
    return inputs, wrt


def main():
    sys.dont_write_bytecode = True
    sys.path.insert(0, REF_SRC)
    sys.path.insert(0, ROOT)
    import krn  # the reference
    from oracle import interp
    from paper_2507_13204_b200 import lang

    cases = []

    def add(name, source, fn_name, inputs, rng_seed=0):
        ref_in = {k: krn.ViewStorage.from_values(k, np.array(v)) if isinstance(v, np.ndarray) else v
                  for k, v in inputs.items()}
        cfg = krn.ExecutionConfig(rng_seed=rng_seed)
        report = krn.detect_conflicts(krn.parse(source), fn_name, ref_in, cfg)
        records = [[r.kernel, r.view, int(r.offset), [int(i) for i in r.iterations], list(r.kinds)]
                   for r in report.records]
        mine_in = {k: (np.array(v) if isinstance(v, np.ndarray) else v) for k, v in inputs.items()}
        mine = interp.detect(lang.parse(source), fn_name, mine_in, rng_seed=rng_seed)
        assert [[k, v, o, list(it), list(kd)] for k, v, o, it, kd in mine] == records, name
        for k, v in ref_in.items():  # the instrumented run executes the function as well
            if isinstance(v, krn.ViewStorage):
                assert np.array_equal(v.buffer, mine_in[k], equal_nan=True), (name, k)
        cases.append(dict(
            name=name, source=source, fn=fn_name, rng_seed=rng_seed,
            inputs={k: (dict(shape=list(v.shape), data=[float(x) for x in v.reshape(-1)])
                        if isinstance(v, np.ndarray) else float(v)) for k, v in inputs.items()},
            records=records))
        return records

    for path in sorted(glob.glob(os.path.join(PROGRAMS, "*.krn"))):
        stem = os.path.splitext(os.path.basename(path))[0]
        text = open(path).read()
        program = krn.parse(text)
        fn = program.functions[0]
        for n in SIZES:
            rng = np.random.default_rng(500 + n)
            inputs, wrt = corpus_inputs(fn, n, rng)
            assert add(f"{stem}/primal/n{n}", text, fn.name, inputs) == []
            gp = krn.differentiate(program, fn.name, wrt)
            gtext = krn.emit(gp)
            gfn = gp.functions[-1]
            ginputs = dict(inputs)
            for sp, primal in zip([p.name for p in gfn.params[len(fn.params):]], wrt):
                ginputs[sp] = np.zeros_like(np.asarray(inputs[primal]))
            assert add(f"{stem}/grad/n{n}", gtext, gfn.name, ginputs) == []
            stripped = strip_atomics_text(gtext)
            if stripped != gtext and n in (5, 64):
                got = add(f"{stem}/grad_stripped/n{n}", stripped, gfn.name, ginputs, rng_seed=n)
                print(f"{stem} stripped n={n}: {len(got)} records on {sorted({r[1] for r in got})}")
    for name, (source, inputs) in EXTRA.items():
        got = add(name, source, "f", inputs, rng_seed=3)
        print(f"{name}: {len(got)} records")
    with open(os.path.join(GOLDEN, "conflicts.json"), "w") as f:
        json.dump(cases, f, separators=(",", ":"))
    print(len(cases), "cases,", sum(len(c["records"]) for c in cases), "records,",
          os.path.getsize(os.path.join(GOLDEN, "conflicts.json")), "bytes")


if __name__ == "__main__":
    main()
