"""TEST INFRASTRUCTURE - golden vectors for the programs in
paper_2507_13204_b200/extra_programs/ (not part of the reference's corpus), produced by
running the REFERENCE ITSELF on them (imported from /root/reference/pkg/src, which exists
only in the build container).  While generating it asserts that oracle/interp.py and this
repository's front-end (emitted gradient text) agree with the reference bit for bit / byte
for byte.

    python -m oracle.make_golden_extra        # from the repo root

Writes tests/golden/extra.npz (inputs, primal value + mutated parameters, gradient shadows +
mutated parameters where the reference's transform accepts the program, at n in SIZES) and
tests/golden/grad_text_extra/<program>.krn.
"""

from __future__ import annotations

import glob
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
EXTRA = os.path.join(ROOT, "paper_2507_13204_b200", "extra_programs")
SIZES = (1, 2, 5, 130, 1030)


def inputs_for(fn, n, rows, rng):
    """Views of n rows (rank-2: n x 3), except that a View indexed indirectly has `rows` rows
    and the index View holds integers in [0, rows)."""
    out = {}
    for p in fn.params:
        if not p.is_view:
            out[p.name] = float(rng.uniform(0.5, 1.5))
        elif p.name == "idx":
            out[p.name] = rng.integers(0, rows, size=n).astype(np.float64)
        elif p.name == "q" and any(q.name == "idx" for q in fn.params):
            out[p.name] = rng.normal(size=(rows, 3))
        elif p.name == "fine":
            out[p.name] = rng.normal(size=2 * n + 1)  # read at 2*i - 1 .. 2*i + 1 for i < n
        elif p.type.rank == 2:
            out[p.name] = rng.normal(size=(n, 3))
        else:
            out[p.name] = rng.normal(size=n)
    return out


def main():
    sys.dont_write_bytecode = True
    sys.path.insert(0, REF_SRC)
    sys.path.insert(0, ROOT)
    import krn  # the reference
    from oracle import interp
    from paper_2507_13204_b200 import lang

    def same_bits(a, b):
        # bit equality; all NaNs compare equal (sign/payload is not part of the contract)
        a, b = np.array(a, dtype=np.float64, ndmin=1), np.array(b, dtype=np.float64, ndmin=1)
        if a.shape != b.shape:
            return False
        na, nb = np.isnan(a), np.isnan(b)
        return bool(np.array_equal(na, nb) and np.array_equal(a[~na].view(np.uint64), b[~nb].view(np.uint64)))

    os.makedirs(os.path.join(GOLDEN, "grad_text_extra"), exist_ok=True)
    cfg = krn.ExecutionConfig(threads=1, deterministic_reduction=True)

    def ref_call(program, fn_name, arrays):
        call = {k: krn.ViewStorage.from_values(k, v) if isinstance(v, np.ndarray) else v for k, v in arrays.items()}
        value = krn.execute(program, fn_name, call, cfg).value
        return value, {k: v.buffer for k, v in call.items() if isinstance(v, krn.ViewStorage)}

    def fresh(d):
        return {k: (np.array(v) if isinstance(v, np.ndarray) else v) for k, v in d.items()}

    out = {}
    for path in sorted(glob.glob(os.path.join(EXTRA, "*.krn"))):
        stem = os.path.splitext(os.path.basename(path))[0]
        text = open(path).read()
        program, mine = krn.parse(text), lang.parse(text)
        fn = program.functions[0]
        wrt = tuple(p.name for p in fn.params if p.is_view and p.name != "idx")
        try:
            gp = krn.differentiate(program, fn.name, wrt)
        except (krn.NotFeasible, ValueError):
            gp = None  # overwrites a value its own reversal needs / returns nothing: primal only
        if gp is not None:
            ref_text = krn.emit(gp.functions[-1])
            assert lang.emit(lang.differentiate(mine, fn.name, wrt).functions[-1]) == ref_text, stem
            with open(os.path.join(GOLDEN, "grad_text_extra", stem + ".krn"), "w") as f:
                f.write(ref_text)
        out[f"{stem}/wrt"] = np.array(",".join(wrt))
        out[f"{stem}/has_grad"] = np.array(gp is not None)
        for n in SIZES:
            rows = max(1, (2 * n) // 3)  # fewer target rows than iterations: collisions guaranteed
            rng = np.random.default_rng(77 + n)
            inputs = inputs_for(fn, n, rows, rng)
            key = f"{stem}/n{n}"
            for k, v in inputs.items():
                out[f"{key}/in/{k}"] = np.asarray(v, dtype=np.float64)
            value, after = ref_call(program, fn.name, fresh(inputs))
            out[f"{key}/primal/value"] = np.float64(np.nan if value is None else value)
            for k, v in after.items():
                out[f"{key}/primal/after/{k}"] = v
            mine_in = fresh(inputs)
            mv = interp.run(mine, fn.name, mine_in)
            assert (value is None and mv is None) or same_bits(mv, value), (key, mv, value)
            for k, v in after.items():
                assert same_bits(mine_in[k], v), (key, k)
            if gp is None:
                continue
            gfn = gp.functions[-1]
            shadows = [p.name for p in gfn.params[len(fn.params):]]
            garr, marr = fresh(inputs), fresh(inputs)
            for sp, primal in zip(shadows, wrt):
                # pre-filled shadows: the gradient ACCUMULATES (verify.py:165-173)
                init = rng.normal(size=np.shape(inputs[primal]))
                out[f"{key}/grad/in/{sp}"] = init
                garr[sp], marr[sp] = init.copy(), init.copy()
            _, gafter = ref_call(gp, gfn.name, garr)
            for k, v in gafter.items():
                out[f"{key}/grad/after/{k}"] = v
            interp.run(lang.differentiate(mine, fn.name, wrt), gfn.name, marr)
            for k, v in gafter.items():
                assert same_bits(marr[k], v), (key, "grad", k)
        print("extra", stem, "ok", "(gradient)" if gp is not None else "(primal only)")
    np.savez_compressed(os.path.join(GOLDEN, "extra.npz"), **out)
    print("wrote", os.path.join(GOLDEN, "extra.npz"), f"{len(out)} arrays")


if __name__ == "__main__":
    main()
