"""TEST INFRASTRUCTURE - generates tests/golden/ by running the REFERENCE
ITSELF (imported from /root/reference/pkg/src, which exists only in the build
container), and at the same time pins the two oracle restatements
(oracle/interp.py, oracle/krn_oracle.c) against it bit for bit.

    python -m oracle.make_golden          # from the repo root

Fixtures written (all small):

  tests/golden/grad_text/<program>.krn     emitted <fn>_grad for every corpus program
  tests/golden/corpus.npz                  every corpus program at n in SIZES: inputs,
                                           primal value + mutated params, gradient shadows
                                           + mutated params (reference execute, threads=1,
                                           deterministic reduction)
  tests/golden/laplacian.npz               headline objective: bench inputs (default_rng(0)
                                           uniform, verify.py:272-280) at n=1000 and 10000,
                                           acceptance-C2 style normal draws (rng 42), seed
                                           scaling, double-run accumulation
  tests/golden/pairwise.npz                pairwise_sum over assorted lengths incl. 2^k±1

  paper_2507_13204_b200/programs/*.krn     the corpus programs = the workload definition
                                           (SURVEY section 8a), re-printed canonically
"""

from __future__ import annotations

import glob
import os
import sys
import warnings

import numpy as np

REF_SRC = "/root/reference/pkg/src"
REF_PROGRAMS = "/root/reference/pkg/programs"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
SIZES = (1, 2, 3, 17, 257)


def corpus_inputs(fn, n, rng):
    """Same recipe as the reference's acceptance tests (test_acceptance.py:44-60):
    unit-scale views, integer-valued index view, rank-2 views are (n, 3)."""
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
    from oracle import cport, interp
    from paper_2507_13204_b200 import lang

    os.makedirs(os.path.join(GOLDEN, "grad_text"), exist_ok=True)
    cfg = krn.ExecutionConfig(threads=1, deterministic_reduction=True)

    def ref_call(program, fn_name, arrays):
        call = {
            k: krn.ViewStorage.from_values(k, v) if isinstance(v, np.ndarray) else v
            for k, v in arrays.items()
        }
        value = krn.execute(program, fn_name, call, cfg).value
        return value, {k: v.buffer for k, v in call.items() if isinstance(v, krn.ViewStorage)}

    def fresh(d):
        return {k: (np.array(v) if isinstance(v, np.ndarray) else v) for k, v in d.items()}

    def same_bits(a, b):
        # bit equality; NaNs compare equal to each other (sign/payload of a NaN
        # is not part of the contract and differs between x86 libm paths and GPUs)
        a, b = np.array(a, dtype=np.float64, ndmin=1), np.array(b, dtype=np.float64, ndmin=1)
        if a.shape != b.shape:
            return False
        na, nb = np.isnan(a), np.isnan(b)
        return bool(np.array_equal(na, nb) and np.array_equal(
            a[~na].view(np.uint64), b[~nb].view(np.uint64)))

    # ---- corpus -----------------------------------------------------------
    corpus = {}
    for path in sorted(glob.glob(os.path.join(REF_PROGRAMS, "*.krn"))):
        stem = os.path.splitext(os.path.basename(path))[0]
        text = open(path).read()
        program = krn.parse(text)
        fn = program.functions[0]
        mine = lang.parse(text)
        # ship the workload definition in canonical printed form (comments dropped)
        with open(os.path.join(ROOT, "paper_2507_13204_b200", "programs", stem + ".krn"), "w") as f:
            f.write(f"// corpus program '{stem}' (benchmark kernel, SURVEY.md section 8a), canonical form\n")
            f.write(krn.emit(program))
        for n in SIZES:
            rng = np.random.default_rng(1000 + n)
            inputs, wrt = corpus_inputs(fn, n, rng)
            gp = krn.differentiate(program, fn.name, wrt)
            if n == SIZES[0]:
                with open(os.path.join(GOLDEN, "grad_text", stem + ".krn"), "w") as f:
                    f.write(krn.emit(gp.functions[-1]))
            key = f"{stem}/n{n}"
            for k, v in inputs.items():
                corpus[f"{key}/in/{k}"] = np.asarray(v, dtype=np.float64)
            corpus[f"{key}/wrt"] = np.array(",".join(wrt))
            # primal
            value, after = ref_call(program, fn.name, fresh(inputs))
            corpus[f"{key}/primal/value"] = np.float64(value)
            for k, v in after.items():
                corpus[f"{key}/primal/after/{k}"] = v
            # pin oracle/interp.py on the primal
            mine_in = fresh(inputs)
            mv = interp.run(mine, fn.name, mine_in)
            assert same_bits(mv, value), (key, mv, value)
            for k, v in after.items():
                assert same_bits(mine_in[k], v), (key, k)
            # gradient: zero shadows, then a second run into non-zero shadows
            gfn = gp.functions[-1]
            shadow_names = [p.name for p in gfn.params[len(fn.params):]]
            garr = fresh(inputs)
            for sp, primal in zip(shadow_names, wrt):
                garr[sp] = np.zeros_like(np.asarray(inputs[primal], dtype=np.float64))
            _, gafter = ref_call(gp, gfn.name, garr)
            for k, v in gafter.items():
                corpus[f"{key}/grad/after/{k}"] = v
            mg = lang.differentiate(mine, fn.name, wrt)
            mine_g = fresh(inputs)
            for sp, primal in zip(shadow_names, wrt):
                mine_g[sp] = np.zeros_like(np.asarray(inputs[primal], dtype=np.float64))
            interp.run(mg, gfn.name, mine_g)
            for k, v in gafter.items():
                assert same_bits(mine_g[k], v), (key, "grad", k)
        print("corpus", stem, "ok")
    np.savez_compressed(os.path.join(GOLDEN, "corpus.npz"), **corpus)

    # ---- headline ---------------------------------------------------------
    lap_text = open(os.path.join(REF_PROGRAMS, "laplacian.krn")).read()
    lap = krn.parse(lap_text)
    FN = "normRes1DLaplacianSQ"
    out = {}

    def lap_case(tag, x, b, seed=1.0, dx0=None, db0=None, store_inputs=True):
        gp = krn.differentiate(lap, FN, ("x", "b"), seed_value=seed)
        n = x.size
        value, after = ref_call(lap, FN, {"x": x.copy(), "b": b.copy()})
        dx = np.zeros(n) if dx0 is None else dx0.copy()
        db = np.zeros(n) if db0 is None else db0.copy()
        _, gafter = ref_call(gp, FN + "_grad", {"x": x.copy(), "b": b.copy(), "_d_x": dx, "_d_b": db})
        if store_inputs:
            out[f"{tag}/x"], out[f"{tag}/b"] = x, b
        if dx0 is not None:
            out[f"{tag}/dx0"], out[f"{tag}/db0"] = dx0, db0
        out[f"{tag}/seed"] = np.float64(seed)
        out[f"{tag}/f"] = np.float64(value)
        out[f"{tag}/x_after"] = after["x"]
        out[f"{tag}/dx"], out[f"{tag}/db"] = gafter["_d_x"], gafter["_d_b"]
        assert same_bits(gafter["x"], after["x"])
        # pin the C restatement
        xc = x.copy()
        fc = cport.laplacian_primal(xc, b.copy())
        assert same_bits(fc, value) and same_bits(xc, after["x"]), tag
        xg, dxc = x.copy(), (np.zeros(n) if dx0 is None else dx0.copy())
        dbc = np.zeros(n) if db0 is None else db0.copy()
        cport.laplacian_grad(xg, b.copy(), dxc, dbc, seed)
        assert same_bits(dxc, gafter["_d_x"]) and same_bits(dbc, gafter["_d_b"]), tag
        assert same_bits(xg, after["x"]), tag
        # analytic oracle agreement (reference criterion 2: rtol 1e-12, atol 0)
        f, gx, gb = krn.laplacian_oracle(x, b)
        if dx0 is None and seed == 1.0 and np.isfinite(x).all() and np.isfinite(b).all() and np.abs(x).max() < 1e100:
            assert np.all(np.abs(gafter["_d_x"] - gx) <= 1e-12 * np.abs(gx)), tag
            assert np.all(np.abs(gafter["_d_b"] - gb) <= 1e-12 * np.abs(gb)), tag
        return value, gafter

    for n in (1000, 10000):  # bench_ratio's inputs (verify.py:272-280)
        rng = np.random.default_rng(0)
        x = rng.uniform(-1.0, 1.0, n)
        b = rng.uniform(-1.0, 1.0, n)
        lap_case(f"bench_n{n}", x, b, store_inputs=(n == 1000))
        out[f"bench_n{n}/input_checksum"] = np.float64(float(np.sum(x) + 2.0 * np.sum(b)))
    rng = np.random.default_rng(42)  # acceptance criterion 2 style draws
    for n in (1, 2, 3, 17, 1000):
        for draw in range(2):
            lap_case(f"c2_n{n}_d{draw}", rng.normal(size=n), rng.normal(size=n))
    rng = np.random.default_rng(7)
    x, b = rng.normal(size=64), rng.normal(size=64)
    for c in (0.5, 2.0, -1.0):  # seed linearity (criterion 8)
        lap_case(f"seed_{c}", x, b, seed=c)
    first = lap_case("acc_first", x, b)[1]
    lap_case("acc_second", x, b, dx0=first["_d_x"], db0=first["_d_b"])  # run into non-zero shadows
    # non-finite / signed-zero propagation through the cancelling statements
    xs = np.zeros(24)
    bs = np.zeros(24)
    xs[1], xs[2], xs[3] = -0.0, 0.0, -0.0
    bs[2], bs[3] = -0.0, 0.0
    xs[8] = np.inf          # inf - inf -> NaN in the cancelling statements, locally
    xs[14] = 1e308          # 3x overflows to inf
    bs[19] = np.nan
    xs[22], bs[22] = 5e-324, -5e-324   # subnormals
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        lap_case("special", xs, bs)
    np.savez_compressed(os.path.join(GOLDEN, "laplacian.npz"), **out)
    print("laplacian ok")

    # ---- pairwise tree ------------------------------------------------------
    pw = {}
    lengths = sorted(set(list(range(0, 70)) + [127, 128, 129, 255, 256, 257, 1000, 1023, 1024, 1025,
                                               2047, 2048, 2049, 4097, 65535, 65536, 65537,
                                               (1 << 20) + 5]))
    vals = []
    for n in lengths:
        v = np.random.default_rng(n).normal(size=n) * 10.0 ** np.random.default_rng(n + 1).integers(-3, 4, size=n)
        r = krn.runtime.pairwise_sum(v)
        assert same_bits(r, cport.pairwise_sum(v)) and same_bits(r, interp.pairwise_sum(v)), n
        vals.append(r)
    pw["lengths"] = np.array(lengths, dtype=np.int64)
    pw["sums"] = np.array(vals, dtype=np.float64)
    # signed zeros: all -0.0 input keeps -0.0 only when no level is padded
    for n in (1, 2, 3, 4, 5, 8, 12, 16):
        v = np.full(n, -0.0)
        r = krn.runtime.pairwise_sum(v)
        assert same_bits(r, cport.pairwise_sum(v)), n
        pw[f"negzero_{n}"] = np.float64(r)
    np.savez_compressed(os.path.join(GOLDEN, "pairwise.npz"), **pw)
    print("pairwise ok")
    for f in sorted(glob.glob(os.path.join(GOLDEN, "*.npz"))):
        print(os.path.basename(f), os.path.getsize(f) // 1024, "KiB")


if __name__ == "__main__":
    main()
