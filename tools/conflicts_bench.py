"""Conflict detector timings: device `detect_conflicts` on the headline gradient (clean) and on
the same gradient with its atomics stripped (every row of _d_x a conflict), next to the CPU
oracle's dictionary log (oracle/interp.detect, the reference's algorithm) at a size it finishes.

    python tools/conflicts_bench.py [--rows 262144 4194304] > gpurun_out/conflicts_bench.md
"""

import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2507_13204_b200 as krn  # noqa: E402
from oracle import interp  # noqa: E402  (the CPU column only)
from oracle.make_golden_conflicts import strip_atomics_text  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, nargs="*", default=[1 << 14, 1 << 18, 1 << 22])
    ap.add_argument("--cpu-rows", type=int, default=1 << 14)
    args = ap.parse_args()
    lap = krn.load_program("laplacian")
    fn = "normRes1DLaplacianSQ"
    gp = krn.differentiate(lap, fn, ("x", "b"))
    text = krn.emit(gp)
    stripped = krn.parse(strip_atomics_text(text))
    print("| rows | program | device s | records | plain statements run s | CPU oracle s |")
    print("|---|---|---|---|---|---|")
    for n in args.rows:
        rng = np.random.default_rng(0)
        x, b = rng.normal(size=n), rng.normal(size=n)
        for tag, prog in (("gradient (clean)", gp), ("gradient, atomics stripped", stripped)):
            def call():
                return {"x": krn.ViewStorage.from_values("x", x), "b": krn.ViewStorage.from_values("b", b),
                        "_d_x": krn.ViewStorage.zeros("_d_x", (n,)), "_d_b": krn.ViewStorage.zeros("_d_b", (n,))}
            krn.detect_conflicts(prog, fn + "_grad", call())  # compile + warm
            inputs = call()
            t0 = time.perf_counter()
            rep = krn.detect_conflicts(prog, fn + "_grad", inputs)
            t1 = time.perf_counter()
            inputs = call()
            krn.execute(prog, fn + "_grad", inputs, krn.ExecutionConfig(policy="statements"))
            t2 = time.perf_counter()
            krn.execute(prog, fn + "_grad", call(), krn.ExecutionConfig(policy="statements"))
            t3 = time.perf_counter()
            cpu = ""
            if n <= args.cpu_rows:
                arrays = {"x": x.copy(), "b": b.copy(), "_d_x": np.zeros(n), "_d_b": np.zeros(n)}
                c0 = time.perf_counter()
                want = interp.detect(prog, fn + "_grad", arrays)
                cpu = f"{time.perf_counter() - c0:.2f}"
                assert len(want) == len(rep.records)
            print(f"| {n} | {tag} | {t1 - t0:.4f} | {len(rep.records)} | {t3 - t2:.4f} | {cpu} |", flush=True)


if __name__ == "__main__":
    main()
