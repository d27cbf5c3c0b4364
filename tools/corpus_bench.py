"""Device time of every corpus program and its generated gradient under the generic
policies (statement granularity vs the fusion pass), with the achieved ALGORITHMIC
bandwidth (compulsory bytes of the program / time).  CUDA events around an
asynchronous execute() on resident Views; best of 4.

    python tools/corpus_bench.py [--n 16777216] [--md out.md]
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_13204_b200 as krn  # noqa: E402
from paper_2507_13204_b200 import ExecutionConfig, ViewStorage  # noqa: E402

# compulsory bytes per row (primal, gradient with zero-provenance shadows): inputs read once,
# observable outputs written once (SURVEY.md section 8d gives laplacian, sum_squares, rowscale)
BYTES = {
    "laplacian": (24, 40), "sum_squares": (8, 16), "affine_weighted": (16, 16), "safe_divide": (8, 16),
    "inplace_axpy": (24, 40), "copy_chain": (8, 16), "fill_scale": (8, 8), "mean_shift": (16, 24),
    "gather_indirect": (16, 24), "stencil_smooth": (8, 16), "rowscale_rank2": (32, 64),
    # extra_programs/: 2-D View through a non-injective index map (BASELINE.json configs[3]):
    # idx, w, 3 gathered columns; gradient adds _d_w and read-modify-write of 3 scattered columns
    "gather_rows_rank2": (40, 96),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1 << 24)
    ap.add_argument("--md")
    ap.add_argument("--only", help="comma-separated program stems")
    args = ap.parse_args()
    n = args.n
    dev = krn.Device.get()
    e0, e1 = dev.event(), dev.event()
    rows = []
    # a long kernel enqueued ahead of every timed call: the host prepares and enqueues the launch
    # sequence while it runs, so the event interval is device time, not Python time.  The pad is a
    # READ-ONLY reduction: a fill would leave ~100 MB of dirty lines in L2 whose write-back lands
    # inside the timed interval (15 us at 7 TB/s, 8 % of a 0.2 ms call).
    pad_rows = 1 << 28
    pad = dev.alloc(8 * pad_rows)
    pad_out = dev.alloc(8)
    dev.fill(pad, pad_rows, 1.0)
    for stem in sorted(BYTES):
        if args.only and stem not in args.only.split(","):
            continue
        prog = krn.load_program(stem)
        fn = prog.functions[0]
        rng = np.random.default_rng(1)
        base = {}
        for p in fn.params:
            if not p.is_view:
                base[p.name] = 0.75
            elif p.name == "idx":
                base[p.name] = ViewStorage.from_values("idx", rng.integers(0, n, size=n).astype(np.float64))
            elif p.type.rank == 2:
                base[p.name] = ViewStorage.from_values(p.name, rng.normal(size=(n, 3)))
            else:
                base[p.name] = ViewStorage.from_values(p.name, rng.normal(size=n))
        for v in base.values():
            if isinstance(v, ViewStorage):
                v.device_ptr(dev, write=False)
        wrt = tuple(p.name for p in fn.params if p.is_view and p.name != "idx")
        gp = krn.differentiate(prog, fn.name, wrt)
        gfn = gp.functions[-1]
        policies = ["statements", "pointwise", "compiled"] + (["fused"] if stem == "laplacian" else [])
        for policy in policies:
            # "pointwise" = the fusion pass without halo recompute; "fused" = the hand-written kernels
            cfg = ExecutionConfig(policy="compiled" if policy == "pointwise" else policy, synchronous=False,
                                  device=dev, fuse_neighbours=policy != "pointwise")
            best = {"primal": 1e9, "grad": 1e9}
            launches = {}
            for rep in range(4):
                for which in ("primal", "grad"):
                    call = {k: v.copy() if isinstance(v, ViewStorage) else v for k, v in base.items()}
                    if which == "grad":
                        for sp, primal in zip(gfn.params[len(fn.params):], wrt):
                            call[sp.name] = ViewStorage.zeros(sp.name, base[primal].extents)
                    dev.sync()
                    dev.reduce_pairwise(pad, pad_rows, pad_out, False)
                    l0 = dev.launches()
                    dev.record(e0)
                    krn.execute(prog if which == "primal" else gp, fn.name if which == "primal" else gfn.name, call, cfg)
                    dev.record(e1)
                    ms = dev.elapsed_ms(e0, e1)
                    launches[which] = dev.launches() - l0
                    if rep:
                        best[which] = min(best[which], ms)
                    del call
            bp, bg = BYTES[stem]
            rows.append((stem, policy, best["primal"], bp * n / best["primal"] / 1e6, launches["primal"],
                         best["grad"], bg * n / best["grad"] / 1e6, launches["grad"], best["grad"] / best["primal"]))
            print("%-16s %-10s primal %8.3f ms %7.0f GB/s (%d launches)   grad %8.3f ms %7.0f GB/s (%d launches)   ratio %.2f"
                  % rows[-1])
    if args.md:
        with open(args.md, "w") as f:
            f.write(f"# Corpus programs under the generic policies, {n} rows, one B200\n\n"
                    "`tools/corpus_bench.py`.  Policies: statements = one launch per statement; pointwise = fusion pass "
                    "without halo recompute; compiled = fusion pass with window kernels; fused = hand-written kernels.  GB/s = compulsory bytes of the program (inputs read once, observable "
                    "outputs written once; zero-provenance shadows) / device time of the whole launch sequence, so it "
                    "falls with every byte a policy moves beyond the minimum.  Launches = kernels of this library "
                    "(memsets and D2D copies not counted).\n\n"
                    "| program | policy | primal ms | primal GB/s | launches | grad ms | grad GB/s | launches | grad/primal |\n"
                    "|---|---|---|---|---|---|---|---|---|\n")
            for r in rows:
                f.write("| %s | %s | %.3f | %.0f | %d | %.3f | %.0f | %d | %.2f |\n" % r)


if __name__ == "__main__":
    main()
