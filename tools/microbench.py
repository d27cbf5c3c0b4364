"""Device-time microbenchmark of the fused kernels and builtins through the C ABI
(resident buffers, CUDA events on the library's stream, best and median of reps).

    python tools/microbench.py [--rows 125000000] [--reps 10]
"""
import argparse
import ctypes as C
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_13204_b200 as krn  # noqa: E402
from paper_2507_13204_b200 import _cabi  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, nargs="*", default=[125_000_000])
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    dev = krn.Device.get()
    lib = dev.lib
    out = {}
    for n in args.rows:
        bufs = {k: dev.alloc(8 * n) for k in ("x", "xo", "b", "dx", "db")}
        f = dev.alloc(8)
        rng = np.random.default_rng(1)
        chunk = 1 << 24
        for k in ("x", "b", "dx", "db"):
            for lo in range(0, n, chunk):
                a = rng.uniform(-1, 1, min(chunk, n - lo))
                dev.upload(bufs[k] + 8 * lo, a)
                dev.sync()
        p = {k: C.c_void_p(v) for k, v in bufs.items()}

        def primal():
            _cabi.check(lib.krn_laplacian_primal(dev.h, p["x"], p["xo"], p["b"], n, 0, n, None, C.c_void_p(f), 0))

        def grad(zero=0):
            _cabi.check(lib.krn_laplacian_grad(dev.h, p["x"], p["xo"], p["b"], p["dx"], p["db"], zero, zero,
                                               n, 0, n, None, 1.0))

        cases = {
            "primal": (primal, 24), "grad_acc": (lambda: grad(0), 56), "grad_zero": (lambda: grad(1), 40),
            "reduce": (lambda: dev.reduce_pairwise(bufs["x"], n, f, False), 8),
            "add_view": (lambda: dev.add_view(bufs["dx"], bufs["db"], n), 24),
            "add_scalar": (lambda: dev.add_scalar(bufs["dx"], n, 1e-9), 16),
            "fill": (lambda: dev.fill(bufs["xo"], n, 1.5), 8),
            "copy": (lambda: dev.copy(bufs["xo"], bufs["x"], n), 16),
        }
        e0, e1 = dev.event(), dev.event()
        res = {}
        for name, (fn, bpr) in cases.items():
            for _ in range(3):
                fn()
            ts = []
            for _ in range(args.reps):
                dev.record(e0)
                fn()
                dev.record(e1)
                ts.append(dev.elapsed_ms(e0, e1))
            best, med = min(ts), float(np.median(ts))
            res[name] = {"best_us": 1e3 * best, "median_us": 1e3 * med, "gbs_best": bpr * n / best / 1e6,
                         "gbs_median": bpr * n / med / 1e6}
        out[str(n)] = res
        for v in bufs.values():
            dev.free(v)
        dev.free(f)
        dev.sync()
    for n, res in out.items():
        print(f"rows={n}")
        for name, r in res.items():
            print(f"  {name:10s} best {r['best_us']:10.1f} us  median {r['median_us']:10.1f} us   "
                  f"{r['gbs_best']:8.1f} GB/s best  {r['gbs_median']:8.1f} GB/s median")
    print(json.dumps(out))


if __name__ == "__main__":
    main()
