"""The fused headline kernels from 1e4 to 1e7 rows: device time by CUDA events with L2 flushed
before every launch (as bench.py's sweep), plus an empty-stream event pair and a null-size launch
for the fixed cost; meant to run plain and under `ncu --metrics gpu__time_duration.sum`.

    python tools/sweep_mid.py [--reps 12]
"""
import argparse
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_13204_b200 as krn  # noqa: E402
from paper_2507_13204_b200 import _cabi  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=12)
    ap.add_argument("--rows", type=int, nargs="*", default=[10_000, 100_000, 300_000, 1_000_000, 3_000_000, 10_000_000])
    args = ap.parse_args()
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    dev = krn.Device(0, s.cuda_stream)
    peak = 6541.5
    flush = torch.empty(1 << 28, dtype=torch.uint8, device="cuda")

    def timed(fn):
        ts = []
        for _ in range(args.reps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        ts = sorted(ts[2:])
        return ts[0], ts[len(ts) // 2]

    print("empty event pair: %.2f us (best), %.2f us (median)" % timed(lambda: None))
    for n in args.rows:
        x, b, dx, db = (torch.rand(n, dtype=torch.float64, device="cuda") * 2.0 - 1.0 for _ in range(4))
        xo = torch.empty_like(x)
        f = torch.zeros(1, dtype=torch.float64, device="cuda")
        P = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
        tp = timed(lambda: _cabi.check(dev.lib.krn_laplacian_primal(dev.h, P(x), P(xo), P(b), n, 0, n, None, P(f), 0)))
        tg = timed(lambda: _cabi.check(dev.lib.krn_laplacian_grad(dev.h, P(x), P(xo), P(b), P(dx), P(db), 0, 0, n, 0, n,
                                                                 None, 1.0)))
        tz = timed(lambda: _cabi.check(dev.lib.krn_laplacian_grad(dev.h, P(x), P(xo), P(b), P(dx), P(db), 1, 1, n, 0, n,
                                                                 None, 1.0)))
        tc = timed(lambda: xo.copy_(x))
        print(f"rows={n:>9}  primal {tp[0]:8.2f} us ({24.0 * n / tp[0] / 1e3 / peak:4.2f} of peak)  "
              f"grad {tg[0]:8.2f} us ({56.0 * n / tg[0] / 1e3 / peak:4.2f})  grad0 {tz[0]:8.2f} us "
              f"({40.0 * n / tz[0] / 1e3 / peak:4.2f})  torch copy {tc[0]:8.2f} us ({16.0 * n / tc[0] / 1e3 / peak:4.2f})")


if __name__ == "__main__":
    main()
