"""Device time of krn_ordered_accumulate (csrc/krn_ordered.cu) alone, through the raw C ABI:
records already staged in HBM, CUDA events around the call, across queue lengths, target sizes
and key distributions; achieved GB/s over the ALGORITHMIC bytes of the call:
per record 4 B key + 8*width B values (planes) read, per distinct target 16 B read-modify-write.

    python tools/ordered_bench.py [--records 16777216] [--json out.json] [--only rows:map]
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
    ap.add_argument("--records", type=int, default=1 << 24)
    ap.add_argument("--width", type=int, default=1)
    ap.add_argument("--json")
    ap.add_argument("--only")
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    m, w = args.records, args.width
    dev = krn.Device.get()
    lib = dev.lib
    rng = np.random.default_rng(0)
    vals = rng.normal(size=m * w)
    d_vals = dev.alloc(vals.nbytes)
    dev.upload(d_vals, vals)
    d_keys = dev.alloc(4 * m)
    e0, e1 = dev.event(), dev.event()
    out = []
    for rows in (64, 4096, 1 << 16, 1 << 20, 1 << 24, m):
        maps = {
            "uniform": rng.integers(0, rows, size=m),
            "clustered8": (np.arange(m) // 8) % rows,
            "hot90": np.where(rng.random(m) < 0.9, 3 % rows, rng.integers(0, rows, size=m)),
            "sorted": np.sort(rng.integers(0, rows, size=m)),  # already in bucket order: no record moves
        }
        d_t = dev.alloc(8 * rows)
        for label, keys in maps.items():
            if args.only and args.only != f"{rows}:{label}":
                continue
            k32 = keys.astype(np.uint32)
            dev.upload(d_keys, k32)
            distinct = int(np.unique(k32).size)
            ts = []
            for _ in range(args.reps):
                dev.fill(d_t, rows, 0.0)
                dev.sync()
                l0 = dev.launches()
                dev.record(e0)
                _cabi.check(lib.krn_ordered_accumulate(dev.h, C.c_void_p(d_t), rows, C.c_void_p(d_keys),
                                                       C.c_void_p(d_vals), m, w))
                dev.record(e1)
                ts.append(dev.elapsed_ms(e0, e1))
                launches = dev.launches() - l0
            best = min(ts[1:])
            alg = m * (4 + 8 * w) + 16 * distinct
            rec = dict(rows=rows, map=label, records=m, width=w, distinct_targets=distinct, ms=best, launches=launches,
                       records_per_s=m / best * 1e3, algorithmic_bytes=alg, algorithmic_gbs=alg / best / 1e6)
            out.append(rec)
            print(f"rows={rows:>9} {label:>10}: {best:9.3f} ms  {m / best / 1e6:8.2f} Grec/s  "
                  f"{alg / best / 1e6:8.1f} GB/s algorithmic  {launches} launches")
        dev.free(d_t)
    if args.json:
        with open(args.json, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
