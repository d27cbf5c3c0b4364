"""Throughput of the accumulation policies for a non-injective scatter
(`atomic_add(acc(idx(i)), v(i))`, the adjoint of an indirect gather) across index
maps and target sizes.  Device time of the generated kernel, CUDA events.

    python tools/atomic_policies.py [--n 16777216] [--json out.json]
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_13204_b200 as krn  # noqa: E402
from paper_2507_13204_b200 import ExecutionConfig, ViewStorage  # noqa: E402

SRC = """fn scatter(idx: view<f64, 1>, v: view<f64, 1>, acc: view<f64, 1>) {
    parallel_for i in 0..extent(idx, 0) { atomic_add(acc(idx(i)), v(i)); } }"""


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1 << 24)
    ap.add_argument("--json")
    ap.add_argument("--only", help="rows:map:policy to run a single case (for ncu)")
    args = ap.parse_args()
    n = args.n
    dev = krn.Device.get()
    prog = krn.parse(SRC)
    rng = np.random.default_rng(0)
    v = ViewStorage.from_values("v", rng.normal(size=n))
    v.device_ptr(dev, write=False)
    e0, e1 = dev.event(), dev.event()
    out = []
    for rows in (64, 4096, 1 << 16, 1 << 20, n):
        maps = {
            "uniform": rng.integers(0, rows, size=n),
            "clustered8": (np.arange(n) // 8) % rows,
            "hot90": np.where(rng.random(n) < 0.9, 3 % rows, rng.integers(0, rows, size=n)),
        }
        for label, idx in maps.items():
            iv = ViewStorage.from_values("idx", idx.astype(np.float64))
            iv.device_ptr(dev, write=False)
            want = None
            for apol in ("ordered", "red", "lead", "warp", "smem"):
                if apol == "smem" and rows > 6144:
                    continue
                if args.only and args.only != f"{rows}:{label}:{apol}":
                    continue
                cfg = ExecutionConfig(atomic_policy=apol, synchronous=False, device=dev)
                ts = []
                for rep in range(5):
                    acc = ViewStorage.zeros("acc", (rows,))
                    acc.device_ptr(dev)
                    dev.sync()
                    dev.record(e0)
                    krn.execute(prog, "scatter", {"idx": iv, "v": v, "acc": acc}, cfg)
                    dev.record(e1)
                    ts.append(dev.elapsed_ms(e0, e1))
                got = acc.buffer.copy()
                if apol == "ordered":
                    # two runs of the ordered policy must agree bit for bit (the last two repetitions ran
                    # on fresh zero targets): checked against one more run
                    again = ViewStorage.zeros("acc", (rows,))
                    krn.execute(prog, "scatter", {"idx": iv, "v": v, "acc": again},
                                ExecutionConfig(atomic_policy=apol, device=dev))
                    assert np.array_equal(again.buffer, got), "ordered policy is not reproducible"
                if want is None:
                    want = np.bincount(idx, weights=v.peek(), minlength=rows)
                err = float(np.max(np.abs(got - want) / np.maximum(np.abs(want), 1e-300)))
                best = min(ts[1:])
                rec = dict(rows=rows, map=label, policy=apol, ms=best, contributions_per_s=n / best * 1e3,
                           max_rel_err=err)
                out.append(rec)
                print(f"rows={rows:>9} {label:>10} {apol:>5}: {best:9.3f} ms  {n / best / 1e6:9.1f} Gcontrib/s  "
                      f"err {err:.1e}")
    if args.json:
        with open(args.json, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
