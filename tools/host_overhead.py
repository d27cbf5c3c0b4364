"""Wall-clock cost of one synchronous execute() at the paper's size, per policy (what a
caller of the Python API sees; device time is a small part of it)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_13204_b200 as krn  # noqa: E402
from paper_2507_13204_b200 import ExecutionConfig, ViewStorage  # noqa: E402

FN = "normRes1DLaplacianSQ"
lap = krn.load_program("laplacian")
gp = krn.differentiate(lap, FN, ("x", "b"))
dev = krn.Device.get()
n = 10_000
rng = np.random.default_rng(0)
x0, b0 = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
for policy in ("fused", "compiled", "statements"):
    cfg = ExecutionConfig(policy=policy)
    for which in ("primal", "grad"):
        ts = []
        for rep in range(60):
            call = {"x": ViewStorage.from_values("x", x0), "b": ViewStorage.from_values("b", b0)}
            if which == "grad":
                call["_d_x"] = ViewStorage.zeros("_d_x", (n,))
                call["_d_b"] = ViewStorage.zeros("_d_b", (n,))
            for v in call.values():
                v.device_ptr(dev, write=False) if not v._zero else None
            dev.sync()
            t0 = time.perf_counter()
            krn.execute(lap if which == "primal" else gp, FN if which == "primal" else FN + "_grad", call, cfg)
            ts.append(time.perf_counter() - t0)
        ts = sorted(ts[10:])
        print(f"{policy:>10} {which:>6}: median {1e6 * ts[len(ts) // 2]:8.1f} us   min {1e6 * ts[0]:8.1f} us")
