"""Accumulate-shadow gradient (56 B/row: the shadows are read as well) through execute(), hand-written
vs generated kernels: python tools/accumulate_probe.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_13204_b200 as krn
from paper_2507_13204_b200 import ExecutionConfig, ViewStorage
n = 125_000_000
dev = krn.Device.get()
lap = krn.load_program("laplacian")
gp = krn.differentiate(lap, "normRes1DLaplacianSQ", ("x", "b"))
rng = np.random.default_rng(0)
base = {k: ViewStorage.from_values(k, rng.uniform(-1, 1, n)) for k in ("x", "b", "_d_x", "_d_b")}
for v in base.values():
    v.device_ptr(dev, write=False)
e0, e1 = dev.event(), dev.event()
pad = dev.alloc(8 << 28)
for policy in ("fused", "compiled"):
    cfg = ExecutionConfig(policy=policy, synchronous=False)
    best = 1e9
    for rep in range(5):
        call = {k: v.copy() for k, v in base.items()}
        dev.sync()
        dev.fill(pad, 1 << 28, 1.0)
        dev.record(e0)
        krn.execute(gp, "normRes1DLaplacianSQ_grad", call, cfg)
        dev.record(e1)
        ms = dev.elapsed_ms(e0, e1)
        if rep:
            best = min(best, ms)
        del call
    print(f"{policy:>9}: accumulate-shadow gradient {best:.3f} ms  {56 * n / best / 1e6:.0f} GB/s")
