"""Launches the headline objective + gradient at the paper's sizes, all three policies,
a few times each (meant to run under `ncu --metrics gpu__time_duration.sum`)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_13204_b200 as krn  # noqa: E402

FN = "normRes1DLaplacianSQ"
lap = krn.load_program("laplacian")
gp = krn.differentiate(lap, FN, ("x", "b"))
for n in (5000, 10000):
    rng = np.random.default_rng(0)
    x, b = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
    for policy in ("fused", "compiled", "statements"):
        cfg = krn.ExecutionConfig(policy=policy)
        for rep in range(3):
            krn.execute(lap, FN, {"x": x.copy(), "b": b.copy()}, cfg)
            krn.execute(gp, FN + "_grad", {"x": x.copy(), "b": b.copy(), "_d_x": krn.ViewStorage.zeros("_d_x", (n,)),
                                            "_d_b": krn.ViewStorage.zeros("_d_b", (n,))}, cfg)
print("done")
