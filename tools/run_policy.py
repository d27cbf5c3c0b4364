"""Runs the headline objective + gradient once or a few times under one policy at one size
(for ncu): python tools/run_policy.py compiled 16777216 [reps]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_13204_b200 as krn  # noqa: E402

policy, n = sys.argv[1], int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
FN = "normRes1DLaplacianSQ"
lap = krn.load_program("laplacian")
gp = krn.differentiate(lap, FN, ("x", "b"))
rng = np.random.default_rng(0)
x, b = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
cfg = krn.ExecutionConfig(policy=policy)
for rep in range(reps):
    krn.execute(lap, FN, {"x": x.copy(), "b": b.copy()}, cfg)
    krn.execute(gp, FN + "_grad", {"x": x.copy(), "b": b.copy(), "_d_x": krn.ViewStorage.zeros("_d_x", (n,)),
                                    "_d_b": krn.ViewStorage.zeros("_d_b", (n,))}, cfg)
print("done")
