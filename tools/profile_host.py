"""cProfile of the host side of execute() under one policy at the paper's size:
python tools/profile_host.py compiled grad"""
import cProfile
import os
import pstats
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_13204_b200 as krn  # noqa: E402
from paper_2507_13204_b200 import ExecutionConfig, ViewStorage  # noqa: E402

policy, which = sys.argv[1], sys.argv[2]
FN = "normRes1DLaplacianSQ"
lap = krn.load_program("laplacian")
gp = krn.differentiate(lap, FN, ("x", "b"))
dev = krn.Device.get()
n = 10_000
rng = np.random.default_rng(0)
x0, b0 = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
cfg = ExecutionConfig(policy=policy)


def call_once():
    call = {"x": ViewStorage.from_values("x", x0), "b": ViewStorage.from_values("b", b0)}
    if which == "grad":
        call["_d_x"] = ViewStorage.zeros("_d_x", (n,))
        call["_d_b"] = ViewStorage.zeros("_d_b", (n,))
    krn.execute(lap if which == "primal" else gp, FN if which == "primal" else FN + "_grad", call, cfg)


for _ in range(20):
    call_once()
pr = cProfile.Profile()
pr.enable()
for _ in range(300):
    call_once()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(28)
