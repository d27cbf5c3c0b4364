"""Small runs of every generated-kernel shape (window kernels with halos, rank-2 register columns,
fused flat reductions, scatter policies) for compute-sanitizer:

    compute-sanitizer --tool memcheck  python tools/sanitize_run.py
    compute-sanitizer --tool racecheck python tools/sanitize_run.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_13204_b200 as krn  # noqa: E402
from paper_2507_13204_b200 import ExecutionConfig, ViewStorage  # noqa: E402

rng = np.random.default_rng(0)
ran = 0
for stem in ("laplacian", "stencil_smooth", "rowscale_rank2", "gather_indirect", "mean_shift", "copy_chain",
             "window_wide", "window_partial", "window_war", "window_scatter", "rank2_bulk", "gather_rows_rank2",
             "taped_overwrites"):
    prog = krn.load_program(stem)
    fn = prog.functions[0]
    for n in (1, 129, 1030, 9000):
        data = {}
        for p in fn.params:
            if not p.is_view:
                data[p.name] = 0.75
            elif p.name == "idx":
                data[p.name] = rng.integers(0, n, size=n).astype(np.float64)
            elif p.type.rank == 2:
                data[p.name] = rng.normal(size=(n, 3))
            else:
                data[p.name] = rng.uniform(0.5, 1.5, size=n)
        wrt = tuple(p.name for p in fn.params if p.is_view and p.name != "idx")
        for policy in ("compiled", "statements"):
            cfg = ExecutionConfig(policy=policy)
            call = {k: ViewStorage.from_values(k, v) if isinstance(v, np.ndarray) else v for k, v in data.items()}
            krn.execute(prog, fn.name, call, cfg)
            try:
                gp = krn.differentiate(prog, fn.name, wrt, tape=True)
            except (krn.NotFeasible, ValueError):
                continue
            gfn = gp.functions[-1]
            call = {k: ViewStorage.from_values(k, v) if isinstance(v, np.ndarray) else v for k, v in data.items()}
            for sp, w in zip(gfn.params[len(fn.params):], wrt):
                call[sp.name] = ViewStorage.zeros(sp.name, np.shape(data[w]))
            krn.execute(gp, gfn.name, call, cfg)
            ran += 1
krn.Device.get().sync()
print("sanitize_run: done,", ran, "gradient runs")
