"""Runs one corpus program (primal and gradient) a few times under one policy at one size, for ncu:
python tools/run_corpus_once.py sum_squares compiled 67108864 [reps] [hardware|check]   (hardware:
deterministic_reduction=False, i.e. hardware fp64 reductions instead of the ordered accumulation of atomic_add
queues; check: check_finite=True)"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_13204_b200 as krn  # noqa: E402
from paper_2507_13204_b200 import ExecutionConfig, ViewStorage  # noqa: E402

stem, policy, n = sys.argv[1], sys.argv[2], int(sys.argv[3])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 2
prog = krn.load_program(stem)
fn = prog.functions[0]
rng = np.random.default_rng(1)
base = {}
for p in fn.params:
    if not p.is_view:
        base[p.name] = 0.75
    elif p.name == "idx":
        base[p.name] = rng.integers(0, n, size=n).astype(np.float64)
    elif p.type.rank == 2:
        base[p.name] = rng.normal(size=(n, 3))
    else:
        base[p.name] = rng.normal(size=n)
wrt = tuple(p.name for p in fn.params if p.is_view and p.name != "idx")
gp = krn.differentiate(prog, fn.name, wrt)
gfn = gp.functions[-1]
hardware = len(sys.argv) > 5 and sys.argv[5] == "hardware"
check = len(sys.argv) > 5 and sys.argv[5] == "check"  # check_finite=True: the tracked plan
cfg = ExecutionConfig(policy="compiled" if policy == "pointwise" else policy, fuse_neighbours=policy != "pointwise",
                      deterministic_reduction=not hardware, check_finite=check)
for rep in range(reps):
    call = {k: ViewStorage.from_values(k, v) if isinstance(v, np.ndarray) else v for k, v in base.items()}
    krn.execute(prog, fn.name, call, cfg)
    call = {k: ViewStorage.from_values(k, v) if isinstance(v, np.ndarray) else v for k, v in base.items()}
    for sp, primal in zip(gfn.params[len(fn.params):], wrt):
        call[sp.name] = ViewStorage.zeros(sp.name, np.shape(base[primal]))
    krn.execute(gp, gfn.name, call, cfg)
print("done")
