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
             "taped_overwrites", "stride2_scatter", "stride2_collide", "rank2_row_offset"):
    prog = krn.load_program(stem)
    fn = prog.functions[0]
    for n in (1, 129, 1030, 9000):
        data = {}
        for p in fn.params:
            if not p.is_view:
                data[p.name] = 0.75
            elif p.name == "idx":
                data[p.name] = rng.integers(0, n, size=n).astype(np.float64)
            elif p.name == "fine":
                data[p.name] = rng.normal(size=2 * n + 1)
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
            if n == 1030:  # the same gradient with check_finite on the fused path and with hardware reductions
                for extra in (ExecutionConfig(policy=policy, check_finite=True),
                              ExecutionConfig(policy=policy, deterministic_reduction=False)):
                    call = {k: ViewStorage.from_values(k, v) if isinstance(v, np.ndarray) else v for k, v in data.items()}
                    for sp, w in zip(gfn.params[len(fn.params):], wrt):
                        call[sp.name] = ViewStorage.zeros(sp.name, np.shape(data[w]))
                    krn.execute(gp, gfn.name, call, extra)
# neighbour registers over a local that is still lazily zero, and over a parameter (tile kernels, both layouts)
zero_local = krn.parse("""fn f(a: view<f64,1>) -> f64 {
    let t1: view<f64,1> = view("t1", extent(a, 0));
    let t2: view<f64,1> = view("t2", extent(a, 0));
    parallel_for i in 0..extent(a, 0) {
        t2(i) = t1(i) + a(i);
        if (i != 0) { t2(i) += 2.0 * t1(i - 1) + a(i - 1); }
        if (i != extent(a, 0) - 1) { t2(i) -= 0.125 * t1(i + 1); }
    }
    r = parallel_sum(t2);
    return r; }""")
for n in (1, 5, 130, 1030, 9000):
    for fuse in (True, False):
        for check in (False, True):
            krn.execute(zero_local, "f", {"a": ViewStorage.from_values("a", rng.normal(size=n))},
                        ExecutionConfig(policy="compiled", fuse_neighbours=fuse, check_finite=check))
            ran += 1
# the ordered queue through the raw ABI: holes, hot keys, widths, row records
import ctypes as C  # noqa: E402

from paper_2507_13204_b200 import _cabi  # noqa: E402

dev = krn.Device.get()
for records, size in ((1, 1), (4097, 300), (70_001, 5000), (70_001, 1 << 20)):
    keys = rng.integers(0, size, size=records).astype(np.uint32)
    keys[rng.random(records) < 0.2] = 0xFFFFFFFF
    keys[: records // 3] = 7 % size
    for width in (1, 2, 4):
        vals = rng.normal(size=records * width)
        bufs = [dev.alloc(8 * size), dev.alloc(4 * records), dev.alloc(8 * records * width)]
        dev.fill(bufs[0], size, 0.0)
        dev.upload(bufs[1], keys)
        dev.upload(bufs[2], vals)
        _cabi.check(dev.lib.krn_ordered_accumulate(dev.h, C.c_void_p(bufs[0]), size, C.c_void_p(bufs[1]),
                                                   C.c_void_p(bufs[2]), records, width))
        if size % 3 == 0:
            cols = (C.c_int * 3)(2, 0, 1)
            k2 = np.where(keys == 0xFFFFFFFF, keys, keys % (size // 3)).astype(np.uint32)
            dev.upload(bufs[1], k2)
            if width * records >= 3 * records:
                _cabi.check(dev.lib.krn_ordered_accumulate_rows(dev.h, C.c_void_p(bufs[0]), size // 3, 3, cols, 3,
                                                                C.c_void_p(bufs[1]), C.c_void_p(bufs[2]), records))
        dev.sync()
        for b in bufs:
            dev.free(b)
# queues that are already in bucket order (no record moves) and queues that are not 16-byte aligned
for records, size in ((4097, 300), (70_001, 1 << 20)):
    srt = np.sort(rng.integers(0, size, size=records)).astype(np.uint32)
    srt[records - records // 5:] = 0xFFFFFFFF
    vals = rng.normal(size=records)
    for shift in (0, 1, 3):
        bufs = [dev.alloc(8 * size), dev.alloc(4 * (records + 4)), dev.alloc(8 * (records + 4))]
        dev.fill(bufs[0], size, 0.0)
        for keys in (srt, rng.integers(0, size, size=records).astype(np.uint32)):
            dev.upload(bufs[1] + 4 * shift, keys)
            dev.upload(bufs[2] + 8 * shift, vals)
            _cabi.check(dev.lib.krn_ordered_accumulate(dev.h, C.c_void_p(bufs[0]), size, C.c_void_p(bufs[1] + 4 * shift),
                                                       C.c_void_p(bufs[2] + 8 * shift), records, 1))
        dev.sync()
        for b in bufs:
            dev.free(b)
krn.Device.get().sync()
print("sanitize_run: done,", ran, "gradient runs")
