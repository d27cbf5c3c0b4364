import sys, numpy as np
sys.path.insert(0,'/root/repo')
import paper_2507_13204_b200 as krn
from paper_2507_13204_b200 import ExecutionConfig, ViewStorage, compiled
stem = sys.argv[1] if len(sys.argv)>1 else "inplace_axpy"
prog = krn.load_program(stem); fn = prog.functions[0]
wrt = tuple(p.name for p in fn.params if p.is_view and p.name != "idx")
gp = krn.differentiate(prog, fn.name, wrt); gfn = gp.functions[-1]
for tr in (False, True):
    pl = compiled.plan_for(gfn, True, tr)
    print(tr, [s[0] for s in pl.steps], pl.launch_count)
n = 1 << 25
rng = np.random.default_rng(0)
base = {p.name: (ViewStorage.from_values(p.name, rng.normal(size=(n,3) if p.type.rank==2 else n)) if p.is_view else 0.75) for p in fn.params}
dev = krn.Device.get()
for v in base.values():
    if isinstance(v, ViewStorage): v.device_ptr(dev, write=False)
import time
for check in (False, True, False, True):
    best = 1e9; bw=1e9
    for rep in range(6):
        call = {k: (v.copy() if isinstance(v, ViewStorage) else v) for k, v in base.items()}
        for sp, w in zip(gfn.params[len(fn.params):], wrt):
            call[sp.name] = ViewStorage.zeros(sp.name, base[w].extents)
        dev.sync()
        e0, e1 = dev.event(), dev.event()
        l0=dev.launches(); t0=time.perf_counter()
        dev.record(e0)
        krn.execute(gp, gfn.name, call, ExecutionConfig(policy="compiled", check_finite=check))
        dev.record(e1)
        ms=dev.elapsed_ms(e0, e1); bw=min(bw,(time.perf_counter()-t0)*1e3)
        best = min(best, ms)
    print(stem, "check", check, "event ms %.3f wall %.3f launches %d" % (best, bw, dev.launches()-l0))
