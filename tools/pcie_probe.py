"""Host<->device copy bandwidth of this box (pinned memory): the ceiling of the e2e leg of bench.py.
python tools/pcie_probe.py [GB]"""
import sys
import time

import torch

gb = float(sys.argv[1]) if len(sys.argv) > 1 else 2.0
n = int(gb * 1e9 / 8)
h_in = torch.empty(n, dtype=torch.float64).pin_memory()
h_out = torch.empty(n, dtype=torch.float64).pin_memory()
h_in.uniform_(-1, 1)
d_a = torch.empty(n, dtype=torch.float64, device="cuda")
d_b = torch.ones(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timeit(fn, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best


def h2d():
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)


def both():
    h2d()
    d2h()


def chunked(chunk_rows):
    def run():
        for lo in range(0, n, chunk_rows):
            hi = min(n, lo + chunk_rows)
            with torch.cuda.stream(s1):
                d_a[lo:hi].copy_(h_in[lo:hi], non_blocking=True)
            with torch.cuda.stream(s2):
                h_out[lo:hi].copy_(d_b[lo:hi], non_blocking=True)
    return run


for name, fn in (("h2d", h2d), ("d2h", d2h), ("both directions at once", both),
                 ("both, 4 Mi-row chunks", chunked(1 << 22)), ("both, 16 Mi-row chunks", chunked(1 << 24))):
    t = timeit(fn)
    print(f"{name:>28}: {t * 1e3:8.2f} ms  {gb / t:6.1f} GB/s per direction")
