"""Experiment: the fused gradient kernel reading x, b from PINNED HOST memory and writing the
shadows to pinned host memory (unified addressing: the kernel's own loads and stores are the PCIe
transfer), against the chunked copy pipeline of fused.run_streamed.
python tools/zero_copy_probe.py [rows]"""
import ctypes as C
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_13204_b200 as krn  # noqa: E402
from paper_2507_13204_b200 import _cabi  # noqa: E402
from paper_2507_13204_b200.runtime import _DeviceBuffer, pinned_array  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 125_000_000
dev = krn.Device.get()
lib = dev.lib
rng = np.random.default_rng(0)
hx, hb, hdx, hdb = (pinned_array((n,)) for _ in range(4))
step = 1 << 24
for lo in range(0, n, step):
    hx[lo:lo + step] = rng.uniform(-1, 1, min(step, n - lo))
    hb[lo:lo + step] = rng.uniform(-1, 1, min(step, n - lo))
xo = _DeviceBuffer(dev, 8 * n)
P = C.c_void_p


def zero_copy(dx_host=True):
    dxp = hdx.ctypes.data
    dbp = hdb.ctypes.data
    _cabi.check(lib.krn_laplacian_grad(dev.h, P(hx.ctypes.data), P(xo.ptr), P(hb.ctypes.data), P(dxp), P(dbp),
                                       1, 1, n, 0, n, None, 1.0))
    dev.sync()


for rep in range(4):
    t0 = time.perf_counter()
    zero_copy()
    dt = time.perf_counter() - t0
    print(f"zero-copy gradient: {dt * 1e3:8.2f} ms   {2 * n / dt / 1e9:6.2f} G entries/s   "
          f"{16 * n / dt / 1e9:5.1f} GB/s per direction")
print("checksum", float(hdx[:1000].sum()), float(hdb[-1000:].sum()))

lap = krn.load_program("laplacian")
gp = krn.differentiate(lap, "normRes1DLaplacianSQ", ("x", "b"))
for rep in range(3):
    call = {"x": krn.ViewStorage.pinned("x", (n,)), "b": krn.ViewStorage.pinned("b", (n,)),
            "_d_x": krn.ViewStorage.pinned("_d_x", (n,), zero=True), "_d_b": krn.ViewStorage.pinned("_d_b", (n,), zero=True)}
    call["x"].buffer[:] = hx
    call["b"].buffer[:] = hb
    t0 = time.perf_counter()
    krn.execute(gp, "normRes1DLaplacianSQ_grad", call, krn.ExecutionConfig(stream_host_io=True))
    dt = time.perf_counter() - t0
    print(f"chunked copy pipeline: {dt * 1e3:8.2f} ms")
print("checksum", float(call["_d_x"].peek()[:1000].sum()), float(call["_d_b"].peek()[-1000:].sum()))

# ---- which direction limits zero-copy? --------------------------------------------------------
dx_d, db_d = _DeviceBuffer(dev, 8 * n), _DeviceBuffer(dev, 8 * n)
x_d, b_d = _DeviceBuffer(dev, 8 * n), _DeviceBuffer(dev, 8 * n)
dev.upload(x_d.ptr, hx)
dev.upload(b_d.ptr, hb)
for label, xs, bs, dxs, dbs in (("reads over PCIe, writes to HBM", hx.ctypes.data, hb.ctypes.data, dx_d.ptr, db_d.ptr),
                                ("reads from HBM, writes over PCIe", x_d.ptr, b_d.ptr, hdx.ctypes.data, hdb.ctypes.data)):
    for rep in range(3):
        t0 = time.perf_counter()
        _cabi.check(lib.krn_laplacian_grad(dev.h, P(xs), P(xo.ptr), P(bs), P(dxs), P(dbs), 1, 1, n, 0, n, None, 1.0))
        dev.sync()
        dt = time.perf_counter() - t0
    print(f"{label}: {dt * 1e3:8.2f} ms  {16 * n / dt / 1e9:5.1f} GB/s")

# ---- hybrid: DMA uploads (chunked) + the kernel stores the shadows straight to pinned host memory ----
s_in = dev.aux_stream("in")
for chunk in (1 << 21, 1 << 22, 1 << 23):
    cuts = list(range(0, n, chunk)) + [n]
    nch = len(cuts) - 1
    ev = dev.event_pool(nch + 1)
    halos = np.zeros((nch, 6))
    for c in range(nch):
        lo, hi = cuts[c], cuts[c + 1]
        if lo >= 2:
            halos[c, 0:2] = hx[lo - 2:lo]
        if lo >= 1:
            halos[c, 2] = hb[lo - 1]
        m = min(2, n - hi)
        if m > 0:
            halos[c, 3:3 + m] = hx[hi:hi + m]
            halos[c, 5] = hb[hi]
    d_halo = _DeviceBuffer(dev, halos.nbytes)
    dev.upload(d_halo.ptr, halos)
    for rep in range(3):
        hdx[:] = 0.0
        hdb[:] = 0.0
        dev.sync()
        t0 = time.perf_counter()
        for c in range(nch):
            lo, hi = cuts[c], cuts[c + 1]
            off, nb = 8 * lo, 8 * (hi - lo)
            _cabi.check(lib.krn_upload_on(s_in, P(x_d.ptr + off), P(hx.ctypes.data + off), nb))
            _cabi.check(lib.krn_upload_on(s_in, P(b_d.ptr + off), P(hb.ctypes.data + off), nb))
            _cabi.check(lib.krn_event_record_on(s_in, P(ev[c])))
            _cabi.check(lib.krn_ctx_wait_event(dev.h, P(ev[c])))
            _cabi.check(lib.krn_laplacian_grad(dev.h, P(x_d.ptr + off), P(xo.ptr + off), P(b_d.ptr + off),
                                               P(hdx.ctypes.data + off), P(hdb.ctypes.data + off), 1, 1,
                                               hi - lo, lo, n, P(d_halo.ptr + 48 * c), 1.0))
        _cabi.check(lib.krn_stream_sync(s_in))
        dev.sync()
        dt = time.perf_counter() - t0
    print(f"hybrid (DMA up, kernel stores down), {chunk >> 20} Mi-row chunks: {dt * 1e3:8.2f} ms")
    print("   checksum", float(hdx[:1000].sum()), float(hdb[-1000:].sum()))
