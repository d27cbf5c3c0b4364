"""GPU tier, maximum size of the bandwidth sweep (BASELINE configs[2]): 10^9 rows on one
device (40 GB of Views).  The inputs come from an integer formula that host and device
evaluate identically, so sampled windows - both ends, block and chunk boundaries, the
4 GiB byte-offset boundary - are checked bit for bit against the C oracle, and the
objective against an independent device-side sum."""

import ctypes as C

import numpy as np
import pytest
import torch

import paper_2507_13204_b200 as krn
from paper_2507_13204_b200 import _cabi
from conftest import assert_bits

pytestmark = pytest.mark.gpu
N = 1_000_000_000


def _formula_np(lo, hi, mult, mod):
    j = np.arange(lo, hi, dtype=np.int64)
    # only exact operations (integer arithmetic, scaling by a power of two, one subtraction), so
    # numpy and torch-on-CUDA produce the same bits (torch turns `/ scalar` into `* (1/scalar)`)
    return ((j * mult) % mod).astype(np.float64) * 2.0 ** -19 - 1.0


def _formula_torch(n, mult, mod, out):
    step = 1 << 26
    for lo in range(0, n, step):
        hi = min(n, lo + step)
        j = torch.arange(lo, hi, dtype=torch.int64, device="cuda")
        out[lo:hi] = ((j * mult) % mod).to(torch.float64) * 2.0 ** -19 - 1.0
    return out


def test_one_billion_rows():
    from oracle import cport

    free, _ = torch.cuda.mem_get_info()
    if free < 56 * (1 << 30):
        pytest.skip("needs 56 GB of free device memory")
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    dev = krn.Device(0, s.cuda_stream)
    x = _formula_torch(N, 2654435761, 1048573, torch.empty(N, dtype=torch.float64, device="cuda"))
    b = _formula_torch(N, 40503, 1048571, torch.empty(N, dtype=torch.float64, device="cuda"))
    xo, dx, db = torch.empty_like(x), torch.empty_like(x), torch.empty_like(x)
    f = torch.zeros(1, dtype=torch.float64, device="cuda")
    P = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    _cabi.check(dev.lib.krn_laplacian_primal(dev.h, P(x), P(xo), P(b), N, 0, N, None, P(f), 0))
    _cabi.check(dev.lib.krn_laplacian_grad(dev.h, P(x), P(xo), P(b), P(dx), P(db), 1, 1, N, 0, N, None, 1.0))
    torch.cuda.synchronize()
    # objective: independent evaluation with torch ops (different summation order)
    xs = 3.0 * x
    y = 2.0 * xs - b
    y[1:] -= xs[:-1]
    y[:-1] -= xs[1:]
    f_ref = float(torch.sum(y * y).item())
    assert abs(float(f.item()) - f_ref) <= 1e-12 * abs(f_ref)
    assert torch.equal(xo, xs)
    del xs, y
    # windows, bit for bit against the oracle
    w = 4096
    starts = [0, N - w, (1 << 29) - w // 2, 8192 * 1000 - 7, 536_870_912 - 2, 123_456_789, N // 2 + 1]
    for lo in starts:
        lo = max(0, min(lo, N - w))
        hi = lo + w
        xa, ba = _formula_np(lo, hi, 2654435761, 1048573), _formula_np(lo, hi, 40503, 1048571)
        assert_bits(x[lo:hi].cpu().numpy(), xa, "input formula")  # host and device agree on the inputs
        dxo, dbo = np.zeros(w), np.zeros(w)
        cport.laplacian_grad(xa.copy(), ba, dxo, dbo, 1.0)
        a = 0 if lo == 0 else 2           # rows whose stencil support lies inside the window
        z = w if hi == N else w - 2
        assert_bits(dx[lo + a:lo + z].cpu().numpy(), dxo[a:z], f"_d_x window {lo}")
        assert_bits(db[lo + a:lo + z].cpu().numpy(), dbo[a:z], f"_d_b window {lo}")


def test_generated_window_kernels_beyond_4gib_offsets():
    """The headline through the fusion pass (ONE generated window kernel per side) at 2^29 + 5 rows:
    byte offsets exceed 4 GiB, 65 k blocks of 8 steps.  Checked bit for bit against the hand-written
    kernels (themselves pinned to the oracle above): objective, scaled x, both shadows."""
    from paper_2507_13204_b200 import ExecutionConfig, ViewStorage

    free, _ = torch.cuda.mem_get_info()
    n = (1 << 29) + 5
    if free < 14 * 8 * n:
        pytest.skip("needs ~60 GB of free device memory")
    lap = krn.load_program("laplacian")
    gp = krn.differentiate(lap, "normRes1DLaplacianSQ", ("x", "b"))
    xh, bh = _formula_np(0, n, 2654435761, 1048573), _formula_np(0, n, 40503, 1048571)
    results = {}
    for policy in ("fused", "compiled"):
        cfg = ExecutionConfig(policy=policy)
        call = {"x": ViewStorage.from_values("x", xh), "b": ViewStorage.from_values("b", bh)}
        f = krn.execute(lap, "normRes1DLaplacianSQ", call, cfg).value
        g = {"x": ViewStorage.from_values("x", xh), "b": ViewStorage.from_values("b", bh),
             "_d_x": ViewStorage.zeros("_d_x", (n,)), "_d_b": ViewStorage.zeros("_d_b", (n,))}
        krn.execute(gp, "normRes1DLaplacianSQ_grad", g, cfg)
        results[policy] = (f, call["x"].peek().copy(), g["_d_x"].peek().copy(), g["_d_b"].peek().copy(),
                           g["x"].peek().copy())
        del call, g
    a, c = results["fused"], results["compiled"]
    assert_bits(c[0], a[0], "objective")
    for k, name in ((1, "x after primal"), (2, "_d_x"), (3, "_d_b"), (4, "x after gradient")):
        assert np.array_equal(c[k].view(np.uint64), a[k].view(np.uint64)), name


def test_quarter_billion_ordered_records():
    """BASELINE-scale queue for the ordered accumulation (2^28 records onto 2^27 + 5 targets: three
    8-bit partition passes' worth of tiles, a 16 M-entry digit table, 32-bit destinations close to
    2^28).  Keys and values are generated on the device; contributions are small integers, exact in any
    order, so the result has a closed form: the size-independent properties checked are (a) every
    target equals its bincount-weighted sum, (b) a second identical call doubles it, (c) -values
    bring it back to zero - with sampled windows compared element by element."""
    free, _ = torch.cuda.mem_get_info()
    records, size = 1 << 28, (1 << 27) + 5
    if free < 24 * (1 << 30):
        pytest.skip("needs 24 GB of free device memory")
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    dev = krn.Device(0, s.cuda_stream)
    j = torch.arange(records, dtype=torch.int64, device="cuda")
    keys64 = (j * 2654435761 + (j >> 7) * 40503) % size
    keys64[::1001] = 12345  # a mildly hot target: a run of ~268 k records in one bucket
    keys = keys64.to(torch.int32)  # bit pattern of uint32 (all keys < 2^31)
    vals = ((j % 7) + 1).to(torch.float64)
    del j
    target = torch.zeros(size, dtype=torch.float64, device="cuda")
    P = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    want = torch.zeros(size, dtype=torch.float64, device="cuda").index_add_(0, keys64, vals)
    _cabi.check(dev.lib.krn_ordered_accumulate(dev.h, P(target), size, P(keys), P(vals), records, 1))
    torch.cuda.synchronize()
    assert torch.equal(target, want)
    _cabi.check(dev.lib.krn_ordered_accumulate(dev.h, P(target), size, P(keys), P(vals), records, 1))
    torch.cuda.synchronize()
    assert torch.equal(target, 2.0 * want)
    neg = -2.0 * vals
    _cabi.check(dev.lib.krn_ordered_accumulate(dev.h, P(target), size, P(keys), P(neg), records, 1))
    torch.cuda.synchronize()
    assert int(torch.count_nonzero(target).item()) == 0
