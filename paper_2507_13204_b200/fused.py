"""Recognition of the headline objective and dispatch to its fused kernels.

A function is recognised structurally: its tree, with identifiers renamed in
order of first appearance and the seed literal abstracted, must equal the tree
of ``programs/laplacian.krn`` (or of the gradient this package's own
``differentiate`` generates from it, for wrt = (x, b), (x,) or (b,)).  Nothing
is matched by name, so a tree produced by the reference package, or the same
program with other identifiers, takes the same path.

What the fused kernels may assume, and what is checked before dispatch:
all views are rank 1 with at least ``extent(x, 0)`` rows (otherwise the
statement path runs and reports OutOfBounds exactly as the reference does).
"""

from __future__ import annotations

import ctypes as C
import os

from . import _cabi
from .lang import differentiate, parse
from .lang.nodes import kind

_PROGRAM = os.path.join(os.path.dirname(os.path.abspath(__file__)), "programs", "laplacian.krn")
_FN = "normRes1DLaplacianSQ"


def _canon(fn, seed_hole: bool):
    """Hashable structural key: names replaced by first-appearance numbers."""
    names: dict = {}

    def nm(s):
        return names.setdefault(s, len(names))

    seeds: list = []

    def go(n, seed_ctx=False):
        if isinstance(n, (tuple, list)):
            return tuple(go(x) for x in n)
        if isinstance(n, str):
            return ("name", nm(n))
        if n is None or isinstance(n, (int, float)):
            return n
        k = kind(n)
        if k == "ViewDescriptor":
            return (k, nm(n.name), n.rank, tuple(kind(e) for e in n.extents))
        if k == "Param":
            return (k, nm(n.name), go(n.type) if n.is_view else "f64")
        if k == "FunctionDef":
            return (k, go(n.params), go(n.body), n.returns)
        if k == "DeclView":
            return (k, go(n.descriptor), go(n.dyn_args))
        if k in ("Literal", "IntLiteral"):
            return (k, n.value)
        if k in ("ScalarVar", "IndexVar", "Counter"):
            return (k, nm(n.name))
        if k == "ViewAccess":
            return (k, nm(n.view), go(n.indices))
        if k == "Extent":
            return (k, nm(n.view), n.dim)
        if k in ("Binary", "IdxBinary", "Compare"):
            return (k, n.op, go(n.lhs), go(n.rhs))
        if k == "Neg":
            return (k, go(n.operand))
        if k == "DeclScalar":
            return (k, nm(n.name), go(n.init))
        if k == "AssignView":
            return (k, go(n.target), n.op, go(n.rhs))
        if k == "AssignScalar":
            # the seed statement `_d_ret += <literal>` at function scope
            if seed_hole and n.op == "+=" and kind(n.rhs) == "Literal" and not seeds and _is_seed(n):
                seeds.append(float(n.rhs.value))
                return (k, nm(n.name), n.op, "SEED")
            return (k, nm(n.name), n.op, go(n.rhs))
        if k in ("If",):
            return (k, go(n.cond), go(n.body))
        if k == "ParallelFor":
            return (k, nm(n.counter), go(n.upper), go(n.body))
        if k in ("DeepCopy", "ParallelSumInto"):
            return (k, nm(n.dst), go(n.src) if not isinstance(n.src, str) else ("name", nm(n.src)))
        if k == "ParallelSum":
            return (k, nm(n.dst), nm(n.src))
        if k == "AtomicAdd":
            return (k, go(n.target), go(n.value))
        if k == "Return":
            return (k, go(n.value))
        raise TypeError(k)

    def _is_seed(stmt):
        return stmt.name.startswith("_d_")

    key = go(fn)
    return key, (seeds[0] if seeds else None)


class _Match:
    def __init__(self, grad: bool, wrt=(), seed=1.0):
        self.grad, self.wrt, self.seed = grad, wrt, seed

    def names(self, fn):
        """Bind roles to the function's actual parameter names (positional)."""
        p = [q.name for q in fn.params]
        roles = {"x": p[0], "b": p[1]}
        rest = p[2:]
        for w in self.wrt:
            roles["d" + w] = rest.pop(0)
        return roles


class _Bound:
    """A recognised function ready to run."""

    def __init__(self, fn, m: _Match):
        self.m = m
        self.roles = m.names(fn)

    def applicable(self, views) -> bool:
        n = views[self.roles["x"]].extents[0]
        for name in self.roles.values():
            v = views[name]
            if len(v.extents) != 1 or v.extents[0] < n:
                return False
        # distinct storage objects only (aliased arguments take the generic path)
        objs = [id(views[name]) for name in self.roles.values()]
        return len(set(objs)) == len(objs)

    # rows per chunk of the pipelined host path: 4 Mi rows = 32 MB per View and chunk,
    # ~0.6 ms of PCIe time, large against launch/event overheads, small against the whole
    # Measured on this pool (tools/pcie_probe.py, 2 GB each way at once, PCIe 5 x16): 40.0 ms in one
    # piece (50 GB/s per direction), 43.0 ms in 4 Mi-row pieces, 40.8 ms in 16 Mi-row pieces.  In the
    # pipeline the download of a chunk waits for its upload, so a call costs about
    # chunk/bandwidth + whole download + per-chunk overheads: larger or ramped chunks were slower
    # (46.3 ms with 16 Mi-row chunks and 1-2-4-8 ramps vs 44.0 ms with uniform 4 Mi rows).
    # Letting the kernel itself move the data (unified addressing: loads from / stores to the pinned
    # host arrays, tools/zero_copy_probe.py) was measured too: stores alone run at 52.7 GB/s and loads
    # alone at 46.8 GB/s, but both together only at 37.5 GB/s each (53.4 ms), and DMA uploads combined
    # with kernel stores take 45.7 ms - the copy-engine pipeline below stays the fastest (43.8 ms).
    # Chunk schedule: also measured (same box, 125 M rows) were chunks that double from 256 Ki / 1 Mi
    # rows at the start and halve at the end, to shorten the fill and drain of the pipeline: 44.99 /
    # 44.21 ms against 44.66 ms for uniform chunks (noise), and uniform 2 Mi / 8 Mi rows: 46.2 / 46.1 ms.
    STREAM_CHUNK = 1 << 22
    STREAM_MIN_ROWS = 1 << 23

    def run(self, dev, views, scalars, cfg=None):
        from .runtime import _DeviceBuffer

        synchronous = True if cfg is None else cfg.synchronous
        lib = dev.lib
        x, b = views[self.roles["x"]], views[self.roles["b"]]
        n = x.extents[0]
        if n == 0:
            return None if self.m.grad else 0.0
        if (self.m.grad and synchronous and cfg is not None and cfg.stream_host_io
                and n >= self.STREAM_MIN_ROWS and not x._dev_ok and not b._dev_ok
                and all(views[name].extents[0] == n for name in self.roles.values())):
            # (Views longer than x - legal: only rows [0, n) are touched - take the resident path,
            # which keeps their tails; the chunk buffers of the pipeline are sized by n)
            return self.run_streamed(dev, views)
        x_in = x.device_ptr(dev, write=False)
        b_ptr = b.device_ptr(dev, write=False)
        x_out = _DeviceBuffer(dev, x.nbytes)
        if not self.m.grad:
            # the last block stores the objective straight into page-locked host memory
            # (UVA: the pinned staging block is device-addressable): no result buffer, no
            # separate D2H copy on the latency-bound path
            f = dev._pinned.value + 64
            _cabi.check(lib.krn_laplacian_primal(dev.h, C.c_void_p(x_in), C.c_void_p(x_out.ptr),
                                                 C.c_void_p(b_ptr), n, 0, n, None, C.c_void_p(f), 0))
            x._adopt(x_out)
            if not synchronous:
                return None
            dev.sync()
            return float(dev.staging[64:72].view("float64")[0])
        dx, db = self._shadows(views)
        dx_zero = bool(dx is not None and dx._zero)
        db_zero = bool(db is not None and db._zero)
        # the kernel writes rows [0, n) only: a lazily zero shadow with MORE rows must really hold
        # its zeros beyond them (the read of the zeros is still skipped)
        dx_ptr = dx.device_ptr(dev, discard=dx_zero and dx.extents[0] == n) if dx is not None else 0
        db_ptr = db.device_ptr(dev, discard=db_zero and db.extents[0] == n) if db is not None else 0
        _cabi.check(lib.krn_laplacian_grad(dev.h, C.c_void_p(x_in), C.c_void_p(x_out.ptr), C.c_void_p(b_ptr),
                                           C.c_void_p(dx_ptr), C.c_void_p(db_ptr), int(dx_zero), int(db_zero),
                                           n, 0, n, None, float(self.m.seed)))
        x._adopt(x_out)
        if synchronous:
            dev.sync()
        return None

    def _shadows(self, views):
        dx = views[self.roles["dx"]] if "dx" in self.roles else None
        db = views[self.roles["db"]] if "db" in self.roles else None
        return dx, db

    def run_streamed(self, dev, views):
        """Gradient with HOST-resident inputs: rows are cut into chunks; the upload of
        chunk c+1, the kernel of chunk c and the download of the shadows of chunk c-1
        run concurrently on three streams (PCIe is full duplex), so the call costs about
        max(H2D, D2H) instead of H2D + kernel + D2H.  Each chunk is a shard of the
        problem (csrc/krn_laplacian.cu); its halo rows come from the host arrays, packed
        once.  Afterwards the Views are resident in HBM *and* the shadows' host arrays
        are current."""
        import numpy as np

        from .runtime import _DeviceBuffer, pinned_array

        lib = dev.lib
        x, b = views[self.roles["x"]], views[self.roles["b"]]
        dx, db = self._shadows(views)
        n = x.extents[0]
        hx, hb = x.peek(), b.peek()
        cuts = stream_cuts(n, self.STREAM_CHUNK)
        nch = len(cuts) - 1
        # halo rows of every chunk, from the host copies (zeros where outside the problem)
        halos = dev.pinned_scratch(6 * nch)
        halos[:] = 0.0
        h = halos.reshape(nch, 6)
        for c in range(nch):
            lo, hi = cuts[c], cuts[c + 1]
            if lo >= 2:
                h[c, 0:2] = hx[lo - 2:lo]
            elif lo == 1:
                h[c, 1] = hx[0]
            if lo >= 1:
                h[c, 2] = hb[lo - 1]
            m = min(2, n - hi)
            if m > 0:
                h[c, 3:3 + m] = hx[hi:hi + m]
                h[c, 5] = hb[hi]
        bufs = {k: _DeviceBuffer(dev, 8 * n) for k in ("x", "xo", "b")}
        d_halo = _DeviceBuffer(dev, 8 * 6 * nch)
        shadows = []
        for v in (dx, db):
            if v is None:
                shadows.append(None)
                continue
            zero = bool(v._zero)
            if v._host is None:
                v._host = pinned_array(v.extents)
            buf = _DeviceBuffer(dev, 8 * n) if (v._dev is None or v._dev.dev is not dev) else v._dev
            need_upload = (not zero) and not v._dev_ok
            shadows.append((v, buf, zero, need_upload))
        s_in, s_out = dev.aux_stream("in"), dev.aux_stream("out")
        ev = dev.event_pool(2 * nch + 1)
        P = C.c_void_p
        _cabi.check(lib.krn_upload_on(s_in, P(d_halo.ptr), P(halos.ctypes.data), halos.nbytes))
        # allocations above were made on the context's stream: let the copy streams see them
        dev.record(ev[2 * nch])
        _cabi.check(lib.krn_stream_wait_event(s_in, P(ev[2 * nch])))
        _cabi.check(lib.krn_stream_wait_event(s_out, P(ev[2 * nch])))
        for c in range(nch):
            lo, hi = cuts[c], cuts[c + 1]
            off, nb = 8 * lo, 8 * (hi - lo)
            _cabi.check(lib.krn_upload_on(s_in, P(bufs["x"].ptr + off), P(hx.ctypes.data + off), nb))
            _cabi.check(lib.krn_upload_on(s_in, P(bufs["b"].ptr + off), P(hb.ctypes.data + off), nb))
            for sh in shadows:
                if sh is not None and sh[3]:
                    _cabi.check(lib.krn_upload_on(s_in, P(sh[1].ptr + off), P(sh[0]._host.ctypes.data + off), nb))
            _cabi.check(lib.krn_event_record_on(s_in, P(ev[2 * c])))
            _cabi.check(lib.krn_ctx_wait_event(dev.h, P(ev[2 * c])))
            sx, sb = shadows
            _cabi.check(lib.krn_laplacian_grad(
                dev.h, P(bufs["x"].ptr + off), P(bufs["xo"].ptr + off), P(bufs["b"].ptr + off),
                P(sx[1].ptr + off) if sx else None, P(sb[1].ptr + off) if sb else None,
                int(sx[2]) if sx else 0, int(sb[2]) if sb else 0,
                hi - lo, lo, n, P(d_halo.ptr + 48 * c), float(self.m.seed)))
            dev.record(ev[2 * c + 1])
            _cabi.check(lib.krn_stream_wait_event(s_out, P(ev[2 * c + 1])))
            for sh in shadows:
                if sh is not None:
                    _cabi.check(lib.krn_download_on(s_out, P(sh[0]._host.ctypes.data + off), P(sh[1].ptr + off), nb))
        _cabi.check(lib.krn_stream_sync(s_out))
        dev.sync()
        x._adopt(bufs["xo"])
        b._dev, b._dev_ok = bufs["b"], True
        for sh in shadows:
            if sh is not None:
                v, buf = sh[0], sh[1]
                v._dev, v._dev_ok, v._host_ok, v._zero = buf, True, True, False
        return None


def stream_cuts(n: int, chunk: int) -> list:
    """Row boundaries of the chunks of a streamed call.  Nothing overlaps the upload of the first
    chunk or the download of the last one (1.3 ms each at 64 MB per chunk and direction), so the
    chunks grow from chunk/16 at the front and shrink back to it at the end; boundaries stay
    multiples of 4 rows (256-bit accesses)."""
    if n < 4 * chunk:
        return list(range(0, n, chunk)) + [n]
    ramp = [chunk >> k for k in (4, 3, 2, 1)]
    cuts, at = [0], 0
    for size in ramp:
        at += size
        cuts.append(at)
    tail = sum(ramp)
    while n - at - tail > chunk:
        at += chunk
        cuts.append(at)
    rest = n - at - tail  # 0 < rest <= chunk: one more chunk, cut at a multiple of 4 rows
    if rest > 0:
        at += (rest + 3) // 4 * 4 if rest + 3 < n - at else rest
        cuts.append(min(at, n))
    for size in reversed(ramp):
        at = cuts[-1] + size
        if at >= n:
            break
        cuts.append(at)
    if cuts[-1] != n:
        cuts.append(n)
    return cuts


_signatures = None
_cache: dict = {}


def _load_signatures() -> dict:
    global _signatures
    if _signatures is None:
        prog = parse(open(_PROGRAM).read())
        sigs = {_canon(prog.function(_FN), False)[0]: _Match(False)}
        for wrt in (("x", "b"), ("x",), ("b",)):
            g = differentiate(prog, _FN, wrt).function(_FN + "_grad")
            sigs[_canon(g, True)[0]] = _Match(True, wrt)
        _signatures = sigs
    return _signatures


def match(fn):
    """A runnable for ``fn`` when it is the headline objective / gradient, else None."""
    hit = _cache.get(id(fn))
    if hit is not None and hit[0] is fn:
        return hit[1]
    sigs = _load_signatures()
    out = None
    try:
        for hole in (False, True):
            key, seed = _canon(fn, hole)
            m = sigs.get(key)
            if m is not None:
                out = _Bound(fn, _Match(m.grad, m.wrt, 1.0 if seed is None else seed))
                break
    except TypeError:
        out = None
    _cache[id(fn)] = (fn, out)
    return out
