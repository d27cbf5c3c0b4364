"""Execution of kernel-language functions on a B200.

Drop-in for the reference's ``krn.runtime``
(/root/reference/pkg/src/krn/runtime.py): same names, argument meaning and
error behaviour for ``ViewStorage``, ``ExecutionConfig``, ``execute`` and the
exception classes - but Views live in HBM and every array operation is a CUDA
kernel in libkrn_b200.so (or generated through it).  There is no CPU
execution path: without the library or without a device ``execute`` raises.

Two execution policies (``ExecutionConfig.policy``):

``"fused"`` (default)
    a function whose tree matches the headline objective or its generated
    gradient runs as ONE hand-written kernel (csrc/krn_laplacian.cu); anything
    else falls through to ``"statements"``.
``"statements"``
    every statement is one launch, like the reference (and like Kokkos): bulk
    builtins from the library, ``parallel_for`` bodies generated from the tree
    (codegen.py).  This is the like-for-like granularity for the
    gradient/primal ratio.

Host/device coherence of a View: ``.buffer`` / ``.flat`` hand out the host
array (refreshed from the device when stale) and, because the caller may write
through it, mark the device copy stale; ``.peek()`` reads without invalidating.
"""

from __future__ import annotations

import ctypes as C
import dataclasses as _dc
import os
import struct
import weakref

import numpy as np

from . import _cabi, codegen
from .lang import nodes as N
from .lang.nodes import ViewDescriptor, kind


class ShapeMismatch(ValueError):
    pass


class OutOfBounds(IndexError):
    pass


class NonFiniteDetected(ArithmeticError):
    pass


# ---------------------------------------------------------------------------
# device


class Device:
    """One libkrn_b200 context (device + stream + pool).  ``Device.get()``
    returns the process-wide default for a device ordinal."""

    _default: dict = {}

    def __init__(self, ordinal: int = 0, stream: int = 0):
        self.lib = _cabi.lib()
        self.ordinal = ordinal
        h = C.c_void_p()
        _cabi.check(self.lib.krn_ctx_create(ordinal, C.c_void_p(stream), C.byref(h)))
        self.h = h
        # pinned staging block for small transfers: [0:64) status, [64:...) scalars
        p = C.c_void_p()
        _cabi.check(self.lib.krn_host_alloc(4096, C.byref(p)))
        self._pinned = p
        self.staging = np.frombuffer((C.c_char * 4096).from_address(p.value), dtype=np.uint8)
        sp = C.c_void_p()
        _cabi.check(self.lib.krn_status_device_ptr(self.h, C.byref(sp)))
        self.status_ptr = sp.value
        self._modules: dict = {}

    @classmethod
    def get(cls, ordinal=None) -> "Device":
        if isinstance(ordinal, Device):
            return ordinal
        if ordinal is None:
            ordinal = int(os.environ.get("KRN_DEVICE", os.environ.get("LOCAL_RANK", "0")))
        d = cls._default.get(ordinal)
        if d is None:
            d = cls._default[ordinal] = Device(ordinal)
        return d

    # memory ----------------------------------------------------------------
    def alloc(self, nbytes: int) -> int:
        p = C.c_void_p()
        _cabi.check(self.lib.krn_alloc(self.h, nbytes, C.byref(p)))
        return p.value

    def free(self, ptr: int):
        if ptr:
            self.lib.krn_free(self.h, C.c_void_p(ptr))

    def upload(self, dptr: int, arr: np.ndarray):
        _cabi.check(self.lib.krn_upload(self.h, C.c_void_p(dptr), C.c_void_p(arr.ctypes.data), arr.nbytes))

    def download(self, arr: np.ndarray, dptr: int):
        _cabi.check(self.lib.krn_download(self.h, C.c_void_p(arr.ctypes.data), C.c_void_p(dptr), arr.nbytes))

    def download_async(self, arr: np.ndarray, dptr: int):
        _cabi.check(
            self.lib.krn_download_async(self.h, C.c_void_p(arr.ctypes.data), C.c_void_p(dptr), arr.nbytes)
        )

    def sync(self):
        _cabi.check(self.lib.krn_sync(self.h))

    def launches(self) -> int:
        n = C.c_uint64()
        _cabi.check(self.lib.krn_ctx_launch_count(self.h, C.byref(n)))
        return n.value

    def sm_count(self) -> int:
        n = C.c_int()
        _cabi.check(self.lib.krn_ctx_sm_count(self.h, C.byref(n)))
        return n.value

    # auxiliary streams / scratch for the pipelined host path --------------------
    def aux_stream(self, name: str):
        streams = self.__dict__.setdefault("_aux_streams", {})
        if name not in streams:
            s = C.c_void_p()
            _cabi.check(self.lib.krn_stream_create(self.h, C.byref(s)))
            streams[name] = s
        return streams[name]

    def event_pool(self, count: int) -> list:
        pool = self.__dict__.setdefault("_event_pool", [])
        while len(pool) < count:
            pool.append(self.event())
        return pool[:count]

    def ticket_ptr(self) -> int:
        """Arrival counter for block-level reductions of generated kernels (kept at zero
        between launches: the last block re-arms it)."""
        t = self.__dict__.get("_ticket")
        if t is None:
            t = self.__dict__["_ticket"] = self.alloc(8)
            self.fill(t, 1, 0.0)
        return t

    def pinned_scratch(self, count: int) -> np.ndarray:
        cur = self.__dict__.get("_pinned_scratch")
        if cur is None or cur.size < count:
            cur = self.__dict__["_pinned_scratch"] = pinned_array((max(count, 1024),))
        return cur[:count]

    # events ------------------------------------------------------------------
    def event(self) -> int:
        e = C.c_void_p()
        _cabi.check(self.lib.krn_event_create(C.byref(e)))
        return e.value

    def record(self, event: int):
        _cabi.check(self.lib.krn_event_record(self.h, C.c_void_p(event)))

    def elapsed_ms(self, start: int, stop: int) -> float:
        ms = C.c_float()
        _cabi.check(self.lib.krn_event_elapsed_ms(C.c_void_p(start), C.c_void_p(stop), C.byref(ms)))
        return ms.value

    # builtins (thin) -----------------------------------------------------------
    def fill(self, ptr, n, value=0.0, d_value=0):
        _cabi.check(self.lib.krn_fill(self.h, C.c_void_p(ptr), n, float(value), C.c_void_p(d_value)))

    def copy(self, dst, src, n):
        _cabi.check(self.lib.krn_copy(self.h, C.c_void_p(dst), C.c_void_p(src), n))

    def add_scalar(self, ptr, n, s=0.0, d_s=0):
        _cabi.check(self.lib.krn_add_scalar(self.h, C.c_void_p(ptr), n, float(s), C.c_void_p(d_s)))

    def add_view(self, dst, src, n):
        _cabi.check(self.lib.krn_add_view(self.h, C.c_void_p(dst), C.c_void_p(src), n))

    def reduce_pairwise(self, ptr, n, d_out, accumulate):
        _cabi.check(
            self.lib.krn_reduce_pairwise(self.h, C.c_void_p(ptr), n, C.c_void_p(d_out), int(accumulate))
        )

    def check_finite(self, ptr, n, d_flag):
        _cabi.check(self.lib.krn_check_finite(self.h, C.c_void_p(ptr), n, C.c_void_p(d_flag)))

    def module(self, source: str):
        m = self._modules.get(source)
        if m is None:
            h = C.c_void_p()
            _cabi.check(self.lib.krn_module_compile(self.h, source.encode(), C.byref(h)))
            m = self._modules[source] = h
        return m

    def kernel_info(self, module, name: str) -> tuple:
        """(registers per thread, local bytes per thread, static shared bytes) of a compiled kernel."""
        regs, local, smem = C.c_int(), C.c_int(), C.c_int()
        _cabi.check(self.lib.krn_module_kernel_info(module, name.encode(), C.byref(regs), C.byref(local),
                                                    C.byref(smem)))
        return regs.value, local.value, smem.value


# ---------------------------------------------------------------------------
# View storage


class _DeviceBuffer:
    """Owns one device allocation; returned to the pool when collected."""

    __slots__ = ("dev", "ptr", "nbytes", "__weakref__")

    def __init__(self, dev: Device, nbytes: int):
        self.dev, self.nbytes = dev, nbytes
        self.ptr = dev.alloc(nbytes)

    def __del__(self):
        try:
            self.dev.free(self.ptr)
        except Exception:
            pass


class _PinnedBlock:
    """Owns one cudaMallocHost block; numpy views keep it alive via ``base``."""

    def __init__(self, nbytes: int):
        lib = _cabi.lib()
        p = C.c_void_p()
        _cabi.check(lib.krn_host_alloc(max(nbytes, 8), C.byref(p)))
        self.ptr, self.nbytes, self._lib = p.value, nbytes, lib
        self.raw = (C.c_char * max(nbytes, 8)).from_address(p.value)

    def __del__(self):
        try:
            self._lib.krn_host_free(C.c_void_p(self.ptr))
        except Exception:
            pass


def pinned_array(extents) -> np.ndarray:
    """Zero-filled float64 array in page-locked host memory."""
    shape = tuple(int(e) for e in extents)
    n = int(np.prod(shape)) if shape else 1
    block = _PinnedBlock(8 * n)
    arr = np.frombuffer(block.raw, dtype=np.float64, count=n).reshape(shape)
    arr[...] = 0.0
    # numpy keeps `block.raw` alive through arr.base; tie the block's lifetime to it
    block.raw._owner = block
    return arr


class ViewStorage:
    """A rank-1 or rank-2 float64 View with reference semantics, resident in
    HBM (reference: runtime.py:74-115).

    State: ``_host`` (ndarray or None), ``_dev`` (_DeviceBuffer or None) and
    which of them is current.  ``_zero`` marks a View known to hold +0.0
    everywhere with no storage touched yet (``ViewStorage.zeros`` provenance):
    the fused gradient kernel skips reading such a shadow.
    """

    __slots__ = ("descriptor", "_shape", "_host", "_dev", "_host_ok", "_dev_ok", "_zero")

    def __init__(self, descriptor, buffer):
        buffer = np.asarray(buffer)
        if buffer.dtype != np.float64 or not buffer.flags.c_contiguous:
            buffer = np.ascontiguousarray(buffer, dtype=np.float64)
        if buffer.ndim != descriptor.rank:
            raise ShapeMismatch(
                f"view '{descriptor.name}': rank {descriptor.rank} descriptor, rank {buffer.ndim} data"
            )
        self.descriptor = descriptor
        self._shape = tuple(buffer.shape)
        self._host = buffer
        self._dev = None
        self._host_ok, self._dev_ok, self._zero = True, False, False

    # -- construction -----------------------------------------------------------
    @classmethod
    def _blank(cls, name, extents) -> "ViewStorage":
        self = object.__new__(cls)
        self._shape = tuple(int(e) for e in extents)
        self.descriptor = ViewDescriptor(name, rank=len(self._shape))
        self._host = self._dev = None
        self._host_ok = self._dev_ok = False
        self._zero = False
        return self

    @classmethod
    def zeros(cls, name: str, extents) -> "ViewStorage":
        self = cls._blank(name, extents)
        self._zero = True
        return self

    @classmethod
    def from_values(cls, name: str, values) -> "ViewStorage":
        arr = np.array(values, dtype=np.float64, order="C")
        return cls(ViewDescriptor(name, rank=arr.ndim), arr)

    @classmethod
    def pinned(cls, name: str, extents, zero: bool = False) -> "ViewStorage":
        """A View whose host array lives in page-locked memory (zero filled), so
        host<->device copies run at full PCIe speed and asynchronously.  ``zero=True``
        additionally records the zeros provenance (like ``ViewStorage.zeros``): kernels
        that can exploit a known-zero shadow skip its upload and its read."""
        self = cls(ViewDescriptor(name, rank=len(tuple(extents))), pinned_array(extents))
        self._zero = bool(zero)
        return self

    def mark_zero(self):
        """Declare that the host array has been refilled with +0.0 by the caller."""
        self._host_ok, self._dev_ok, self._zero = True, False, True

    def copy(self) -> "ViewStorage":
        out = ViewStorage._blank(self.descriptor.name, self._shape)
        out.descriptor = self.descriptor
        if self._zero:
            out._zero = True
        elif self._dev_ok:
            out._dev = _DeviceBuffer(self._dev.dev, self.nbytes)
            self._dev.dev.copy(out._dev.ptr, self._dev.ptr, self.size)
            out._dev_ok = True
        else:
            out._host = self._host.copy()
            out._host_ok = True
        return out

    # -- shape --------------------------------------------------------------------
    @property
    def extents(self) -> tuple:
        return self._shape

    @property
    def name(self) -> str:
        return self.descriptor.name

    @property
    def size(self) -> int:
        n = 1
        for e in self._shape:
            n *= e
        return n

    @property
    def nbytes(self) -> int:
        return 8 * self.size

    # -- host side -------------------------------------------------------------------
    def _sync_host(self):
        if self._host is None:
            self._host = np.zeros(self._shape, dtype=np.float64)
            if self._zero:
                self._host_ok = True
        elif self._zero and not self._host_ok:
            self._host.fill(0.0)
            self._host_ok = True
        if not self._host_ok:
            self._dev.dev.download(self._host, self._dev.ptr)
            self._host_ok = True

    def peek(self) -> np.ndarray:
        """Current contents as a read-only host array; the device copy stays valid."""
        self._sync_host()
        out = self._host.view()
        out.flags.writeable = False
        return out

    @property
    def buffer(self) -> np.ndarray:
        """The host array (same object on every call).  The caller may write
        through it, so the device copy is considered stale afterwards."""
        self._sync_host()
        self._dev_ok = False
        self._zero = False
        return self._host

    @property
    def flat(self) -> np.ndarray:
        return self.buffer.reshape(-1)

    # -- device side ---------------------------------------------------------------------
    def device_ptr(self, dev: Device, *, write: bool = True, discard: bool = False) -> int:
        """Device pointer with current contents (``discard``: contents will be
        fully overwritten, skip upload / zero fill).  ``write`` marks the host
        copy stale."""
        if self._dev is None or self._dev.dev is not dev:
            if self._dev is not None and self._dev_ok and not self._host_ok:
                self._sync_host()
            self._dev = _DeviceBuffer(dev, self.nbytes)
            self._dev_ok = False
        if not self._dev_ok and not discard:
            if self._zero:
                dev.fill(self._dev.ptr, self.size, 0.0)
            else:
                dev.upload(self._dev.ptr, self._host)
        self._dev_ok = True
        if write or discard:
            self._host_ok = False
            self._zero = False
        return self._dev.ptr

    def _adopt(self, buf: _DeviceBuffer):
        """Replace the device storage (out-of-place kernels swap buffers)."""
        self._dev = buf
        self._dev_ok, self._host_ok, self._zero = True, False, False

    def __repr__(self) -> str:
        return f"ViewStorage({self.name!r}, shape={self._shape})"


# ---------------------------------------------------------------------------
# configuration / results


@_dc.dataclass
class ExecutionConfig:
    """Reference fields (runtime.py:118-128) plus the GPU knobs.  ``threads``
    is accepted for compatibility and ignored: iterations map to CUDA threads."""

    threads: int = 1
    deterministic_reduction: bool = True
    conflict_detect: bool = False
    rng_seed: int = 0
    check_finite: bool = False
    policy: str = "fused"  # "fused" | "statements"
    device: object = None  # device ordinal or Device; None = KRN_DEVICE / LOCAL_RANK / 0
    # False: enqueue only (no host sync, no status check, value not fetched); for timing
    # the launch sequence with events.  The reference contract is synchronous.
    synchronous: bool = True
    # True: when the Views of a recognised gradient call live on the host, cut the rows into
    # chunks and overlap upload / kernel / download of the shadows (fused.run_streamed)
    stream_host_io: bool = False
    # how atomic_add contributions to non-injective targets are accumulated (generated kernels):
    # "ordered" the reference's own order - queue sorted by (iteration, program order), applied as a
    # left fold per location (runtime.py:615-620) - through a stable radix sort by target and a
    # segmented in-order fold (csrc/krn_ordered.cu): bit-identical to the reference, identical from
    # run to run; "red" hardware fp64 reductions, "warp" warp-aggregated, "lead" leader-aggregated,
    # "smem" block-privatised in shared memory (targets of <= 6144 elements): exact up to
    # reassociation (relative 1e-12).  "auto" = "ordered" when deterministic_reduction is set (the
    # reference's default and its determinism contract), else smem for small hot
    # targets and lead for the rest
    atomic_policy: str = "auto"
    # fusion pass: also merge statements across neighbour dependencies (a stencil after an in-place
    # update, deferred atomics and the rows they land on) by recomputing the few halo iterations
    # each warp needs (tilegen.window_kernel); False = only pointwise fusion
    fuse_neighbours: bool = True

    def __post_init__(self):
        if self.threads < 1:
            raise ValueError("threads must be >= 1")
        if self.policy not in ("fused", "compiled", "statements"):
            raise ValueError("policy must be 'fused', 'compiled' or 'statements'")
        if self.atomic_policy not in ("auto", "ordered", "red", "warp", "smem", "lead"):
            raise ValueError("atomic_policy must be 'auto', 'ordered', 'red', 'warp', 'smem' or 'lead'")


def effective_threads(cfg: ExecutionConfig) -> int:
    env = os.environ.get("KRN_THREADS")
    return max(1, int(env)) if env else cfg.threads


@_dc.dataclass(frozen=True)
class ConflictRecord:
    kernel: int
    view: str
    offset: int
    iterations: tuple
    kinds: tuple


@_dc.dataclass(frozen=True)
class ConflictReport:
    records: tuple = ()

    def __bool__(self) -> bool:
        return bool(self.records)

    def write_write(self) -> tuple:
        return tuple(r for r in self.records if "write" in r.kinds)


@_dc.dataclass
class ExecResult:
    value: object
    conflicts: object = None


# ---------------------------------------------------------------------------
# statement-granular plan


class _Plan:
    """Compiled form of one function: generated module + step list."""

    def __init__(self, fn, trace: bool = False):
        self.fn = fn
        b = self.builder = codegen.ModuleBuilder(fn)
        self.steps: list = []
        bound = {p.name for p in fn.params if not p.is_view}
        run: list = []

        def flush():
            if run:
                self.steps.append(("scalars", b.scalar_block(list(run), f"s{len(self.steps)}")))
                run.clear()

        for s in fn.body:
            k = kind(s)
            if k in codegen._ELEMENT:
                run.append(s)
                if k == "DeclScalar":
                    bound.add(s.name)
                continue
            flush()
            if k == "DeclView":
                self.steps.append(("declview", s))
            elif k == "ParallelFor":
                recipe = b.kernel(s, f"k{len(self.steps)}")
                # iterations that may touch one location with a plain write among the accesses: the
                # result depends on their order (see _Run.do_kernel)
                recipe["carried"] = codegen.carries_across_iterations(s)
                if trace or recipe["carried"]:
                    # conflict detector: a dry, access-tagging replay precedes the kernel
                    recipe["trace"] = b.kernel_trace(s, f"k{len(self.steps)}_t")
                self.steps.append(("kernel", s, recipe))
            elif k == "DeepCopy":
                self.steps.append(("deepcopy", s))
            elif k == "ParallelSum":
                self.steps.append(("gather", s, s.dst in bound))
                bound.add(s.dst)
                b.slot(s.dst)
            elif k == "ParallelSumInto":
                self.steps.append(("suminto", s))
            elif k == "Return":
                self.steps.append(("return", b.return_block(s.value, f"r{len(self.steps)}")))
            else:
                raise TypeError(f"cannot execute {k}")
        flush()
        self.source = b.source()
        self.nslots = max(len(b.slots), 1) + 1
        self.carried = any(st[0] == "kernel" and st[2]["carried"] for st in self.steps)


_plans: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()
_plans_by_id: dict = {}


def _plan_for(fn, trace: bool = False) -> _Plan:
    key = (id(fn), trace)
    hit = _plans_by_id.get(key)
    if hit is not None and hit[0] is fn:
        return hit[1]
    plan = _Plan(fn, trace)
    _plans_by_id[key] = (fn, plan)  # holds fn alive so the id stays unique
    return plan


SMEM_PRIVATE_MAX = 6144  # doubles: 48 KB of dynamic shared memory


NO_ATOMICS = (0, 0, 0, 0, 0, 0)
ENV_TAIL = "qiiQQqQ"  # Env: priv_rows, apol, priv_vid, okeys, ovals, on, fin (codegen._PREAMBLE)
ORDERED_LIMIT = 1 << 31  # 32-bit keys and record numbers (krn_ordered_accumulate)


class OrderedStage:
    """Queue of one launch's deferred atomic_add records under the ordered policy: the kernel
    writes (target offset, values) per site group at record = iteration * groups + group
    (codegen.assign_ordered), `apply` hands each target's queue to krn_ordered_accumulate."""

    def __init__(self, dev: Device, entries, views: dict, n: int):
        self.dev, self.entries, self.views, self.n = dev, entries, views, n
        groups = sum(e["groups"] for e in entries)
        self.keys = _DeviceBuffer(dev, 4 * n * groups)
        self.vals = _DeviceBuffer(dev, 8 * n * sum(e["groups"] * e["width"] for e in entries))
        # all-ones key = "this site did not execute" (guarded sites, iterations that failed a check)
        _cabi.check(dev.lib.krn_memset(dev.h, C.c_void_p(self.keys.ptr), 0xFF, 4 * n * groups))
        for e in entries:  # values of guarded sites that do not execute are never written: defined, not garbage
            if e.get("guarded"):
                _cabi.check(dev.lib.krn_memset(dev.h, C.c_void_p(self.vals.ptr + 8 * e["val_off"] * n), 0,
                                               8 * n * e["groups"] * e["width"]))

    @staticmethod
    def feasible(entries, views: dict, n: int) -> bool:
        return all(views[e["view"]].size <= ORDERED_LIMIT and n * e["groups"] < ORDERED_LIMIT for e in entries)

    def apply(self):
        dev, n = self.dev, self.n
        for e in self.entries:
            v = self.views[e["view"]]
            keys = C.c_void_p(self.keys.ptr + 4 * e["key_off"] * n)
            vals = C.c_void_p(self.vals.ptr + 8 * e["val_off"] * n)
            if e.get("cols"):  # row records of a rank-2 target: key = row, one value plane per literal column
                cols = (C.c_int * len(e["cols"]))(*e["cols"])
                _cabi.check(dev.lib.krn_ordered_accumulate_rows(
                    dev.h, C.c_void_p(v.device_ptr(dev)), v.extents[0], v.extents[1], cols, len(e["cols"]), keys, vals,
                    n * e["groups"]))
            else:
                _cabi.check(dev.lib.krn_ordered_accumulate(dev.h, C.c_void_p(v.device_ptr(dev)), v.size, keys, vals,
                                                           n * e["groups"], e["width"]))


def atomic_choice(dev, cfg, recipe, views, builder, n, static_smem: int = 0):
    """(Env tail, OrderedStage or None): how a kernel accumulates its hardware-atomic
    atomic_add sites.  Env tail = (privatised rows, policy, privatised view id, key queue,
    value queue, trip count)."""
    entries = recipe.get("ordered") or []
    want = cfg.atomic_policy
    if entries and n > 0 and (want == "ordered" or (want == "auto" and cfg.deterministic_reduction)):
        if OrderedStage.feasible(entries, views, n):
            stage = OrderedStage(dev, entries, views, n)
            return (0, 4, 0, stage.keys.ptr, stage.vals.ptr, n), stage
        if want == "ordered":
            raise ValueError("atomic_policy='ordered' needs targets and queues of at most 2^31 entries")
    if want in ("ordered", "auto") and cfg.deterministic_reduction and entries:
        want = "lead"  # targets beyond 32-bit keys: hardware reductions, exact up to reassociation
    atomic_views = recipe.get("atomic_views") or []
    if not atomic_views:
        return NO_ATOMICS, None
    name = atomic_views[0]
    rows = views[name].size
    if want in ("auto", "ordered"):
        # measured (tools/atomic_policies.py, profiles/r1_atomic_policies.json): privatisation wins by
        # 2-20x on small targets; leader aggregation costs nothing on spread-out targets and removes
        # the same-address serialisation of a hot row
        want = "smem" if (0 < rows <= SMEM_PRIVATE_MAX and n >= 4 * rows) else "lead"
    if want == "smem" and not (0 < rows <= SMEM_PRIVATE_MAX):
        want = "red"
    if want == "smem" and 8 * rows + static_smem > 48 * 1024:
        # the kernel's own shared memory (windows, reduction scratch) and the privatised rows
        # together exceed what a launch gets without opting in: aggregate in the warp instead
        want = "lead"
    return (rows, {"red": 0, "warp": 1, "smem": 2, "lead": 3}[want], builder.vid(name), 0, 0, 0), None


def _scalar_src(dev, plan, S, src):
    """(host value, device pointer) for a Literal / ScalarVar bulk operand."""
    if kind(src) == "Literal":
        return float(src.value), 0
    return 0.0, S + 8 * plan.builder.slot(src.name)


def _index_value(e, views) -> int:
    """Host evaluation of a view-free index expression (extents are host data)."""
    k = kind(e)
    if k == "IntLiteral":
        return e.value
    if k == "Extent":
        return views[e.view].extents[e.dim]
    if k == "IdxBinary":
        a, b = _index_value(e.lhs, views), _index_value(e.rhs, views)
        return a + b if e.op == "+" else a - b if e.op == "-" else a * b
    raise TypeError(f"index expression is not host-evaluable: {kind(e)}")


class _Run:
    """One call of a function under the statement policy."""

    def __init__(self, dev: Device, plan: _Plan, views: dict, scalars: dict, cfg):
        self.dev, self.plan, self.views, self.cfg = dev, plan, views, cfg
        self.b = plan.builder
        self.mod = dev.module(plan.source)
        nslots = plan.nslots
        self.S = _DeviceBuffer(dev, 8 * nslots)
        init = np.zeros(nslots)
        for name, v in scalars.items():
            init[self.b.slot(name)] = v
        host = dev.staging[64 : 64 + 8 * nslots].view(np.float64) if 8 * nslots <= 4096 - 64 else init
        host[:] = init
        dev.upload(self.S.ptr, host)
        _cabi.check(dev.lib.krn_status_reset(dev.h))
        self.kernel_index = 0
        self.conflicts: list = []

    def env(self, atomic=NO_ATOMICS) -> bytes:
        nv = max(len(self.b.views), 1)
        ptrs, e0, e1 = [0] * nv, [0] * nv, [0] * nv
        for i, name in enumerate(self.b.views):
            v = self.views.get(name)
            if v is not None:
                ptrs[i] = v.device_ptr(self.dev)
                e0[i] = v.extents[0]
                e1[i] = v.extents[1] if len(v.extents) == 2 else 1
        nh = max(len(self.b.hslots), 1)  # Env.H: unused on the statement path, but part of the layout
        return struct.pack(f"{nv}Q{nv}q{nv}qQQ{nh}d" + ENV_TAIL, *ptrs, *e0, *e1, self.S.ptr, self.dev.status_ptr,
                           *([0.0] * nh), *atomic, 0)

    def launch(self, name: str, n: int, extra=(), atomic=NO_ATOMICS, sequential=False):
        env = C.create_string_buffer(self.env(atomic))
        holders = [env]
        args = [C.addressof(env)]
        for x in extra:
            h = C.c_longlong(x) if isinstance(x, int) else x
            holders.append(h)
            args.append(C.addressof(h))
        arr = (C.c_void_p * len(args))(*args)
        shared = 8 * atomic[0] if atomic[1] == 2 else 0
        if sequential:  # one thread: the grid-stride loop of the kernel runs iterations 0..n-1 in order
            _cabi.check(self.dev.lib.krn_module_launch_exact(self.dev.h, self.mod, name.encode(), 1, 1, shared, arr))
            return
        _cabi.check(self.dev.lib.krn_module_launch(self.dev.h, self.mod, name.encode(), n, shared, arr))

    def go(self):
        for step in self.plan.steps:
            getattr(self, "do_" + step[0])(*step[1:])
        return self.finish()

    # -- steps ----------------------------------------------------------------------
    def do_declview(self, s):
        args = iter(s.dyn_args)
        dims = [
            e.size if kind(e) == "StaticExtent" else int(_index_value(next(args), self.views))
            for e in s.descriptor.extents
        ]
        if any(d < 0 for d in dims):
            raise ShapeMismatch(f"view '{s.name}': negative extent {dims}")
        self.views[s.name] = ViewStorage.zeros(s.name, dims)

    def do_scalars(self, recipe):
        self.launch(recipe["name"], 1)
        self.guard()

    def do_kernel(self, loop, recipe):
        n = int(_index_value(loop.upper, self.views))
        stage = ostage = None
        extra = [max(n, 0), C.c_void_p(0), C.c_void_p(0)]
        if recipe["n_staged"] and n > 0:
            stage = _DeviceBuffer(self.dev, 8 * recipe["n_staged"] * n)
            extra[1] = C.c_void_p(stage.ptr)
            if recipe["needs_offsets"]:
                ostage = _DeviceBuffer(self.dev, 8 * recipe["n_staged"] * n)
                extra[2] = C.c_void_p(ostage.ptr)
        sequential = False
        if n > 0 and self.cfg.conflict_detect:
            # a kernel with conflicts then runs in iteration order (deterministic: the values of the
            # reference's plain threads=1 run; its instrumented run uses a seeded shuffle instead)
            sequential = self.trace_kernel(recipe["trace"], n) > 0
        elif n > 1 and recipe["carried"]:
            # Order-dependent as far as the index expressions tell.  The reference (threads=1, its
            # default) runs iterations 0..n-1 one after the other (runtime.py:586-593) and its
            # tests rely on that (a scan through v(i) = v(i-1) + i, tests/test_runtime.py:101-115).
            # The tag replay decides on the actual indices: no location shared between two
            # iterations with a plain write -> any order gives the same result, run in parallel;
            # otherwise run the kernel on ONE thread, in order - slow, and exactly the reference.
            sequential = self.trace_kernel(recipe["trace"], n, collect=False) > 0
        if n > 0:
            choice, ordered = (NO_ATOMICS, None) if sequential else atomic_choice(self.dev, self.cfg, recipe, self.views, self.b, n)
            self.launch(recipe["name"], n, extra, choice, sequential=sequential)
            for ap in recipe["apply"]:
                if ordered is not None and ap["over"] == "iterations":
                    continue  # the staged contributions went to the ordered queue instead
                count = self.views[ap["view"]].extents[0] if ap["over"] == "rows" else n
                if count > 0:
                    self.launch(ap["name"], count, extra)
            if ordered is not None:
                ordered.apply()
        self.kernel_index += 1
        self.guard()

    # -- conflict detector -----------------------------------------------------------------
    TRIPLES_FIRST = 1 << 18  # triples the first collect pass has room for (6 MB)

    def trace_kernel(self, recipe, n: int, collect: bool = True) -> int:
        """Reference: _Tracer + the instrumented replay of parallel_for (runtime.py:198-227,
        574-585): one record per location touched by two or more distinct iterations of this
        kernel with a plain write among the accesses.  Here: a dry replay of the kernel tags
        every location it touches (codegen._TRACE); if any location turned into a conflict a
        second replay lists the iterations that touch those locations.  Both replays read the
        Views as they are BEFORE the kernel and store nothing; the real kernel runs afterwards."""
        dev, b = self.dev, self.b
        nv = max(len(b.views), 1)
        tags, tag_ptrs = [], [0] * nv
        for name in recipe["views"]:
            v = self.views.get(name)
            if v is None or v.size == 0:
                continue
            v.device_ptr(dev, write=False)  # materialise lazily zero Views: the replay loads from them
            buf = _DeviceBuffer(dev, 8 * v.size)
            dev.fill(buf.ptr, v.size, 0.0)
            tags.append(buf)
            tag_ptrs[b.vid(name)] = buf.ptr
        counts = _DeviceBuffer(dev, 16)
        dev.fill(counts.ptr, 2, 0.0)
        host = np.zeros(2, dtype=np.uint64)

        def replay(phase, triples_ptr, cap):
            tr = C.create_string_buffer(struct.pack(f"{nv}QQQqi4x", *tag_ptrs, counts.ptr, triples_ptr, cap, phase))
            self.launch(recipe["name"], n, [n, tr])
            self.read_status()  # an access out of bounds fails here exactly as it would in the kernel
            dev.download(host, counts.ptr)

        replay(0, 0, 0)
        conflicts = int(host[0])
        if conflicts == 0 or not collect:
            return conflicts
        cap = self.TRIPLES_FIRST
        while True:
            triples = _DeviceBuffer(dev, 24 * cap)
            dev.fill(counts.ptr + 8, 1, 0.0)
            replay(1, triples.ptr, cap)
            produced = int(host[1])
            if produced <= cap:
                break
            cap = produced
        rows = np.zeros((produced, 3), dtype=np.int64)
        dev.download(rows, triples.ptr)
        if produced == 0:
            return conflicts
        # sort by (view, offset, iteration) and drop repeats (an iteration may touch a location
        # several times); offsets stay below 2^40 elements, so (view, offset) is one 64-bit key
        key = ((rows[:, 0] & 0xFFFFFFFF) << 40) | rows[:, 1]
        order = np.lexsort((rows[:, 2], key))
        rows, key = rows[order], key[order]
        keep = np.ones(len(rows), dtype=bool)
        keep[1:] = (key[1:] != key[:-1]) | (rows[1:, 2] != rows[:-1, 2])
        rows, key = rows[keep], key[keep]
        kinds_of = [tuple(sorted(k for bit, k in enumerate(("read", "write", "atomic")) if mask >> bit & 1))
                    for mask in range(8)]
        cuts = np.flatnonzero(key[1:] != key[:-1]) + 1
        starts = [0, *cuts.tolist(), len(rows)]
        head, offs, its = rows[:, 0].tolist(), rows[:, 1].tolist(), rows[:, 2].tolist()
        found = [
            ConflictRecord(self.kernel_index, b.views[head[lo] & 0xFFFFFFFF], offs[lo], tuple(its[lo:hi]),
                           kinds_of[head[lo] >> 32])
            for lo, hi in zip(starts[:-1], starts[1:])
        ]
        found.sort(key=lambda r: (r.view, r.offset))  # the reference sorts its log by (view, offset)
        self.conflicts.extend(found)
        return conflicts

    def do_deepcopy(self, s):
        d = self.views[s.dst]
        if isinstance(s.src, str):
            src = self.views[s.src]
            if d.extents != src.extents:
                raise ShapeMismatch(f"deep_copy: {s.dst}{d.extents} vs {s.src}{src.extents}")
            self.dev.copy(d.device_ptr(self.dev, discard=True), src.device_ptr(self.dev, write=False), d.size)
        else:
            value, dptr = _scalar_src(self.dev, self.plan, self.S.ptr, s.src)
            self.dev.fill(d.device_ptr(self.dev, discard=True), d.size, value, dptr)
        self.guard()

    def do_gather(self, s, accumulate):
        src = self.views[s.src]
        out = self.S.ptr + 8 * self.b.slot(s.dst)
        self.dev.reduce_pairwise(src.device_ptr(self.dev, write=False), src.size, out, accumulate)
        if self.cfg.check_finite:
            self.guard_scalar(self.b.slot(s.dst))

    def do_suminto(self, s):
        d = self.views[s.dst]
        if isinstance(s.src, str):
            src = self.views[s.src]
            if d.extents != src.extents:
                raise ShapeMismatch(f"parallel_sum: {s.dst}{d.extents} vs {s.src}{src.extents}")
            self.dev.add_view(d.device_ptr(self.dev), src.device_ptr(self.dev, write=False), d.size)
        else:
            value, dptr = _scalar_src(self.dev, self.plan, self.S.ptr, s.src)
            self.dev.add_scalar(d.device_ptr(self.dev), d.size, value, dptr)
        self.guard()

    def do_return(self, recipe):
        self.launch(recipe["name"], 1)
        self.ret_slot = recipe["slot"]

    ret_slot = None

    # -- sync points -------------------------------------------------------------------
    def read_status(self):
        st = self.dev.staging[:64].view(np.int64)
        self.dev.download(st, self.dev.status_ptr)
        if st[0] != 0:
            raise self.error_from(st.copy())

    def error_from(self, st):
        code, line, vid, i0, i1 = (int(x) for x in st[:5])
        name = self.b.views[vid] if 0 <= vid < len(self.b.views) else "?"
        view = self.views.get(name)
        if code == _cabi.KRN_ST_OUT_OF_BOUNDS:
            if view is not None and len(view.extents) == 2:
                n0, n1 = view.extents
                return OutOfBounds(f"line {line}: {name}({i0}, {i1}) outside extents {n0}x{n1}")
            n0 = view.extents[0] if view is not None else "?"
            return OutOfBounds(f"line {line}: {name}({i0}) outside extent {n0}")
        if code == _cabi.KRN_ST_BAD_INDEX:
            if i0:  # infinite
                return OverflowError("cannot convert float infinity to integer")
            return ValueError("cannot convert float NaN to integer")
        return RuntimeError(f"device status {code}")

    def guard(self):
        """check_finite: trap after every kernel / bulk statement (runtime.py:669-672)."""
        if not self.cfg.check_finite:
            return
        self.read_status()
        live = [(n, v) for n, v in self.views.items() if v.size]
        words = (len(live) + 1) // 2 + 1
        flags = _DeviceBuffer(self.dev, 8 * words)
        self.dev.fill(flags.ptr, words, 0.0)
        for i, (_, v) in enumerate(live):
            self.dev.check_finite(v.device_ptr(self.dev, write=False), v.size, flags.ptr + 4 * i)
        host = np.zeros(max(len(live), 1), dtype=np.int32)
        self.dev.download(host, flags.ptr)
        for i, (name, _) in enumerate(live):
            if host[i]:
                raise NonFiniteDetected(f"non-finite value in view '{name}'")

    def guard_scalar(self, slot):
        v = np.zeros(1)
        self.dev.download(v, self.S.ptr + 8 * slot)
        if not np.isfinite(v[0]):
            raise NonFiniteDetected(f"non-finite scalar {float(v[0])!r}")

    def finish(self):
        value = None
        if self.ret_slot is not None:
            out = self.dev.staging[64:72].view(np.float64)
            self.dev.download_async(out, self.S.ptr + 8 * self.ret_slot)
        if not self.cfg.synchronous:
            return None
        self.read_status()  # synchronises the stream
        if self.ret_slot is not None:
            value = float(self.dev.staging[64:72].view(np.float64)[0])
            if self.cfg.check_finite and not np.isfinite(value):
                raise NonFiniteDetected(f"non-finite scalar {value!r}")
        return value


# ---------------------------------------------------------------------------
# entry points


def _bind(fn, inputs: dict):
    """Parameter binding with the reference's checks and messages (runtime.py:481-511)."""
    want, got = {p.name for p in fn.params}, set(inputs)
    if want != got:
        parts = []
        if want - got:
            parts.append(f"missing {sorted(want - got)}")
        if got - want:
            parts.append(f"unexpected {sorted(got - want)}")
        raise ShapeMismatch(f"inputs do not match parameters: {'; '.join(parts)}")
    views, scalars = {}, {}
    for p in fn.params:
        v = inputs[p.name]
        if p.is_view:
            if not isinstance(v, ViewStorage):
                v = ViewStorage.from_values(p.name, v)
                inputs[p.name] = v
            if len(v.extents) != p.type.rank:
                raise ShapeMismatch(
                    f"parameter '{p.name}': rank {p.type.rank} expected, got rank {len(v.extents)}"
                )
            for dim, ext in enumerate(p.type.extents):
                if kind(ext) == "StaticExtent" and v.extents[dim] != ext.size:
                    raise ShapeMismatch(
                        f"parameter '{p.name}' dim {dim}: static extent {ext.size} expected, "
                        f"got {v.extents[dim]}"
                    )
            views[p.name] = v
        else:
            scalars[p.name] = float(v)
    return views, scalars


def _pure_element(stmts) -> bool:
    return all(kind(s) in codegen._ELEMENT and (kind(s) != "If" or _pure_element(s.body)) for s in stmts)


class _Extents:
    __slots__ = ("extents",)

    def __init__(self, extents):
        self.extents = extents


_specialised: dict = {}


def _specialise(fn, views: dict):
    """Function-scope `if` blocks whose body holds more than element statements (a parallel_for,
    a bulk builtin, a View declaration): the reference simply executes the body when the condition
    holds (runtime.py:548-550).  Conditions are index comparisons over extents and literals - host
    data - so they are decided here and the taken bodies spliced into a straight-line function,
    which every execution policy then plans as usual (memoised per function and outcome)."""
    if not any(kind(s) == "If" and not _pure_element(s.body) for s in fn.body):
        return fn
    ext = {k: _Extents(v.extents) for k, v in views.items()}
    outcomes: list = []

    def walk(body):
        out = []
        for s in body:
            k = kind(s)
            if k == "DeclView":
                try:
                    args = iter(s.dyn_args)
                    ext[s.name] = _Extents(tuple(e.size if kind(e) == "StaticExtent" else int(_index_value(next(args), ext))
                                                 for e in s.descriptor.extents))
                except (TypeError, KeyError):
                    pass
            if k == "If" and not _pure_element(s.body):
                a, b = _index_value(s.cond.lhs, ext), _index_value(s.cond.rhs, ext)
                taken = {"<": a < b, "<=": a <= b, ">": a > b, ">=": a >= b, "==": a == b, "!=": a != b}[s.cond.op]
                outcomes.append(taken)
                if taken:
                    out.extend(walk(s.body))
                continue
            out.append(s)
        return out

    body = walk(fn.body)
    key = (id(fn), tuple(outcomes))
    hit = _specialised.get(key)
    if hit is not None and hit[0] is fn:
        return hit[1]
    new = _dc.replace(fn, body=tuple(body))
    _specialised[key] = (fn, new)
    return new


def execute(program, fn_name: str, inputs: dict, cfg: ExecutionConfig | None = None) -> ExecResult:
    """Run ``fn_name`` on the GPU.  View inputs are mutated in place (their
    device storage is; ``.buffer`` shows the result).  Synchronous, like the
    reference (runtime.py:689-706)."""
    from . import fused

    cfg = cfg or ExecutionConfig()
    fn = program.function(fn_name)
    if fn is None:
        raise KeyError(f"no function named '{fn_name}'")
    views, scalars = _bind(fn, inputs)
    fn = _specialise(fn, views)
    dev = Device.get(cfg.device)
    if cfg.conflict_detect:
        # statement granularity (a kernel of the report = a parallel_for of the source), every
        # kernel preceded by its access-tagging replay
        run = _Run(dev, _plan_for(fn, trace=True), views, scalars, _dc.replace(cfg, synchronous=True))
        value = run.go()
        return ExecResult(value, ConflictReport(tuple(run.conflicts)))
    if cfg.policy == "fused" and not cfg.check_finite:
        hit = fused.match(fn)
        if hit is not None and hit.applicable(views):
            return ExecResult(hit.run(dev, views, scalars, cfg))
    plan = _plan_for(fn)
    if cfg.policy in ("fused", "compiled") and not plan.carried and (cfg.synchronous or not cfg.check_finite):
        # check_finite stays on the fused path: the kernels test what their statements leave behind and
        # the reference's checks are replayed from the recorded flags (compiled.finite_replay); a function
        # with a statement no fused kernel can watch takes the statement path inside compiled.run
        from . import compiled

        return ExecResult(compiled.run(dev, fn, views, scalars, cfg))
    return ExecResult(_Run(dev, plan, views, scalars, cfg).go())


def detect_conflicts(program, fn_name: str, inputs: dict, cfg: ExecutionConfig | None = None):
    """Every location touched by two distinct iterations of one kernel where at least one access
    is a plain (non-atomic) write (reference: runtime.py:709-726).  The reference replays each
    kernel sequentially in a shuffled order and logs every access in a dictionary; here a dry
    replay of the kernel on the device tags the locations (`_Run.trace_kernel`).  The function is
    executed as well (inputs are mutated, like the reference's instrumented run); a kernel with
    conflicts runs in iteration order, so a racy program leaves the values of the reference's plain
    threads=1 run rather than those of its seeded shuffle; the report is the same."""
    base = cfg or ExecutionConfig()
    cfg = _dc.replace(base, conflict_detect=True, policy="statements", synchronous=True)
    return execute(program, fn_name, inputs, cfg).conflicts


def pairwise_sum(values) -> float:
    """The reference's fixed-tree sum (runtime.py:166-177), evaluated on the device."""
    a = np.ascontiguousarray(values, dtype=np.float64).reshape(-1)
    if a.size == 0:
        return 0.0
    dev = Device.get()
    v = ViewStorage.from_values("v", a)
    out = _DeviceBuffer(dev, 8)
    dev.reduce_pairwise(v.device_ptr(dev, write=False), a.size, out.ptr, False)
    host = np.zeros(1)
    dev.download(host, out.ptr)
    return float(host[0])


# ---------------------------------------------------------------------------
# tensor files (host-side text format of the reference, runtime.py:733-757)


def save_tensor(path, storage: ViewStorage) -> None:
    data = storage.peek()
    with open(path, "w", encoding="utf-8") as f:
        f.write("f64 %d %s\n" % (data.ndim, " ".join(str(d) for d in data.shape)))
        for x in data.reshape(-1):
            f.write(repr(float(x)) + "\n")


def load_tensor(path, name: str | None = None) -> ViewStorage:
    with open(path, "r", encoding="utf-8") as f:
        header = f.readline().split()
        if len(header) < 3 or header[0] != "f64":
            raise ShapeMismatch(f"{path}: malformed tensor header {header!r}")
        rank = int(header[1])
        dims = [int(d) for d in header[2 : 2 + rank]]
        if len(dims) != rank or rank not in (1, 2):
            raise ShapeMismatch(f"{path}: bad rank/extents {header!r}")
        tokens = f.read().split()
    data = np.array(tokens, dtype=np.float64) if tokens else np.zeros(0)
    if data.size != int(np.prod(dims)):
        raise ShapeMismatch(f"{path}: expected {int(np.prod(dims))} values, found {data.size}")
    if name is None:
        name = os.path.splitext(os.path.basename(path))[0]
    return ViewStorage.from_values(name, data.reshape(dims))
