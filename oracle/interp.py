"""TEST INFRASTRUCTURE - CPU oracle, not product code.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
legs may import this module.  The product path (``paper_2507_13204_b200``)
never does, and fails loudly when its CUDA library is missing.

What it is: a plain sequential restatement, in Python + numpy, of the
reference interpreter's semantics for executing a kernel-language function
(/root/reference/pkg/src/krn/runtime.py).  Parity status: PINNED - checked
against (a) the reference's own known-answer tests and (b) outputs of the
reference itself run in the build container, committed as
``tests/golden/*.npz`` by ``oracle/make_golden.py``.

Semantics restated (reference file:line in brackets):

* views are row-major float64 buffers shared by reference; a function
  mutates its caller's buffers in place [runtime.py:74-115, 481-511]
* statements run in order; every bulk statement / kernel is a sync point
  [runtime.py:520-563]
* a ``parallel_for`` runs iterations 0..n-1 (sequentially here, i.e. the
  reference with threads=1); plain writes land immediately
  [runtime.py:586-593, 409-428]
* ``atomic_add`` inside a kernel is *deferred*: contributions are queued as
  (iteration, sequence-in-iteration) and applied after the kernel in that
  order [runtime.py:430-447, 615-620]; at function scope it applies
  immediately [runtime.py:441-442, 546-547]
* every access is bounds-checked, error text ``line L: v(i) outside extent
  n`` [runtime.py:299-321]; a view value used as an index is truncated
  toward zero [runtime.py:335]
* value arithmetic is IEEE double, division never raises
  [runtime.py:260-270]; a counter read as a value is ``float(i)``
  [runtime.py:245]
* ``parallel_sum`` gather = adjacent-pair tree, odd levels padded with +0.0,
  *added to* the destination scalar (0.0 if unbound) [runtime.py:166-177,
  643-651]; accumulate forms ``dst += src`` / ``dst += scalar``
  [runtime.py:653-665]; ``deep_copy`` copy / fill with exact extent match
  [runtime.py:628-641]
* ``check_finite`` traps non-finite views after each kernel / bulk statement
  and non-finite scalars at gather / return [runtime.py:669-676]
* conflict detection (``detect``): each kernel is replayed sequentially in the order
  ``random.Random(rng_seed + kernel_index).shuffle`` gives; every view read, plain write and
  atomic_add is logged as (view, offset) -> iteration -> kinds; a location touched by two or
  more distinct iterations with a plain write among its accesses is one record, records
  sorted by (view, offset) within a kernel [runtime.py:198-227, 284-285, 418-419, 439-440,
  574-585]; pinned by ``tests/golden/conflicts.json`` (oracle/make_golden_conflicts.py)
"""

from __future__ import annotations

import random

import numpy as np


class ShapeMismatch(ValueError):
    pass


class OutOfBounds(IndexError):
    pass


class NonFiniteDetected(ArithmeticError):
    pass


def pairwise_sum(values) -> float:
    """Adjacent-pair tree; a level of odd length is padded with +0.0
    (reference runtime.py:166-177)."""
    a = np.array(values, dtype=np.float64).reshape(-1)
    if a.size == 0:
        return 0.0
    while a.size > 1:
        if a.size & 1:
            a = np.concatenate([a, [0.0]])
        a = a[0::2] + a[1::2]
    return float(a[0])


def _k(node) -> str:
    return type(node).__name__


class Machine:
    """State of one function call: named views (numpy arrays, shared with the
    caller), function-scope scalars, and the deferred-atomic queue of the
    kernel in flight."""

    def __init__(self, fn, check_finite=False, deterministic=True, threads=1):
        self.fn = fn
        self.threads = max(1, int(threads))
        self.views: dict = {}
        self.scalars: dict = {}
        self.check_finite = check_finite
        self.deterministic = deterministic
        self.local: dict = {}  # counter + loop-local scalars of the running iteration
        self.queue = None  # list while inside a kernel
        self.iteration = -1
        self.seq = 0
        self.value = None
        self.trace = None  # conflict detection: {(view, offset): {iteration: {kinds}}} of the running kernel
        self.rng_seed = None  # not None: conflict detection on
        self.kernel_index = 0
        self.records: list = []

    def touch(self, view, off, what):
        if self.trace is not None:
            self.trace.setdefault((view, off), {}).setdefault(self.iteration, set()).add(what)

    # ---- index sub-language (Python ints) -----------------------------------

    def index(self, e):
        k = _k(e)
        if k == "IntLiteral":
            return e.value
        if k == "Counter":
            return self.local[e.name]
        if k == "Extent":
            return self.views[e.view].shape[e.dim]
        if k == "ViewAccess":
            return int(self.load(e))
        if k == "IdxBinary":
            a, b = self.index(e.lhs), self.index(e.rhs)
            return a + b if e.op == "+" else a - b if e.op == "-" else a * b
        raise TypeError(f"not an index expression: {k}")

    def offset(self, acc):
        buf = self.views[acc.view]
        idx = [self.index(i) for i in acc.indices]
        line = acc.span.line
        if len(idx) == 1:
            (i,) = idx
            n0 = buf.shape[0]
            if not 0 <= i < n0:
                raise OutOfBounds(f"line {line}: {acc.view}({i}) outside extent {n0}")
            return buf.reshape(-1), i
        a, b = idx
        n0, n1 = buf.shape
        if not (0 <= a < n0 and 0 <= b < n1):
            raise OutOfBounds(f"line {line}: {acc.view}({a}, {b}) outside extents {n0}x{n1}")
        return buf.reshape(-1), a * n1 + b

    def load(self, acc):
        flat, off = self.offset(acc)
        self.touch(acc.view, off, "read")
        return flat[off]

    # ---- value sub-language (numpy float64 scalars: IEEE, no exceptions) ----

    def val(self, e):
        k = _k(e)
        if k == "Literal":
            return np.float64(e.value)
        if k == "ScalarVar":
            if e.name in self.local:
                return self.local[e.name]
            return self.scalars[e.name]
        if k == "IndexVar":
            return np.float64(self.local[e.name])
        if k == "ViewAccess":
            return self.load(e)
        if k == "Extent":
            return np.float64(self.views[e.view].shape[e.dim])
        if k == "Neg":
            return -self.val(e.operand)
        if k == "Binary":
            a, b = np.float64(self.val(e.lhs)), np.float64(self.val(e.rhs))
            if e.op == "+":
                return a + b
            if e.op == "-":
                return a - b
            if e.op == "*":
                return a * b
            if e.op == "/":
                return a / b
        raise TypeError(f"cannot evaluate {k}")

    def compare(self, c) -> bool:
        a, b = self.index(c.lhs), self.index(c.rhs)
        return {
            "==": a == b, "!=": a != b, "<": a < b, "<=": a <= b, ">": a > b, ">=": a >= b,
        }[c.op]

    # ---- element statements (kernel bodies; also legal at function scope) ---

    def element(self, s, in_kernel: bool):
        k = _k(s)
        if k == "DeclScalar":
            (self.local if in_kernel else self.scalars)[s.name] = self.val(s.init)
        elif k == "AssignScalar":
            env = self.local if in_kernel else self.scalars
            v = self.val(s.rhs)
            if s.op == "=":
                env[s.name] = v
            elif s.op == "+=":
                env[s.name] = env[s.name] + v
            else:
                env[s.name] = env[s.name] - v
        elif k == "AssignView":
            flat, off = self.offset(s.target)
            v = self.val(s.rhs)
            self.touch(s.target.view, off, "write")
            if s.op == "=":
                flat[off] = v
            elif s.op == "+=":
                flat[off] += v
            else:
                flat[off] -= v
        elif k == "AtomicAdd":
            flat, off = self.offset(s.target)
            v = self.val(s.value)
            self.touch(s.target.view, off, "atomic")
            if self.queue is None:
                flat[off] += v
            else:
                self.queue.append((self.iteration, self.seq, flat, off, v))
                self.seq += 1
        elif k == "If":
            if self.compare(s.cond):
                for inner in s.body:
                    self.element(inner, in_kernel)
        else:
            raise TypeError(f"statement not allowed here: {k}")

    # ---- function-scope statements ------------------------------------------------

    def run(self, inputs: dict):
        self.bind(inputs)
        with np.errstate(all="ignore"):
            for s in self.fn.body:
                self.statement(s)
        return self.value

    def bind(self, inputs: dict):
        want, got = {p.name for p in self.fn.params}, set(inputs)
        if want != got:
            parts = []
            if want - got:
                parts.append(f"missing {sorted(want - got)}")
            if got - want:
                parts.append(f"unexpected {sorted(got - want)}")
            raise ShapeMismatch(f"inputs do not match parameters: {'; '.join(parts)}")
        for p in self.fn.params:
            v = inputs[p.name]
            if p.is_view:
                if not (isinstance(v, np.ndarray) and v.dtype == np.float64 and v.flags.c_contiguous):
                    v = np.ascontiguousarray(v, dtype=np.float64)
                    inputs[p.name] = v
                if v.ndim != p.type.rank:
                    raise ShapeMismatch(
                        f"parameter '{p.name}': rank {p.type.rank} expected, got rank {v.ndim}"
                    )
                for d, ext in enumerate(p.type.extents):
                    if _k(ext) == "StaticExtent" and v.shape[d] != ext.size:
                        raise ShapeMismatch(
                            f"parameter '{p.name}' dim {d}: static extent {ext.size} expected, "
                            f"got {v.shape[d]}"
                        )
                self.views[p.name] = v
            else:
                self.scalars[p.name] = np.float64(v)

    def statement(self, s):
        k = _k(s)
        if k == "DeclView":
            args = iter(s.dyn_args)
            dims = [
                e.size if _k(e) == "StaticExtent" else int(self.index(next(args)))
                for e in s.descriptor.extents
            ]
            if any(d < 0 for d in dims):
                raise ShapeMismatch(f"view '{s.name}': negative extent {dims}")
            self.views[s.name] = np.zeros(dims, dtype=np.float64)
        elif k == "If":
            # function scope: the body may hold any statement (reference runtime.py:548-550, self.body(b))
            if self.compare(s.cond):
                for inner in s.body:
                    self.statement(inner)
        elif k in ("DeclScalar", "AssignScalar", "AssignView", "AtomicAdd"):
            self.element(s, in_kernel=False)
        elif k == "ParallelFor":
            self.kernel(s)
        elif k == "DeepCopy":
            dst = self.views[s.dst]
            if isinstance(s.src, str):
                src = self.views[s.src]
                if dst.shape != src.shape:
                    raise ShapeMismatch(f"deep_copy: {s.dst}{dst.shape} vs {s.src}{src.shape}")
                dst[...] = src
            else:
                dst[...] = self.val(s.src)
            self.guard_views()
        elif k == "ParallelSum":
            flat = self.views[s.src].reshape(-1)
            total = pairwise_sum(flat) if self.deterministic else float(np.sum(flat))
            self.scalars[s.dst] = np.float64(self.scalars.get(s.dst, 0.0)) + np.float64(total)
            self.guard_value(self.scalars[s.dst])
        elif k == "ParallelSumInto":
            dst = self.views[s.dst]
            if isinstance(s.src, str):
                src = self.views[s.src]
                if dst.shape != src.shape:
                    raise ShapeMismatch(f"parallel_sum: {s.dst}{dst.shape} vs {s.src}{src.shape}")
                dst += src
            else:
                dst += self.val(s.src)
            self.guard_views()
        elif k == "Return":
            self.value = float(self.val(s.value))
            self.guard_value(self.value)
        else:
            raise TypeError(f"cannot execute {k}")

    def kernel(self, loop):
        n = int(self.index(loop.upper))
        self.queue = []
        order = list(range(n))
        if self.rng_seed is not None:
            random.Random(self.rng_seed + self.kernel_index).shuffle(order)
            self.trace = {}
        try:
            if self.threads > 1 and n >= 2 * self.threads and self.rng_seed is None:
                self.queue = self.kernel_on_pool(loop, n)
                order = ()
            for i in order:
                self.local = {loop.counter: i}
                self.iteration, self.seq = i, 0
                for s in loop.body:
                    self.element(s, in_kernel=True)
        finally:
            queue, self.queue, self.local = self.queue, None, {}
            log, self.trace = self.trace, None
        if log is not None:
            for (view, off), by_iter in sorted(log.items()):
                if len(by_iter) >= 2 and any("write" in ks for ks in by_iter.values()):
                    self.records.append((self.kernel_index, view, int(off), tuple(sorted(by_iter)),
                                         tuple(sorted({k for ks in by_iter.values() for k in ks}))))
        self.kernel_index += 1
        # kernel boundary: queued contributions land in (iteration, sequence) order
        queue.sort(key=lambda q: (q[0], q[1]))
        for _, _, flat, off, v in queue:
            flat[off] += v
        self.guard_views()

    def kernel_on_pool(self, loop, n):
        """threads > 1: the reference cuts [0, n) into `threads` contiguous chunks and runs them on
        a thread pool, every chunk with its own iteration context but the SAME view storage; plain
        writes land immediately, atomic contributions are queued per chunk and merged (the sort by
        (iteration, sequence) at the kernel boundary makes the result independent of the schedule)
        [runtime.py:594-613].  Python threads share the interpreter lock, so this costs rather
        than saves time - which is exactly what the reference's bench shows."""
        import copy
        from concurrent.futures import ThreadPoolExecutor

        T = self.threads
        bounds = [(n * t) // T for t in range(T + 1)]

        def chunk(t):
            w = copy.copy(self)
            w.queue, w.local = [], {}
            for i in range(bounds[t], bounds[t + 1]):
                w.local = {loop.counter: i}
                w.iteration, w.seq = i, 0
                for s in loop.body:
                    w.element(s, in_kernel=True)
            return w.queue

        with ThreadPoolExecutor(max_workers=T) as pool:
            parts = list(pool.map(chunk, range(T)))
        return [q for part in parts for q in part]

    # ---- optional finiteness traps ----------------------------------------------------

    def guard_views(self):
        if self.check_finite:
            for name, buf in self.views.items():
                if not np.isfinite(buf).all():
                    raise NonFiniteDetected(f"non-finite value in view '{name}'")

    def guard_value(self, v):
        if self.check_finite and v is not None and not np.isfinite(v):
            raise NonFiniteDetected(f"non-finite scalar {float(v)!r}")


def run(program, fn_name: str, inputs: dict, *, check_finite=False, deterministic=True, threads=1):
    """Execute ``fn_name`` on ``inputs`` (name -> float64 ndarray | float).
    Arrays are mutated in place.  Returns the function value (None if void).  ``threads``: the
    reference's thread-pool execution of kernels (same results, see Machine.kernel_on_pool)."""
    fn = program.function(fn_name)
    if fn is None:
        raise KeyError(f"no function named '{fn_name}'")
    return Machine(fn, check_finite, deterministic, threads).run(inputs)


def detect(program, fn_name: str, inputs: dict, *, rng_seed: int = 0):
    """The reference's ``detect_conflicts``: returns the records as tuples
    (kernel, view, offset, iterations, kinds).  Arrays are mutated in place."""
    fn = program.function(fn_name)
    if fn is None:
        raise KeyError(f"no function named '{fn_name}'")
    m = Machine(fn)
    m.rng_seed = rng_seed
    m.run(inputs)
    return m.records
