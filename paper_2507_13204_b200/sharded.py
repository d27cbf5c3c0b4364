"""Sharded mode of the headline objective: the row range [0, N) is split into
one contiguous shard per rank (one process per GPU), the way the reference
splits a kernel's iteration range over its thread pool
(/root/reference/pkg/src/krn/runtime.py:594-613), but across devices.

Per evaluation each rank needs from its neighbours only the *original* values
x[lo-2], x[lo-1], b[lo-1] and x[hi], x[hi+1], b[hi]: the fused kernels recompute
the neighbour rows' adjoints locally (gather form), so no adjoint ever crosses a
shard boundary and the summation order of every ``_d_x`` entry is the
reference's.

**Device-resident step (``attach``)**: the ranks exchange, ONCE, the CUDA IPC
handles of the buffers their x and b live in (one all_gather of 144 bytes at set-up)
and map their neighbours' buffers (peer memory over NVLink / NVSwitch; two
processes on one device work the same way).  The kernels' boundary steps then read
the halo rows straight through those pointers: a gradient step is exactly ONE
launch and NO collective; the primal adds only the all_gather of its tree partials.
A fence (barrier across the ranks) is needed only when a neighbour has rewritten the
rows being read, i.e. when x itself changes between steps.

Without ``attach`` (or for tensors other than the attached ones) the halo travels by
collectives, both latency bound:

* one all_gather of 6 doubles per rank (the halo rows; packed with one ``cat`` and
  unpacked with one ``index_select``)
* for the objective value (primal only; the gradient does not depend on it) one
  all_gather of the per-block tree partials (one double per 1024 or 4096 rows;
  244 KB per rank at 125 M rows), folded by every rank with the reference's tree:
  shard cuts are multiples of the partial span, so the partials of all ranks in
  rank order ARE the nodes of the single-device tree and the result is
  bit-identical to the single-device and to the reference's value for any number
  of GPUs (``exact=False``: a plain all_reduce(SUM) of 1 double instead, exact
  only up to reassociation)

``torch.distributed`` is the plumbing (NCCL on GPUs; gloo for the CPU tests of
the partition/halo logic).  Device memory here is torch tensors whose
``data_ptr()`` goes straight into the C ABI.
"""

from __future__ import annotations

import ctypes as C


def partition(n_global: int, world: int, align: int = 1) -> list:
    """[(offset, length)] per rank: contiguous, covering, boundaries rounded down
    to a multiple of ``align`` (the primal kernel's partial span, so that block
    partials stay nodes of the reference's reduction tree)."""
    cuts = [0]
    for r in range(1, world):
        c = (n_global * r) // world
        c -= c % align
        cuts.append(max(c, cuts[-1]))
    cuts.append(n_global)
    return [(cuts[r], cuts[r + 1] - cuts[r]) for r in range(world)]


def partial_count(n_local: int, span: int) -> int:
    """Tree partials one shard produces (one per started span of rows)."""
    return (n_local + span - 1) // span


def combine_partials(gathered, counts):
    """The all-gathered partial matrix (world x width, rows padded) as ONE vector in rank order:
    because every cut is a multiple of the span these are exactly the per-block nodes a single
    device would have produced, so the reference's tree over them is the reference's value."""
    import torch

    if all(c == gathered.shape[1] for c in counts):
        return gathered.reshape(-1)  # equal shards: already one contiguous vector
    return torch.cat([gathered[r, :c] for r, c in enumerate(counts)]).contiguous()


def pack_boundary(x, b):
    """The 6 values a shard contributes to its neighbours' halos:
    x[0], x[1], b[0], x[-2], x[-1], b[-1] (torch tensors, any device; one kernel)."""
    import torch

    if x.numel() < 2:
        raise ValueError("a shard needs at least 2 rows")
    return torch.cat([x[:2], b[:1], x[-2:], b[-1:]])


def assemble_halo(gathered, rank: int, world: int):
    """From the all-gathered boundaries (world x 6) build this rank's halo
    [x[lo-2], x[lo-1], b[lo-1], x[hi], x[hi+1], b[hi]]; sides that fall outside
    the problem are zero and never read (the kernels guard on the global row)."""
    import torch

    halo = torch.zeros(6, dtype=gathered.dtype, device=gathered.device)
    if rank > 0:
        halo[0:3] = gathered[rank - 1, 3:6]
    if rank < world - 1:
        halo[3:6] = gathered[rank + 1, 0:3]
    return halo


_ipc_maps: dict = {}  # (device ordinal, handle bytes) -> [mapped base, users]: a handle opens once per process


class ShardedLaplacian:
    """One rank's view of the sharded objective."""

    def __init__(self, n_global: int, device, group=None, shortcut_single: bool = True):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        # a group of ONE rank needs no collective at all; False keeps them in (a way to drive the NCCL
        # code path on a single GPU)
        self.shortcut_single = shortcut_single
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.dev = device
        self.n_global = n_global
        self.span = int(device.lib.krn_laplacian_partial_span(n_global))
        self.parts = partition(n_global, self.world, self.span)
        # decided identically on every rank, BEFORE any collective: a shard must hold the two rows its
        # neighbours' gather-form adjoints reach for
        short = [r for r, (_, length) in enumerate(self.parts) if length < 2]
        if self.world > 1 and short:
            raise ValueError(f"{n_global} rows over {self.world} ranks (cuts aligned to {self.span} rows) leaves "
                             f"ranks {short} fewer than 2 rows: use fewer ranks")
        self.offset, self.n_local = self.parts[self.rank]
        self.block_counts = [partial_count(length, self.span) for _, length in self.parts]
        self._peers = None
        self.attach_failure = None  # why attach() fell back to the collective halo exchange, if it did
        self._halo_index = None
        self._ext_stream = None

    # ---- stream order between torch and the library ---------------------------------------------
    def _streams(self):
        """(torch's current stream, the context's stream as a torch stream or None when they are one)"""
        import torch

        cur = torch.cuda.current_stream()
        sp = C.c_void_p()
        self.dev.lib.krn_ctx_stream(self.dev.h, C.byref(sp))
        if (sp.value or 0) == cur.cuda_stream:
            return cur, None
        if self._ext_stream is None or self._ext_stream.cuda_stream != (sp.value or 0):
            self._ext_stream = torch.cuda.ExternalStream(sp.value)
        return cur, self._ext_stream

    def _before(self, x):
        """torch work queued so far (producers of x, b, the halo) precedes the library's kernels"""
        if x.is_cuda:
            cur, ext = self._streams()
            if ext is not None:
                ext.wait_stream(cur)

    def _after(self, x):
        if x.is_cuda:
            cur, ext = self._streams()
            if ext is not None:
                cur.wait_stream(ext)

    # ---- peer memory ---------------------------------------------------------------------------------
    def _gather_bytes(self, mine):
        """all_gather of a small uint8 tensor (set-up only); staged on the device for NCCL"""
        import torch

        nccl = self.dist.get_backend(self.group) == "nccl"
        t = mine.cuda() if nccl else mine
        out = torch.empty(self.world * t.numel(), dtype=torch.uint8, device=t.device)
        self.dist.all_gather_into_tensor(out, t, group=self.group)
        return out.cpu().view(self.world, -1)

    def attach(self, x, b):
        """Map the neighbours' x and b (these very tensors: attach again when they are replaced).
        Collective: every rank of the group calls it."""
        import numpy as np
        import torch

        from . import _cabi

        self.detach()
        if self.world == 1:
            return self
        lib, dev = self.dev.lib, self.dev
        rec = np.zeros(144, dtype=np.uint8)
        for k, t in enumerate((x, b)):
            handle = (C.c_ubyte * 64)()
            off = C.c_size_t()
            _cabi.check(lib.krn_ipc_export(dev.h, C.c_void_p(t.data_ptr()), handle, C.byref(off)))
            rec[72 * k:72 * k + 64] = np.frombuffer(handle, dtype=np.uint8)
            rec[72 * k + 64:72 * k + 72] = np.frombuffer(np.uint64(off.value).tobytes(), dtype=np.uint8)
        everyone = self._gather_bytes(torch.from_numpy(rec)).numpy()

        def open_(rank, k):
            raw = everyone[rank, 72 * k:72 * k + 72].tobytes()
            handle, off = raw[:64], int(np.frombuffer(raw[64:], dtype=np.uint64)[0])
            key = (dev.ordinal, handle)
            hit = _ipc_maps.get(key)
            if hit is None:
                base, ptr = C.c_void_p(), C.c_void_p()
                buf = (C.c_ubyte * 64).from_buffer_copy(handle)
                _cabi.check(lib.krn_ipc_open(dev.h, buf, 0, C.byref(base), C.byref(ptr)))
                hit = _ipc_maps[key] = [base.value, 0]
            hit[1] += 1
            self._mapped.append(key)
            return hit[0] + off

        self._mapped = []
        peers = dict(x=x.data_ptr(), b=b.data_ptr(), xp=0, bp=0, xn=0, bn=0)
        failure = None
        try:
            if self.rank > 0:
                n_prev = self.parts[self.rank - 1][1]
                peers["xp"] = open_(self.rank - 1, 0) + 8 * n_prev
                peers["bp"] = open_(self.rank - 1, 1) + 8 * n_prev
            if self.rank < self.world - 1:
                peers["xn"] = open_(self.rank + 1, 0)
                peers["bn"] = open_(self.rank + 1, 1)
        except _cabi.KrnNativeError as exc:  # no peer access between the two devices, handles not importable, ...
            failure = str(exc)
        # all or nothing: a rank that cannot map its neighbours takes everybody to the collective halo path
        ok = torch.tensor([0 if failure else 1], dtype=torch.uint8)
        if not bool(self._gather_bytes(ok).min()):
            self._peers = peers  # (so that detach releases what this rank did map)
            self.detach()
            self.attach_failure = failure or "a neighbour could not map this rank's memory"
            return self
        self.attach_failure = None
        self._peers = peers
        self.fence()  # everybody has mapped (and the tensors' producers have finished) before anyone reads
        return self

    def detach(self):
        from . import _cabi

        if self._peers is None:
            return
        self._peers = None
        for key in getattr(self, "_mapped", []):
            hit = _ipc_maps.get(key)
            if hit is None:
                continue
            hit[1] -= 1
            if hit[1] <= 0:
                _cabi.check(self.dev.lib.krn_ipc_close(self.dev.h, C.c_void_p(hit[0])))
                del _ipc_maps[key]
        self._mapped = []

    def fence(self):
        """Every rank's queued work is complete: call after x or b CHANGED on some rank and before the
        next step reads it through the peer pointers (not needed while the inputs stay as they are)."""
        import torch

        if torch.cuda.is_available():
            torch.cuda.synchronize()
        self.dev.sync()
        if self.world > 1:
            self.dist.barrier(group=self.group)

    def _attached(self, x, b):
        p = self._peers
        return p is not None and p["x"] == x.data_ptr() and p["b"] == b.data_ptr()

    # ---- halo by collective (tensors that are not attached) --------------------------------------------
    def exchange_halo(self, x, b):
        import torch

        if self.world == 1 and self.shortcut_single:
            return None
        mine = pack_boundary(x, b)
        gathered = torch.empty(self.world * 6, dtype=x.dtype, device=x.device)  # flat: gloo and nccl agree
        self.dist.all_gather_into_tensor(gathered, mine, group=self.group)
        if self._halo_index is None or self._halo_index.device != x.device:
            # [x[lo-2], x[lo-1], b[lo-1], x[hi], x[hi+1], b[hi]] as positions in the gathered vector; a side
            # outside the problem points at this rank's own entries (never read: the kernels guard on the
            # global row)
            prev = self.rank - 1 if self.rank > 0 else self.rank
            nxt = self.rank + 1 if self.rank < self.world - 1 else self.rank
            idx = [6 * prev + 3, 6 * prev + 4, 6 * prev + 5, 6 * nxt, 6 * nxt + 1, 6 * nxt + 2]
            self._halo_index = torch.tensor(idx, dtype=torch.int64, device=x.device)
        return gathered.index_select(0, self._halo_index)

    def primal(self, x, x_out, b, f_out, *, exact: bool = True):
        """f_out (1-element tensor) <- global objective; x_out <- 3x (local rows)."""
        import torch

        from . import _cabi

        lib = self.dev.lib
        P = C.c_void_p
        if self._attached(x, b):
            p = self._peers
            self._before(x)
            _cabi.check(lib.krn_laplacian_primal_peers(
                self.dev.h, P(x.data_ptr()), P(x_out.data_ptr()), P(b.data_ptr()), self.n_local, self.offset,
                self.n_global, P(p["xp"]), P(p["bp"]), P(p["xn"]), P(p["bn"]), P(f_out.data_ptr()), 0))
        else:
            halo = self.exchange_halo(x, b)
            self._before(x)
            _cabi.check(lib.krn_laplacian_primal(
                self.dev.h, P(x.data_ptr()), P(x_out.data_ptr()), P(b.data_ptr()),
                self.n_local, self.offset, self.n_global,
                P(halo.data_ptr()) if halo is not None else None, P(f_out.data_ptr()), 0))
        if self.world == 1 and self.shortcut_single:
            self._after(x)
            return f_out
        if not exact:
            self._after(x)
            self.dist.all_reduce(f_out, group=self.group)
            return f_out
        # every rank contributes max(block counts) doubles (the tail is padding that is cut off again)
        width = max(self.block_counts)
        mine = torch.zeros(width, dtype=x.dtype, device=x.device)
        self._before(x)
        _cabi.check(lib.krn_laplacian_partials(self.dev.h, P(mine.data_ptr()), self.block_counts[self.rank]))
        self._after(x)
        gathered = torch.empty(self.world * width, dtype=x.dtype, device=x.device)
        self.dist.all_gather_into_tensor(gathered, mine, group=self.group)
        nodes = combine_partials(gathered.view(self.world, width), self.block_counts)
        self._before(x)
        _cabi.check(lib.krn_reduce_pairwise(self.dev.h, P(nodes.data_ptr()), nodes.numel(),
                                            P(f_out.data_ptr()), 0))
        self._after(x)
        return f_out

    def grad(self, x, x_out, b, dx, db, *, seed=1.0, dx_zero=False, db_zero=False):
        from . import _cabi

        P = C.c_void_p
        if self._attached(x, b):
            # one launch, no collective: the boundary steps read the neighbours' rows through peer pointers
            p = self._peers
            self._before(x)
            _cabi.check(self.dev.lib.krn_laplacian_grad_peers(
                self.dev.h, P(x.data_ptr()), P(x_out.data_ptr()), P(b.data_ptr()), P(dx.data_ptr()), P(db.data_ptr()),
                int(dx_zero), int(db_zero), self.n_local, self.offset, self.n_global,
                P(p["xp"]), P(p["bp"]), P(p["xn"]), P(p["bn"]), float(seed)))
            self._after(x)
            return
        halo = self.exchange_halo(x, b)
        self._before(x)
        _cabi.check(self.dev.lib.krn_laplacian_grad(
            self.dev.h, P(x.data_ptr()), P(x_out.data_ptr()), P(b.data_ptr()),
            P(dx.data_ptr()), P(db.data_ptr()), int(dx_zero), int(db_zero),
            self.n_local, self.offset, self.n_global,
            P(halo.data_ptr()) if halo is not None else None, float(seed)))
        self._after(x)
