"""Sharded mode of the headline objective: the row range [0, N) is split into
one contiguous shard per rank (one process per GPU), the way the reference
splits a kernel's iteration range over its thread pool
(/root/reference/pkg/src/krn/runtime.py:594-613), but across devices.

Per evaluation each rank needs from its neighbours only the *original* values
x[lo-2], x[lo-1], b[lo-1] and x[hi], x[hi+1], b[hi]: the fused kernels recompute
the neighbour rows' adjoints locally (gather form), so no adjoint ever crosses a
shard boundary and the summation order of every ``_d_x`` entry is the
reference's.  Collectives, both latency bound:

* one all_gather of 6 doubles per rank (the halo rows)
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
    x[0], x[1], b[0], x[-2], x[-1], b[-1] (torch tensors, any device)."""
    import torch

    if x.numel() < 2:
        raise ValueError("a shard needs at least 2 rows")
    return torch.stack([x[0], x[1], b[0], x[-2], x[-1], b[-1]])


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


class ShardedLaplacian:
    """One rank's view of the sharded objective."""

    def __init__(self, n_global: int, device, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.dev = device
        self.n_global = n_global
        self.span = int(device.lib.krn_laplacian_partial_span(n_global))
        self.parts = partition(n_global, self.world, self.span)
        self.offset, self.n_local = self.parts[self.rank]
        self.block_counts = [partial_count(length, self.span) for _, length in self.parts]

    def exchange_halo(self, x, b):
        import torch

        if self.world == 1:
            return None
        mine = pack_boundary(x, b)
        gathered = torch.empty(self.world * 6, dtype=x.dtype, device=x.device)  # flat: gloo and nccl agree
        self.dist.all_gather_into_tensor(gathered, mine, group=self.group)
        return assemble_halo(gathered.view(self.world, 6), self.rank, self.world)

    def primal(self, x, x_out, b, f_out, *, exact: bool = True):
        """f_out (1-element tensor) <- global objective; x_out <- 3x (local rows)."""
        import torch

        from . import _cabi

        lib = self.dev.lib
        halo = self.exchange_halo(x, b)
        _cabi.check(lib.krn_laplacian_primal(
            self.dev.h, C.c_void_p(x.data_ptr()), C.c_void_p(x_out.data_ptr()), C.c_void_p(b.data_ptr()),
            self.n_local, self.offset, self.n_global,
            C.c_void_p(halo.data_ptr()) if halo is not None else None, C.c_void_p(f_out.data_ptr()), 0))
        if self.world == 1:
            return f_out
        if not exact:
            self.dist.all_reduce(f_out, group=self.group)
            return f_out
        # every rank contributes max(block counts) doubles (the tail is padding that is cut off again)
        width = max(self.block_counts)
        mine = torch.zeros(width, dtype=x.dtype, device=x.device)
        _cabi.check(lib.krn_laplacian_partials(self.dev.h, C.c_void_p(mine.data_ptr()), self.block_counts[self.rank]))
        gathered = torch.empty(self.world * width, dtype=x.dtype, device=x.device)
        self.dist.all_gather_into_tensor(gathered, mine, group=self.group)
        nodes = combine_partials(gathered.view(self.world, width), self.block_counts)
        _cabi.check(lib.krn_reduce_pairwise(self.dev.h, C.c_void_p(nodes.data_ptr()), nodes.numel(),
                                            C.c_void_p(f_out.data_ptr()), 0))
        return f_out

    def grad(self, x, x_out, b, dx, db, *, seed=1.0, dx_zero=False, db_zero=False):
        from . import _cabi

        halo = self.exchange_halo(x, b)
        _cabi.check(self.dev.lib.krn_laplacian_grad(
            self.dev.h, C.c_void_p(x.data_ptr()), C.c_void_p(x_out.data_ptr()), C.c_void_p(b.data_ptr()),
            C.c_void_p(dx.data_ptr()), C.c_void_p(db.data_ptr()), int(dx_zero), int(db_zero),
            self.n_local, self.offset, self.n_global,
            C.c_void_p(halo.data_ptr()) if halo is not None else None, float(seed)))
