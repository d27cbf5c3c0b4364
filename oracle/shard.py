"""TEST INFRASTRUCTURE - numpy restatement of what ONE SHARD of the sharded
headline objective must produce, given the halo rows its neighbours send
(paper_2507_13204_b200/sharded.py, include/krn_b200.h).  Used by the CPU tests
of the multi-GPU logic: concatenating every shard's output must reproduce the
whole-problem oracle (oracle/krn_oracle.c) bit for bit.  Not product code.

The per-row arithmetic is the reference's (gradient text in
/root/reference/pkg/tests/test_adjoint.py:43-94) evaluated in gather form:
row k of _d_x receives -r3[k-1], 2*r1[k], -r2[k+1] in that order
(reference runtime.py:615-620 sorts the queued atomics by iteration)."""

from __future__ import annotations

import numpy as np


def _rows(x_ext, b_ext, g, n_global, seed):
    """y and the adjoint chain for extended rows (global indices g)."""
    xs = 3.0 * x_ext
    r4 = 0.0 + (0.0 + seed)
    m = len(g)
    y = np.zeros(m)
    r3, r2, r1 = np.zeros(m), np.zeros(m), np.zeros(m)
    for k in range(1, m - 1):  # first/last extended entries only serve as neighbours
        gk = g[k]
        if gk < 0 or gk >= n_global:
            continue
        v = 2.0 * xs[k] - b_ext[k]
        if gk != 0:
            v = v - xs[k - 1]
        if gk != n_global - 1:
            v = v - xs[k + 1]
        y[k] = v
        dy = 0.0 + r4 * v
        dy = dy + v * r4
        if gk != n_global - 1:
            r3[k] = dy
            dy = dy - r3[k]
            dy = dy + r3[k]
        if gk != 0:
            r2[k] = dy
            dy = dy - r2[k]
            dy = dy + r2[k]
        r1[k] = dy
    return xs, y, r3, r2, r1


def laplacian_shard(x, b, dx, db, halo, offset, n_global, seed=1.0):
    """x, b, dx, db: this shard's rows (dx/db updated in place); halo = [x[lo-2], x[lo-1],
    b[lo-1], x[hi], x[hi+1], b[hi]] original values.  Returns (3x rows, y2 rows)."""
    n = len(x)
    halo = np.zeros(6) if halo is None else np.asarray(halo, dtype=np.float64)
    x_ext = np.concatenate([halo[0:2], x, halo[3:5]])
    b_ext = np.concatenate([[0.0, halo[2]], b, [halo[5], 0.0]])
    g = np.arange(offset - 2, offset + n + 2)
    with np.errstate(all="ignore"):
        xs, y, r3, r2, r1 = _rows(x_ext, b_ext, g, n_global, seed)
        for i in range(n):
            k, gk = i + 2, offset + i
            acc = dx[i]
            if gk != 0:
                acc = acc + (-r3[k - 1])
            acc = acc + 2.0 * r1[k]
            if gk != n_global - 1:
                acc = acc + (-r2[k + 1])
            r0 = acc
            acc = acc - r0
            acc = acc + 3.0 * r0
            dx[i] = acc
            db[i] = db[i] + (-r1[k])
    return xs[2:-2], (y * y)[2:-2]


def tree_pad(j: int, n: int) -> float:
    """Leaf value of a missing leaf j >= n of the blocked tree (csrc/krn_prelude.cuh:krn_tree_pad):
    +0.0 where the reference pads an odd level (runtime.py:166-177), the identity -0.0 elsewhere."""
    low = j & (-j)
    return 0.0 if (j - low < n and j != low) else -0.0


def block_partials(y2, offset: int, n_global: int, span: int) -> np.ndarray:
    """The per-block tree nodes one shard's primal kernel produces: block k covers global rows
    [offset + k*span, offset + (k+1)*span) as a complete binary tree, leaves past n_global padded."""
    n = len(y2)
    out = []
    for start in range(0, n, span):
        leaves = np.array([y2[start + j] if start + j < n else tree_pad(offset + start + j, n_global)
                           for j in range(span)], dtype=np.float64)
        while len(leaves) > 1:
            leaves = leaves[0::2] + leaves[1::2]
        out.append(leaves[0])
    return np.array(out, dtype=np.float64)
