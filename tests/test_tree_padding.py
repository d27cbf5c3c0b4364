"""CPU tier: the padding rule that lets a blocked, fully padded binary tree
reproduce the reference's pairwise_sum bit for bit (csrc/krn_prelude.cuh:
krn_tree_pad, krn_final_tree), emulated in numpy against the oracle."""

import numpy as np
import pytest

from oracle import interp
from conftest import assert_bits


def tree_pad(j, n):
    low = j & (-j)
    return 0.0 if (j - low < n and j != low) else -0.0


def blocked_tree(v, chunk):
    """What the kernels do: every block reduces an aligned chunk of `chunk` leaves as a
    complete tree with krn_tree_pad leaves past n; the block partials are then folded
    level by level, an odd level getting last + (+0.0)."""
    n = len(v)
    nb = (n + chunk - 1) // chunk
    partials = []
    for blk in range(nb):
        leaves = np.array([v[j] if j < n else tree_pad(j, n) for j in range(blk * chunk, (blk + 1) * chunk)])
        while len(leaves) > 1:
            leaves = leaves[0::2] + leaves[1::2]
        partials.append(leaves[0])
    p = np.array(partials)
    while len(p) > 1:
        if len(p) & 1:
            p = np.concatenate([p[:-1], [p[-1] + 0.0]])
            p = np.concatenate([p[:-1][0::2] + p[:-1][1::2], [p[-1]]]) if len(p) > 1 else p
        else:
            p = p[0::2] + p[1::2]
    return p[0]


@pytest.mark.parametrize("chunk", [4, 16, 64])
def test_blocked_tree_equals_reference_tree(chunk):
    rng = np.random.default_rng(chunk)
    for n in list(range(1, 200)) + [255, 256, 257, 511, 513, 1000]:
        v = rng.normal(size=n) * 10.0 ** rng.integers(-4, 5, size=n)
        assert_bits(blocked_tree(v, chunk), interp.pairwise_sum(v), f"n={n} chunk={chunk}")


@pytest.mark.parametrize("chunk", [4, 16])
def test_signed_zeros(chunk):
    """-0.0 survives exactly where the reference keeps it (no padded level on its path)"""
    for n in range(1, 70):
        for fill in (-0.0, 0.0):
            v = np.full(n, fill)
            assert_bits(blocked_tree(v, chunk), interp.pairwise_sum(v), f"n={n} fill={fill}")
        v = np.full(n, -0.0)
        v[n // 2] = 0.0
        assert_bits(blocked_tree(v, chunk), interp.pairwise_sum(v), f"mixed n={n}")
