"""TEST INFRASTRUCTURE - ctypes front of oracle/krn_oracle.c (the plain-C
restatement of the reference's arithmetic for the headline objective and the
bulk builtins).  Never imported by the product package."""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import build as _build

_lib = None
_dp = C.POINTER(C.c_double)


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(_build.build())
        L.krn_oracle_pairwise_sum.restype = C.c_double
        L.krn_oracle_pairwise_sum.argtypes = [_dp, C.c_size_t, _dp]
        L.krn_oracle_laplacian_primal.restype = C.c_double
        L.krn_oracle_laplacian_primal.argtypes = [_dp, _dp, C.c_size_t, _dp]
        L.krn_oracle_laplacian_grad.restype = None
        L.krn_oracle_laplacian_grad.argtypes = [_dp, _dp, _dp, _dp, C.c_size_t, C.c_double, _dp]
        L.krn_oracle_threads.restype = C.c_int
        L.krn_oracle_apply_queue.restype = None
        L.krn_oracle_apply_queue.argtypes = [_dp, C.c_size_t, C.POINTER(C.c_uint32), _dp, C.c_size_t, C.c_int]
        _lib = L
    return _lib


def _p(a):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def pairwise_sum(v) -> float:
    v = np.ascontiguousarray(v, dtype=np.float64).reshape(-1)
    scratch = np.empty(max(v.size, 1))
    return float(lib().krn_oracle_pairwise_sum(_p(v), v.size, _p(scratch)))


def laplacian_primal(x, b) -> float:
    """x (scaled in place), b: float64 1-D arrays.  Returns f."""
    work = np.empty(3 * x.size + 1)
    return float(lib().krn_oracle_laplacian_primal(_p(x), _p(b), x.size, _p(work)))


def laplacian_grad(x, b, dx, db, seed: float = 1.0) -> None:
    """Accumulates into dx, db; x scaled in place."""
    work = np.empty(5 * x.size + 1)
    lib().krn_oracle_laplacian_grad(_p(x), _p(b), _p(dx), _p(db), x.size, seed, _p(work))


def threads() -> int:
    """OpenMP threads the order-free loops of the C port use."""
    return int(lib().krn_oracle_threads())


def apply_queue(target, keys, vals, width: int = 1) -> None:
    """The reference's apply loop over an already ordered queue of atomic_add records
    (runtime.py:615-620): target[keys[r]] += vals[r, w] for w in order, r in order."""
    keys = np.ascontiguousarray(keys, dtype=np.uint32)
    vals = np.ascontiguousarray(vals, dtype=np.float64).reshape(-1)
    assert vals.size == keys.size * width and target.flags.c_contiguous
    lib().krn_oracle_apply_queue(_p(target.reshape(-1)), target.size, keys.ctypes.data_as(C.POINTER(C.c_uint32)),
                                 _p(vals), keys.size, width)
