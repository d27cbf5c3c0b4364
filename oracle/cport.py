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
