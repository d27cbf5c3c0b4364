"""ctypes binding of libkrn_b200.so (include/krn_b200.h).

This is the only place the package touches native code.  There is no CPU
fallback: if the library cannot be loaded, or a call fails, a ``KrnNativeError``
is raised.  Loading works on a machine without a GPU (the library opens
libcuda/libnvrtc lazily), which is what the CPU-only test tier checks; any
call that needs a device fails loudly there.
"""

from __future__ import annotations

import ctypes as C
import os
import re

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libkrn_b200.so")
HEADER_PATH = os.path.join(os.path.dirname(_PKG), "include", "krn_b200.h")

KRN_ST_OUT_OF_BOUNDS = 1
KRN_ST_BAD_INDEX = 2


class KrnNativeError(RuntimeError):
    """A libkrn_b200 call failed (message from krn_last_error)."""


_vp, _dp, _sz, _i, _d = C.c_void_p, C.c_void_p, C.c_size_t, C.c_int, C.c_double
_pp = C.POINTER(C.c_void_p)

# name -> (restype, argtypes); must cover every function include/krn_b200.h declares
SIGNATURES = {
    "krn_last_error": (C.c_char_p, []),
    "krn_version": (C.c_char_p, []),
    "krn_device_count": (_i, [C.POINTER(_i)]),
    "krn_ctx_create": (_i, [_i, _vp, _pp]),
    "krn_ctx_destroy": (_i, [_vp]),
    "krn_sync": (_i, [_vp]),
    "krn_ctx_stream": (_i, [_vp, _pp]),
    "krn_ctx_sm_count": (_i, [_vp, C.POINTER(_i)]),
    "krn_ctx_launch_count": (_i, [_vp, C.POINTER(C.c_uint64)]),
    "krn_alloc": (_i, [_vp, _sz, _pp]),
    "krn_free": (_i, [_vp, _vp]),
    "krn_host_alloc": (_i, [_sz, _pp]),
    "krn_host_free": (_i, [_vp]),
    "krn_upload": (_i, [_vp, _vp, _vp, _sz]),
    "krn_download": (_i, [_vp, _vp, _vp, _sz]),
    "krn_download_async": (_i, [_vp, _vp, _vp, _sz]),
    "krn_event_create": (_i, [_pp]),
    "krn_event_destroy": (_i, [_vp]),
    "krn_event_record": (_i, [_vp, _vp]),
    "krn_event_elapsed_ms": (_i, [_vp, _vp, C.POINTER(C.c_float)]),
    "krn_stream_create": (_i, [_vp, _pp]),
    "krn_stream_destroy": (_i, [_vp]),
    "krn_stream_sync": (_i, [_vp]),
    "krn_upload_on": (_i, [_vp, _vp, _vp, _sz]),
    "krn_download_on": (_i, [_vp, _vp, _vp, _sz]),
    "krn_event_record_on": (_i, [_vp, _vp]),
    "krn_stream_wait_event": (_i, [_vp, _vp]),
    "krn_ctx_wait_event": (_i, [_vp, _vp]),
    "krn_fill": (_i, [_vp, _dp, _sz, _d, _dp]),
    "krn_copy": (_i, [_vp, _dp, _dp, _sz]),
    "krn_add_scalar": (_i, [_vp, _dp, _sz, _d, _dp]),
    "krn_add_view": (_i, [_vp, _dp, _dp, _sz]),
    "krn_reduce_pairwise": (_i, [_vp, _dp, _sz, _dp, _i]),
    "krn_check_finite": (_i, [_vp, _dp, _sz, _vp]),
    "krn_ordered_accumulate": (_i, [_vp, _dp, _sz, _vp, _dp, _sz, _i]),
    "krn_ordered_accumulate_rows": (_i, [_vp, _dp, _sz, _i, C.POINTER(_i), _i, _vp, _dp, _sz]),
    "krn_memset": (_i, [_vp, _vp, _i, _sz]),
    "krn_laplacian_primal": (_i, [_vp, _dp, _dp, _dp, _sz, _sz, _sz, _dp, _dp, _i]),
    "krn_laplacian_grad": (_i, [_vp, _dp, _dp, _dp, _dp, _dp, _i, _i, _sz, _sz, _sz, _dp, _d]),
    "krn_laplacian_partial_span": (_sz, [_sz]),
    "krn_laplacian_partials": (_i, [_vp, _dp, _sz]),
    "krn_ipc_export": (_i, [_vp, _vp, _vp, C.POINTER(C.c_size_t)]),
    "krn_ipc_open": (_i, [_vp, _vp, _sz, _pp, _pp]),
    "krn_ipc_close": (_i, [_vp, _vp]),
    "krn_laplacian_primal_peers": (_i, [_vp, _dp, _dp, _dp, _sz, _sz, _sz, _dp, _dp, _dp, _dp, _dp, _i]),
    "krn_laplacian_grad_peers": (_i, [_vp, _dp, _dp, _dp, _dp, _dp, _i, _i, _sz, _sz, _sz, _dp, _dp, _dp, _dp, _d]),
    "krn_module_compile": (_i, [_vp, C.c_char_p, _pp]),
    "krn_jit_info": (_i, [C.POINTER(_i), C.POINTER(_i), C.POINTER(_i)]),
    "krn_module_destroy": (_i, [_vp]),
    "krn_module_launch": (_i, [_vp, _vp, C.c_char_p, _sz, _sz, _pp]),
    "krn_module_launch_exact": (_i, [_vp, _vp, C.c_char_p, _sz, C.c_uint, _sz, _pp]),
    "krn_module_kernel_info": (_i, [_vp, C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "krn_status_reset": (_i, [_vp]),
    "krn_run_begin": (_i, [_vp, _pp, C.POINTER(C.c_size_t)]),
    "krn_reduce_workspace": (_i, [_vp, _sz, _pp, _pp, _pp]),
    "krn_status_device_ptr": (_i, [_vp, _pp]),
    "krn_status_read": (_i, [_vp, C.POINTER(C.c_longlong)]),
}

_lib = None


def declared_functions(header_path: str = HEADER_PATH) -> list:
    """Function names declared in include/krn_b200.h (used by the ABI test)."""
    text = open(header_path).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(krn_[a-z0-9_]+)\s*\(", text)))


def lib():
    """The loaded library; raises KrnNativeError when it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise KrnNativeError(
                f"{LIB_PATH} not found: build it with `python -m paper_2507_13204_b200.csrc.build` "
                "(there is no CPU fallback)"
            )
        try:
            L = C.CDLL(LIB_PATH)
        except OSError as e:
            raise KrnNativeError(f"cannot load {LIB_PATH}: {e}") from e
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype, fn.argtypes = res, args
        _lib = L
    return _lib


def check(rc: int):
    if rc != 0:
        msg = lib().krn_last_error().decode("utf-8", "replace")
        raise KrnNativeError(msg or f"libkrn_b200 call failed with code {rc}")


def device_count() -> int:
    n = C.c_int(0)
    try:
        check(lib().krn_device_count(C.byref(n)))
    except KrnNativeError:
        return 0
    return n.value
