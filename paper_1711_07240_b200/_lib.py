"""ctypes binding of the in-tree C-ABI library ``libcgbn.so`` (declared in include/cgbn.h).

There is deliberately no fallback: if the library is missing or fails to load, every
hot-path call raises. The library is built in-tree by ``make`` (or
``__graft_entry__.build()``) so it travels with the repository to the GPU box.
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CGBN_LIB", os.path.join(_HERE, "libcgbn.so"))

# Keep in sync with include/cgbn.h
ABI_VERSION = 7  # CGBN_ABI_VERSION the bindings below were written for
LAYOUT_NCHW = 0
LAYOUT_NHWC = 1
ACT_F32 = 0x00   # activation dtype, OR'd into the layout argument
ACT_BF16 = 0x10
ACT_F16 = 0x20
MAX_GROUP = 64
OK = 0
ERR_INVALID = 1
ERR_CUDA = 2
ERR_UNSUPPORTED = 3
STATUS_NONFINITE = 1
STATUS_SMALL_COUNT = 2
STATUS_EXCHANGE_TIMEOUT = 4
DTYPE_F32 = 0
DTYPE_F64 = 1

_p = ctypes.c_void_p
_i64 = ctypes.c_int64
_i = ctypes.c_int
_d = ctypes.c_double
_sz = ctypes.c_size_t
_pp = ctypes.POINTER(ctypes.c_void_p)

# name -> (restype, argtypes); every symbol include/cgbn.h declares.
SIGNATURES = {
    "cgbn_abi_version": (_i, []),
    "cgbn_build_info": (ctypes.c_char_p, []),
    "cgbn_last_error": (ctypes.c_char_p, []),
    "cgbn_num_sms": (_i, []),
    "cgbn_workspace_bytes": (_sz, [_i64, _i64, _i64, _i]),
    "cgbn_fwd_stats": (_i, [_p, _i64, _i64, _i64, _i, _p, _p, _sz, _p]),
    "cgbn_fwd_normalize": (_i, [_p, _i64, _i64, _i64, _i, _pp, _i, _p, _p, _d, _d, _p, _p, _p,
                                _i, _p, _p, _p, _sz, _p]),
    "cgbn_fwd_train_local": (_i, [_p, _i64, _i64, _i64, _i, _p, _p, _d, _d, _p, _p, _p, _i, _p,
                                  _p, _p, _sz, _p]),
    "cgbn_fwd_eval": (_i, [_p, _i64, _i64, _i64, _i, _p, _p, _p, _p, _d, _i, _p, _p, _sz, _p]),
    "cgbn_bwd_reduce": (_i, [_p, _p, _i64, _i64, _i64, _i, _p, _p, _p, _i, _p, _p, _sz, _p]),
    "cgbn_bwd_dx": (_i, [_p, _p, _i64, _i64, _i64, _i, _pp, _i, _p, _p, _p, _d, _i, _p, _p, _p,
                         _p, _p, _sz, _p]),
    "cgbn_bwd_local": (_i, [_p, _p, _i64, _i64, _i64, _i, _p, _p, _p, _d, _i, _p, _p, _p, _p, _p,
                            _sz, _p]),
    "cgbn_xhat": (_i, [_p, _i64, _i64, _i64, _i, _p, _p, _p, _sz, _p]),
    "cgbn_fold_sum": (_i, [_pp, _i, _i64, _i, _p, _p]),
    "cgbn_channel_sum": (_i, [_p, _i64, _i64, _i64, _i, _p, _p, _p, _sz, _p]),
    "cgbn_centered_sumsq": (_i, [_p, _i64, _i64, _i64, _i, _p, _p, _p, _p, _sz, _p]),
    "cgbn_p2p_region_bytes": (_sz, [_i, _i64]),
    "cgbn_p2p_alloc": (_i, [_sz, _pp, _p]),
    "cgbn_p2p_open": (_i, [_p, _pp]),
    "cgbn_p2p_close": (_i, [_p]),
    "cgbn_p2p_free": (_i, [_p]),
    "cgbn_p2p_exchange": (_i, [_p, _i64, _i, _i, _pp, _i64, _p, _p, _d, _p]),
    "cgbn_p2p_emulate": (_i, [_p, _i64, _i, _pp, _i64, _p, _p, _d, _i, _p]),
    "cgbn_fwd_normalize_sums": (_i, [_p, _i64, _i64, _i64, _i, _p, _p, _p, _i, _p, _p, _d, _d,
                                     _p, _p, _p, _i, _p, _p, _p, _sz, _p]),
    "cgbn_channel_affine": (_i, [_p, _i64, _i64, _i64, _i, _p, _p, _p, _p]),
    "cgbn_fused_supported": (_i, [_i64, _i64, _i64, _i, _i]),
    "cgbn_onchip_selected": (_i, [_i64, _i64, _i64, _i, _i]),
    "cgbn_fwd_fused": (_i, [_p, _i64, _i64, _i64, _i, _p, _p, _d, _d, _p, _p, _p, _i, _p, _p, _p,
                            _sz, _p]),
    "cgbn_bwd_fused": (_i, [_p, _p, _i64, _i64, _i64, _i, _p, _p, _p, _d, _i, _p, _p, _p, _p, _p,
                            _sz, _p]),
    "cgbn_fwd_stats_p2p": (_i, [_p, _i64, _i64, _i64, _i, _i, _i, _pp, _i64, _p, _sz, _p]),
    "cgbn_fwd_normalize_p2p": (_i, [_p, _i64, _i64, _i64, _i, _p, _i, _i64, _d, _p, _p, _d, _d,
                                    _p, _p, _p, _i, _p, _p, _p, _sz, _p]),
    "cgbn_bwd_reduce_p2p": (_i, [_p, _p, _i64, _i64, _i64, _i, _p, _p, _p, _i, _i, _i, _pp, _i64,
                                 _p, _sz, _p]),
    "cgbn_bwd_dx_p2p": (_i, [_p, _p, _i64, _i64, _i64, _i, _p, _i, _i64, _d, _p, _p, _p, _d, _i,
                             _p, _p, _p, _p, _p, _sz, _p]),
    "cgbn_fwd_normalize_slots": (_i, [_p, _i64, _i64, _i64, _i, _p, _p, _p, _d, _d, _p, _p, _p,
                                      _i, _p, _p, _p, _sz, _p]),
    "cgbn_conv1x1_ws_bytes": (_sz, [_i64, _i64, _i64, _i64]),
    "cgbn_conv1x1": (_i, [_p, _p, _p, _i64, _i64, _i64, _i64, _i, _p, _p, _sz, _p]),
    "cgbn_conv1x1_stats": (_i, [_p, _p, _p, _i64, _i64, _i64, _i64, _i, _p, _p, _p, _sz, _p]),
    "cgbn_conv_nhwc_ws_bytes": (_sz, [_i64, _i64, _i64, _i64, _i64, _i, _i]),
    "cgbn_conv_nhwc": (_i, [_p, _p, _p, _i64, _i64, _i64, _i64, _i64, _i, _i, _i, _p, _p, _sz,
                            _p]),
    "cgbn_conv_nhwc_stats": (_i, [_p, _p, _p, _i64, _i64, _i64, _i64, _i64, _i, _i, _i, _p, _p,
                                  _p, _sz, _p]),
}

_lib = None
_lock = threading.Lock()


class CGBNLibraryError(RuntimeError):
    """The native library is missing, failed to load, or a call returned an error."""


def load():
    """Load libcgbn.so once (thread-safe) and bind every exported signature."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise CGBNLibraryError(
                f"native CGBN library not found at {LIB_PATH}; build it with `make` "
                "(there is no CPU fallback)")
        try:
            lib = ctypes.CDLL(LIB_PATH)
        except OSError as exc:  # pragma: no cover - environment specific
            raise CGBNLibraryError(f"failed to load {LIB_PATH}: {exc}") from exc
        # a stale or foreign build must not be called with these argument lists
        missing = [n for n in SIGNATURES if not hasattr(lib, n)]
        if missing:
            raise CGBNLibraryError(
                f"{LIB_PATH} lacks {len(missing)} entry point(s) of include/cgbn.h "
                f"({', '.join(missing[:4])}{', ...' if len(missing) > 4 else ''}); rebuild "
                "it with `make`")
        lib.cgbn_abi_version.restype = _i
        lib.cgbn_abi_version.argtypes = []
        got = lib.cgbn_abi_version()
        if got != ABI_VERSION:
            raise CGBNLibraryError(
                f"{LIB_PATH} implements CGBN ABI v{got}, these bindings need v{ABI_VERSION}; "
                "rebuild it with `make`")
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def check(rc: int, what: str):
    if rc != OK:
        msg = load().cgbn_last_error().decode(errors="replace")
        raise CGBNLibraryError(f"{what} failed (code {rc}): {msg}")


def ptr_array(ptrs):
    """ctypes array of device pointers (ints) for the `const T* const*` parameters."""
    arr = (ctypes.c_void_p * len(ptrs))(*ptrs)
    return ctypes.cast(arr, _pp), arr
