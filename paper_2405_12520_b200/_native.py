"""Loader for the in-tree native library ``libtsb200.so`` (C-ABI in include/tsb200.h).

There is no fallback: if the library is missing or cannot be loaded, every
engine entry point raises ``EngineError``.  The router / host-only entry
points work without a GPU; engine creation needs a CUDA device.
"""

from __future__ import annotations

import ctypes as C
import os

from .cabi import TsbReport
from .errors import EngineError, InputError

HERE = os.path.dirname(os.path.abspath(__file__))
# TSB200_LIB lets kernel experiments load an alternative in-tree build of the
# same C-ABI (default: the library `__graft_entry__.build()` makes).
LIB_PATH = os.environ.get("TSB200_LIB") or os.path.join(HERE, "libtsb200.so")

TSB_EINVAL, TSB_ERANGE = -1, -2

# name -> (restype, argtypes)
_vp, _i32, _i64, _f64 = C.c_void_p, C.c_int32, C.c_int64, C.c_double
SIGNATURES = {
    "tsb_create": (_i32, [_vp, _vp, _vp, _i32, C.POINTER(_vp)]),
    "tsb_destroy": (None, [_vp]),
    "tsb_last_error": (C.c_char_p, []),
    "tsb_step": (_i32, [_vp, _i32, C.POINTER(TsbReport)]),
    "tsb_report_get": (_i32, [_vp, C.POINTER(TsbReport)]),
    "tsb_state": (_i32, [_vp, C.POINTER(_i32), _vp, _vp, _vp, _vp, _vp, _vp]),
    "tsb_status": (_i32, [_vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "tsb_finished": (_i32, [_vp, _i64, _i64, _vp, _vp, C.POINTER(_i64)]),
    "tsb_road_acc": (_i32, [_vp, _i32, _vp, _vp]),
    "tsb_min_front_gap": (_i32, [_vp, C.POINTER(_f64)]),
    "tsb_get_vehicles": (_i32, [_vp, _vp, _i32, _vp]),
    "tsb_grid_build": (_i32, [_i32, _i32, _f64, _i32, _f64, _i32, C.POINTER(_vp)]),
    "tsb_grid_sizes": (_i32, [_vp, _vp]),
    "tsb_grid_export": (_i32, [_vp, _vp]),
    "tsb_grid_destroy": (None, [_vp]),
    "tsb_py_dist": (_f64, [_f64, _f64, _f64, _f64]),
    "tsb_set_geometry": (_i32, [_vp, _vp, _i64, _vp, _vp]),
    "tsb_records": (_i32, [_vp, _i32, _vp, _vp, _vp, _vp, _vp, _vp, C.POINTER(_i32)]),
    "tsb_set_lane": (_i32, [_vp, _i32, _f64, _i32]),
    "tsb_set_signal_phase": (_i32, [_vp, _i32, _i32]),
    "tsb_signal_state": (_i32, [_vp, _vp, _vp]),
    "tsb_route": (_i32, [_vp, _i32, _i32, _i32, _vp, C.POINTER(_i32), C.POINTER(_f64)]),
    "tsb_router_create": (_i32, [_vp, C.POINTER(_vp)]),
    "tsb_router_destroy": (None, [_vp]),
    "tsb_router_route": (_i32, [_vp, _i32, _i32, _i32, _vp, C.POINTER(_i32), C.POINTER(_f64)]),
    "tsb_router_reach": (_i32, [_vp, _i32, _vp, _vp]),
    "tsb_profile_steps": (_i32, [_vp, _i32, _i32, _vp]),
    "tsb_kernel_name": (C.c_char_p, [_i32]),
    "tsb_time_steps": (_i32, [_vp, _i32, C.POINTER(_f64)]),
    "tsb_launches_per_step": (_i32, [_vp, C.POINTER(_i32)]),
    "tsb_set_debug": (_i32, [_vp, _i32]),
    "tsb_path_counters": (_i32, [_vp, _vp]),
    "tsb_timeline": (_i32, [_vp, _vp]),
    "tsb_set_timeline": (_i32, [_vp, _i32]),
    "tsb_fp64_peak": (_i32, [_i32, C.POINTER(_f64)]),
    "tsb_step_sync_bytes": (_i32, [C.POINTER(_i64)]),
    "tsb_create_sharded": (_i32, [_vp, _vp, _vp, _i32, _vp, C.POINTER(_vp)]),
    "tsb_create_sharded_local": (_i32, [_vp, _vp, _vp, _vp, _vp, _i32, _vp, C.POINTER(_vp)]),
    "tsb_mark": (_i32, [_vp, _i32]),
    "tsb_set_pow_mode": (_i32, [_vp, _i32]),
    "tsb_marks_elapsed": (_i32, [_vp, _i32, _i32, C.POINTER(_f64)]),
    "tsb_shard_export": (_i32, [_vp, _vp, _i64, _vp]),
    "tsb_shard_import": (_i32, [_vp, _vp, _vp]),
    "tsb_shard_p2p_alloc": (_i32, [_vp, _vp, _vp, _vp]),
    "tsb_shard_p2p_set_peers": (_i32, [_vp, _vp, _vp]),
    "tsb_shard_p2p_exchange": (_i32, [_vp]),
    "tsb_set_p2p_timeout": (_i32, [_vp, _f64]),
    "tsb_exchange_bytes": (_i32, [_vp, C.POINTER(_i64)]),
    "tsb_step_async": (_i32, [_vp, _i32]),
    "tsb_ipc_handle": (_i32, [_vp, _vp]),
    "tsb_ipc_open": (_i32, [_vp, _vp]),
    "tsb_ipc_close": (_i32, [_vp]),
}

_lib = None


def lib():
    """The loaded library (raises EngineError if it is not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise EngineError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
        try:
            L = C.CDLL(LIB_PATH)
        except OSError as exc:
            raise EngineError(f"cannot load {LIB_PATH}: {exc}") from None
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc == 0:
        return
    msg = (lib().tsb_last_error() or b"").decode("utf-8", "replace")
    if rc in (TSB_EINVAL, TSB_ERANGE):
        raise InputError(msg)
    raise EngineError(f"native engine error {rc}: {msg}")
