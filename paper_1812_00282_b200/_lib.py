"""ctypes binding of libvate_b200.so (declared in include/vate.h).

The library is the product: there is no CPU fallback.  If the shared object is
missing or fails to load, importing this module raises ImportError naming the
build command, and every device call raises if no CUDA device is present.
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import ConfigError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libvate_b200.so")

VATE_OK, VATE_ECONFIG, VATE_EVALUE, VATE_ECUDA, VATE_ENOMEM = 0, -1, -2, -3, -4
VATE_HOST, VATE_DEVICE, VATE_STAGED = 0, 1, 2
KERNEL_KINDS = ("scan", "registry", "bitmap", "g0", "final", "sweep", "sort", "other")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build the CUDA library first "
        "(python -c 'import __graft_entry__; __graft_entry__.build()' or make -C "
        "paper_1812_00282_b200/csrc)")

lib = C.CDLL(LIB_PATH)

class StepResult(C.Structure):
    """vate_step_result (include/vate.h)."""
    _fields_ = [("nhosts", C.c_uint64), ("nkept", C.c_uint64), ("pool_inactive", C.c_uint64),
                ("prev_collected", C.c_int32), ("prev_blocks", C.c_int32 * 2),
                ("prev_maintained", C.c_uint64), ("prev_cleared", C.c_uint64),
                ("prev_t", C.c_int64), ("prev_valid", C.c_int32)]


_p = C.c_void_p
_u64 = C.c_uint64
_i64 = C.c_int64
_i32 = C.c_int32
_int = C.c_int
_dbl = C.c_double
_pu64 = C.POINTER(C.c_uint64)
_pi32 = C.POINTER(C.c_int32)
_pdbl = C.POINTER(C.c_double)

_SIGS = {
    "vate_last_error": ([], C.c_char_p),
    "vate_abi_version": ([], _int),
    "vate_device_count": ([C.POINTER(_int)], _int),
    "vate_pool_create": ([C.POINTER(_p), _int, _int, _int, _int], _int),
    "vate_pool_create_kind": ([C.POINTER(_p), _int, _int, _int, _int, _int], _int),
    "vate_pool_kind": ([_p, C.POINTER(_int), _pu64], _int),
    "vate_get_cells64": ([_p, _p, _u64, _p, _int], _int),
    "vate_put_cells": ([_p, _p, _p, _u64, _int], _int),
    "vate_fill_cells": ([_p, _u64], _int),
    "vate_pool_device_bytes": ([_p, _p], _int),
    "vate_pool_mode": ([_p, _p], _int),
    "vate_pool_set_latency": ([_p, _int], _int),
    "vate_pool_set_peer": ([_p, _p, _int, _int], _int),
    "vate_api_calls": ([_p], _int),
    "vate_tracer_create": ([_p, _p, _u64, _u64], _int),
    "vate_tracer_destroy": ([_p], _int),
    "vate_tracer_buffer": ([_p, _int, _p], _int),
    "vate_tracer_submit": ([_p, _int, _u64, _i64, _u64, _int, _u64, _u64], _int),
    "vate_tracer_collect": ([_p, _int, _p, _u64, _p, _p, _p], _int),
    "vate_tracer_release": ([_p, _int], _int),
    "vate_bench_l2": ([_p, _u64, _u64, _int, _p], _int),
    "vate_bench_scan_skeleton": ([_p, _int, _u64, _u64, _int, _p], _int),
    "vate_bench_scan_ablation": ([_p, _int, _u64, _u64, _int, _int, _p], _int),
    "vate_pool_latency": ([_p, _p], _int),
    "vate_pool_lat_mark": ([_p, _i64, _int], _int),
    "vate_pool_destroy": ([_p], _int),
    "vate_pool_info": ([_p, C.POINTER(_i32), C.POINTER(_i32), C.POINTER(_p)], _int),
    "vate_pool_sync": ([_p], _int),
    "vate_pool_launches": ([_p, _pu64], _int),
    "vate_pool_set_timing": ([_p, _int], _int),
    "vate_pool_timing": ([_p, _int, _pdbl, _pu64], _int),
    "vate_pool_set_option": ([_p, _int, _i64], _int),
    "vate_pool_inc_stats": ([_p, _pu64], _int),
    "vate_pool_sort_stats": ([_p, _pu64], _int),
    "vate_pool_sort_sizes": ([_p, _pu64], _int),
    "vate_pool_timeline": ([_p, _p, _u64, _pu64], _int),
    "vate_profiler": ([_int], _int),
    "vate_mark": ([_p, _int], _int),
    "vate_mark_elapsed": ([_p, _int, _int, _pdbl], _int),
    "vate_set_cells": ([_p, _p, _u64, _int], _int),
    "vate_scan_pairs": ([_p, _u64, _u64, _u64, _p, _p, _u64, _int, _p, _i64], _int),
    "vate_scan_packed": ([_p, _u64, _u64, _u64, _p, _u64, _int, _p, _i64], _int),
    "vate_stage_packed": ([_p, _p, _u64, C.POINTER(_int)], _int),
    "vate_scan_staged": ([_p, _u64, _u64, _u64, _int, _u64, _p, _i64], _int),
    "vate_pair_cells": ([_p, _u64, _int, _u64, _u64, _p, _p, _u64, _int, _p], _int),
    "vate_host_cells": ([_p, _u64, _int, _u64, _p, _u64, _int, _p], _int),
    "vate_advance": ([_p, _pi32, _pu64, _pu64], _int),
    "vate_advance_async": ([_p], _int),
    "vate_advance_result": ([_p, _pi32, _pu64, _pu64], _int),
    "vate_count_inactive": ([_p, _int, _pu64], _int),
    "vate_inactive_mask": ([_p, _p, _u64, _int, _p, _int], _int),
    "vate_get_cells": ([_p, _p, _u64, _p, _int], _int),
    "vate_host_g0": ([_p, _u64, _u64, _p, _u64, _int, _p, _int], _int),
    "vate_set_log_table": ([_p, _u64, _p], _int),
    "vate_reports_from_counts": ([_p, _u64, _p, _u64, _u64, _dbl, _p, _p, _p], _int),
    "vate_estimate_begin": ([_p, _p, _u64, _u64, _i64, _int, _pu64, _pu64], _int),
    "vate_estimate_begin_hosts": ([_p, _p, _u64, _int, _u64, _u64, _int, _pu64], _int),
    "vate_estimate_begin_part": ([_p, _p, _u64, _u64, _i64, _int, _int, _int, _pu64, _pu64], _int),
    "vate_estimate_finish": ([_p, _u64, _u64, _dbl, _dbl, _p, _p, _p, _p, _u64, _pu64], _int),
    "vate_estimate_finish_async": ([_p, _u64, _u64, _dbl, _dbl, _p, _p, _p, _p, _u64, _pu64], _int),
    "vate_estimate_wait": ([_p], _int),
    "vate_reports_device": ([_p, _p, _p, _p, _p], _int),
    "vate_reports_copy": ([_p, _u64, _u64, _p, _p, _p, _p], _int),
    "vate_slice_step": ([_p, _p, _u64, _u64, _u64, _p, _u64, _int, _i64, _int, _dbl, _p,
                         _p, _p, _p, _p, _u64, C.POINTER(StepResult)], _int),
    "vate_slice_step_lagged": ([_p, _p, _u64, _u64, _u64, _p, _u64, _int, _i64, _int, _dbl, _p,
                                _p, _p, _p, _p, _u64, _p], _int),
    "vate_slice_flush": ([_p, _p, _u64, _u64, _dbl, _p, _p, _p, _p, _p, _u64, _p], _int),
    "vate_slice_lagged_begin": ([_p, _p, _u64, _u64, _u64, _p, _u64, _int, _i64, _int, _p], _int),
    "vate_slice_lagged_end": ([_p, _p, _u64, _u64, _u64, _dbl, _dbl, _p, _p, _p, _p, _u64, _p],
                              _int),
    "vate_slice_lagged_flush_begin": ([_p, _p, _u64, _u64, _p], _int),
    "vate_snapshot_size": ([_p, _pu64], _int),
    "vate_snapshot": ([_p, _p, _u64, _pu64], _int),
    "vate_load": ([_p, _p, _u64], _int),
    "vate_hosts_create": ([C.POINTER(_p), _p, _int], _int),
    "vate_hosts_destroy": ([_p], _int),
    "vate_hosts_update": ([_p, _p, _u64, _i64, _int], _int),
    "vate_hosts_active": ([_p, _i64, _int, _p, _u64, _pu64], _int),
    "vate_hosts_prune": ([_p, _i64], _int),
    "vate_hosts_size": ([_p, _pu64], _int),
    "vate_hosts_touched": ([_p, _i64, _p, _u64, _pu64], _int),
    "vate_dirty_bitmap": ([_p, _p], _int),
    "vate_merge_dirty": ([_p, _p, _int], _int),
    "vate_peer_create": ([C.POINTER(_p), _p, _p, _int, _int, _u64, _p], _int),
    "vate_peer_open": ([_p, _p], _int),
    "vate_peer_set_mode": ([_p, _int], _int),
    "vate_peer_exchange": ([_p, _i64, _pu64], _int),
    "vate_peer_info": ([_p, _pu64, _pu64, C.POINTER(_int)], _int),
    "vate_peer_destroy": ([_p], _int),
    "vate_synth_zipf": ([_p, _i64, _u64, _u64, _u64, _u64, _p, _p, _u64, C.c_uint32, _p], _int),
    "vate_bench_sol_scatter": ([_p, _u64, _u64, _int, _pdbl], _int),
    "vate_synth_packets": ([_p, _i64, _u64, _u64, _u64, _u64, _p], _int),
}

for _name, (_args, _res) in _SIGS.items():
    _fn = getattr(lib, _name)  # AttributeError here means header and library drifted
    _fn.argtypes = _args
    _fn.restype = _res

EXPORTED = tuple(_SIGS)

# Handles are destroyed registries-first at interpreter exit, before the CUDA
# runtime inside the library is torn down; __del__ is a no-op from then on.
import atexit as _atexit
import weakref as _weakref

_LIVE = _weakref.WeakValueDictionary()
_SHUTDOWN = [False]


def track(obj) -> None:
    _LIVE[id(obj)] = obj


def shutting_down() -> bool:
    return _SHUTDOWN[0]


@_atexit.register
def _close_all() -> None:
    objs = list(_LIVE.values())
    for o in objs:                       # peer windows before the registries they feed
        if getattr(o, "_is_peer", False):
            o.close()
    for o in objs:                       # registries before the pools they live on
        if getattr(o, "_is_registry", False):
            o.close()
    for o in objs:
        if not getattr(o, "_is_registry", False) and not getattr(o, "_is_peer", False):
            o.close()
    _SHUTDOWN[0] = True


def last_error() -> str:
    msg = lib.vate_last_error()
    return msg.decode() if msg else ""


def check(rc: int) -> None:
    """Map a vate_status to the reference's exception convention (errors.py)."""
    if rc == VATE_OK:
        return
    msg = last_error()
    if rc == VATE_ECONFIG:
        raise ConfigError(msg)
    if rc == VATE_EVALUE:
        raise ValueError(msg)
    if rc == VATE_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(f"libvate_b200: {msg}")


def device_count() -> int:
    n = _int(0)
    rc = lib.vate_device_count(C.byref(n))
    return n.value if rc == VATE_OK else 0


def ptr(arr) -> int:
    """Address of a contiguous numpy array (0 for empty)."""
    return arr.ctypes.data if arr.size else 0
