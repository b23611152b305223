"""ctypes binding of libhkv_b200.so (the C-ABI in include/hkv_b200.h).

The product path has no CPU fallback: if the shared library is missing or
cannot be loaded, importing the table raises immediately.
"""

from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HKV_LIB") or os.path.join(_HERE, "libhkv_b200.so")  # HKV_LIB: experiment builds

HKV_OK, HKV_EINVAL, HKV_ECUDA, HKV_ENOMEM, HKV_EBUSY = 0, 1, 2, 3, 4


class HkvConfig(C.Structure):
    _fields_ = [
        ("capacity", C.c_int64),
        ("value_dim", C.c_int64),
        ("mode", C.c_int32),
        ("score_policy", C.c_int32),
        ("fast_tier_budget", C.c_int64),
        ("digest_filter", C.c_int32),
        ("admit_ties_unified", C.c_int32),
        ("overflow_in_hbm", C.c_int32),
        ("device", C.c_int32),
        ("workers", C.c_int32),
    ]


_vp = C.c_void_p
_i64 = C.c_int64
_i32 = C.c_int32
_u64 = C.c_uint64

# name -> (restype, argtypes); every symbol include/hkv_b200.h declares.
SIGNATURES = {
    "hkv_last_error": (C.c_char_p, []),
    "hkv_version": (C.c_char_p, []),
    "hkv_launch_count": (_i64, []),
    "hkv_create": (C.c_int, [C.POINTER(HkvConfig), C.POINTER(_vp)]),
    "hkv_destroy": (C.c_int, [_vp]),
    "hkv_set_workers": (C.c_int, [_vp, _i32]),
    "hkv_find": (C.c_int, [_vp, _vp, _i64, _vp, _vp, _i32, _vp]),
    "hkv_contains": (C.c_int, [_vp, _vp, _i64, _vp, _vp]),
    "hkv_find_ptr": (C.c_int, [_vp, _vp, _i64, _vp, _vp, _vp, _vp]),
    "hkv_upsert": (C.c_int, [_vp, _i32, _vp, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _u64, _vp]),
    "hkv_find_host": (C.c_int, [_vp, _vp, _i64, _vp, _vp, _i32, _vp]),
    "hkv_ipc_handles": (C.c_int, [_vp, _vp, _i64]),
    "hkv_set_peers": (C.c_int, [_vp, _i32, _i32, _vp]),
    "hkv_set_peers_local": (C.c_int, [_vp, _i32, _vp]),
    "hkv_find_peer": (C.c_int, [_vp, _vp, _i64, _vp, _vp, _i32, _vp]),
    "hkv_upsert_host": (C.c_int, [_vp, _i32, _vp, _vp, _vp, _i64, _vp, _vp, _u64, _vp]),
    "hkv_assign": (C.c_int, [_vp, _vp, _vp, _vp, _i32, _i64, _vp, _vp, _u64, _vp]),
    "hkv_erase": (C.c_int, [_vp, _vp, _i64, _vp, _vp]),
    "hkv_export": (C.c_int, [_vp, _i64, _i64, _i32, _u64, _vp, _i64, _vp, _vp, _vp,
                             C.POINTER(_i64), C.POINTER(_i64), _vp]),
    "hkv_size": (C.c_int, [_vp, C.POINTER(_i64), _vp]),
    "hkv_set_epoch": (C.c_int, [_vp, _u64]),
    "hkv_get_epoch": (C.c_int, [_vp, C.POINTER(_u64)]),
    "hkv_clock": (C.c_int, [_vp, C.POINTER(_u64), _vp]),
    "hkv_first_eviction_lambda": (C.c_int, [_vp, C.POINTER(_i32), C.POINTER(C.c_double), _vp]),
    "hkv_counters": (C.c_int, [_vp, C.POINTER(_i64), _vp]),
    "hkv_reset_counters": (C.c_int, [_vp, _vp]),
    "hkv_device_error": (C.c_int, [_vp, C.POINTER(_i32), _vp]),
    "hkv_import_state": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _u64, _i32, C.c_double]),
    "hkv_export_state": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp]),
    "hkv_snapshot": (C.c_int, [_vp, _vp]),
    "hkv_read_rows": (C.c_int, [_vp, _i64, _i64, _vp, _vp, _vp]),
    "hkv_read_value_rows": (C.c_int, [_vp, _i64, _i64, _vp, _vp]),
    "hkv_lookup": (C.c_int, [_vp, _u64, _vp, _vp]),
    "hkv_find_in_bucket": (C.c_int, [_vp, _i64, _u64, _vp, _vp]),
    "hkv_upsert_single": (C.c_int, [_vp, _u64, _vp, _i32, _u64, _vp, _vp]),
    "hkv_upsert_dual": (C.c_int, [_vp, _u64, _vp, _i32, _u64, _vp, _vp]),
    "hkv_restore": (C.c_int, [_vp, _vp]),
    "hkv_check_consistency": (C.c_int, [_vp, C.POINTER(_i32), _vp]),
    "hkv_route": (C.c_int, [_vp, _i64, _i64, _i32, _vp, _vp, _vp]),
    "hkv_route_gather": (C.c_int, [_vp, _i64, _vp, _vp, _vp, _i64, _u64, _vp, _vp, _vp]),
    "hkv_scatter_rows": (C.c_int, [_vp, _i64, _vp, _vp, _i64, _vp]),
    "hkv_set_kernel_timing": (C.c_int, [_i32]),
    "hkv_gate_create": (C.c_int, [C.POINTER(_vp)]),
    "hkv_gate_destroy": (C.c_int, [_vp]),
    "hkv_table_gate": (C.c_int, [_vp, C.POINTER(_vp)]),
    "hkv_gate_set_hook": (C.c_int, [_vp, _vp, _vp]),
    "hkv_gate_acquire": (C.c_int, [_vp, _i32, _i32, _i32, _vp]),
    "hkv_gate_release": (C.c_int, [_vp, _i32, _i32, _i32, _vp]),
    "hkv_gate_state": (C.c_int, [_vp, _vp, _vp, _vp]),
    "hkv_kernel_times": (C.c_int, [C.c_char_p, C.POINTER(C.c_double), C.POINTER(_i64)]),
}

_lib = None


def load(path: str = LIB_PATH):
    """Load libhkv_b200.so; raises (never falls back) when it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build it with `python -m paper_2603_17168_b200.build` "
            "(there is no CPU fallback for the table)")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


class HkvError(RuntimeError):
    pass


def check(rc: int):
    if rc == HKV_OK:
        return
    msg = load().hkv_last_error().decode(errors="replace")
    if rc == HKV_EINVAL:
        raise ValueError(msg)
    if rc == HKV_ENOMEM:
        raise MemoryError(msg)
    raise HkvError(msg)
