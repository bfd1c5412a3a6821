"""ctypes binding of libfailsafe_b200.so (the C ABI in include/failsafe_b200.h).

The library is built in-tree (``paper_2511_14116_b200/lib``) by
``paper_2511_14116_b200.build``.  There is no fallback: if the library is
missing the import of this module raises, loudly.
"""

from __future__ import annotations

import ctypes as C
import os

from .core import SimulationError, ValidationError

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "lib", "libfailsafe_b200.so")

FS_OK, FS_EVALIDATION, FS_ESIMULATION, FS_ECUDA = 0, 1, 2, 3
REPLICATED = -1
PAGE_TOKENS = 16
HEAD_DIM = 128
PAGE_BYTES = 8192
MAX_Q_PER_KV = 8
FS_AR_MAX_WORLD = 16
MODES = {"naive": 0, "cyclic": 1, "hybrid": 2}

_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)


class DecodeDesc(C.Structure):
    """Mirror of ``fs_decode_desc``."""

    _fields_ = [
        ("q", C.c_void_p), ("kv_pool", C.c_void_p), ("block_table", C.c_void_p),
        ("bt_stride", C.c_int64), ("item_seq", C.c_void_p), ("item_len", C.c_void_p),
        ("item_qoff", C.c_void_p), ("item_ooff", C.c_void_p), ("page_off", C.c_void_p),
        ("kv_new", C.c_void_p), ("item_koff", C.c_void_p), ("item_voff", C.c_void_p),
        ("item_sem", C.c_void_p), ("n_items", C.c_int32), ("q_per_kv", C.c_int32), ("scale", C.c_float),
        ("out_fp32", C.c_int32), ("out", C.c_void_p), ("part_o", C.c_void_p),
        ("part_lse", C.c_void_p), ("partial_slots", C.c_int64), ("device", C.c_int32),
        ("config", C.c_int32), ("flags", C.c_int32),
    ]


DECODE_EARLY_PREFETCH = 1  # FS_DECODE_EARLY_PREFETCH


class PrefillDesc(C.Structure):
    """Mirror of ``fs_prefill_desc``."""

    _fields_ = [
        ("q", C.c_void_p), ("out", C.c_void_p), ("q_stride", C.c_int64), ("o_stride", C.c_int64),
        ("out_fp32", C.c_int32), ("kv_pool", C.c_void_p), ("block_table", C.c_void_p), ("bt_stride", C.c_int64),
        ("item_seq", C.c_void_p), ("item_start", C.c_void_p), ("item_len", C.c_void_p),
        ("item_qoff", C.c_void_p), ("item_ooff", C.c_void_p),
        ("tile_item", C.c_void_p), ("tile_tok0", C.c_void_p), ("tile_page0", C.c_void_p),
        ("tile_page1", C.c_void_p), ("tile_slot", C.c_void_p), ("n_tiles", C.c_int32),
        ("comb_item", C.c_void_p), ("comb_tok0", C.c_void_p), ("comb_slot0", C.c_void_p),
        ("comb_nsplit", C.c_void_p), ("n_comb", C.c_int32), ("q_per_kv", C.c_int32),
        ("scale", C.c_float), ("part_o", C.c_void_p), ("part_lse", C.c_void_p),
        ("partial_slots", C.c_int64), ("variant", C.c_int32),
    ]


# name -> (restype, argtypes)
_SIGS = {
    "fs_abi_version": (C.c_int, []),
    "fs_last_error": (C.c_char_p, []),
    "fs_device_sms": (C.c_int, [C.c_int]),
    "fs_plan_placement": (C.c_int, [C.c_int, C.c_int, C.c_int, _i32p, C.c_int, _i32p]),
    "fs_plan_ffn": (C.c_int, [C.c_int, _i32p, C.c_int, _i32p]),
    "fs_plan_on_demand": (C.c_int, [C.c_int, C.c_int, _i32p, C.c_int, _i32p, _i32p, C.c_int,
                                    _i32p, _i32p]),
    "fs_kv_footprint": (C.c_int, [C.c_int, C.c_int, _i32p, _i32p, C.c_int, _i64p, _i32p,
                                  C.c_int, C.c_int64, _i64p]),
    "fs_plan_pages": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]),
    "fs_decode_partial_slots": (C.c_int64, [C.c_int, C.c_int32, C.c_int32]),
    "fs_decode_attention": (C.c_int, [C.POINTER(DecodeDesc), C.c_void_p]),
    "fs_prefill_tokens_per_tile": (C.c_int, [C.c_int, C.c_int]),
    "fs_plan_prefill_tiles": (C.c_int, [C.c_int32, _i32p, _i32p, C.c_int32, C.c_int32, C.c_int32,
                                        C.c_int32,
                                        _i32p, _i32p, _i32p, _i32p, _i32p, _i32p, C.c_int32,
                                        _i32p, _i32p, _i32p, _i32p, _i32p, _i32p]),
    "fs_prefill_attention": (C.c_int, [C.POINTER(PrefillDesc), C.c_void_p]),
    "fs_kv_write": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                              C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_int64,
                              C.c_void_p]),
    "fs_kv_write_runs": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                                   C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                                   C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]),
    "fs_kv_read": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                             C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_int64,
                             C.c_void_p]),
    "fs_pages_gather": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p,
                                  C.c_int32, C.c_void_p]),
    "fs_pages_scatter": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p,
                                   C.c_int32, C.c_void_p]),
    "fs_kv_backup_tokens": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p,
                                      C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p]),
    "fs_host_register": (C.c_int, [C.c_void_p, C.c_int64, C.POINTER(C.c_void_p)]),
    "fs_host_unregister": (C.c_int, [C.c_void_p]),
    "fs_copy_2d": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_int64,
                             C.c_int64, C.c_void_p]),
    "fs_copy_segments": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p]),
    "fs_gemm_workspace_floats": (C.c_int64, [C.c_int, C.c_int32, C.c_int32]),
    "fs_gemm_skinny": (C.c_int, [C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_void_p,
                                 C.c_int64, C.c_int32, C.c_int32, C.c_void_p, C.c_int64, C.c_void_p,
                                 C.c_int64, C.c_int32, C.c_void_p, C.c_int64, C.c_void_p,
                                 C.c_int32, C.c_void_p]),
    "fs_gemm_plan": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_int32]),
    "fs_swiglu": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_void_p, C.c_int64,
                            C.c_void_p]),
    "fs_fill_normal": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_void_p,
                                 C.c_int64, C.c_void_p, C.c_int64, C.c_uint64, C.c_uint64,
                                 C.c_float, C.c_void_p]),
    "fs_ar_buffer_bytes": (C.c_int64, [C.c_int64]),
    "fs_ar_alloc": (C.c_int, [C.c_int, C.c_int64, C.POINTER(C.c_void_p)]),
    "fs_ar_free": (C.c_int, [C.c_void_p]),
    "fs_ar_ipc_handle": (C.c_int, [C.c_void_p, C.c_void_p]),
    "fs_ar_ipc_open": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "fs_ar_ipc_close": (C.c_int, [C.c_void_p]),
    "fs_ar_residual": (C.c_int, [C.POINTER(C.c_void_p), C.c_int32, C.c_int32, C.c_int64,
                                 C.c_int64, C.c_void_p, C.c_int32, C.c_void_p]),
    "fs_ar_residual_mode": (C.c_int, [C.POINTER(C.c_void_p), C.c_int32, C.c_int32, C.c_int64,
                                      C.c_int64, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p]),
    "fs_enable_peer": (C.c_int, [C.c_int, C.c_int]),
    "fs_copy_peer": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_int64,
                               C.c_void_p]),
    "fs_gemm_debug_timestamps": (None, [C.c_void_p]),
}

EXPORTS = tuple(_SIGS)


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python paper_2511_14116_b200/build.py` "
            "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.fs_abi_version() != 1:
        raise ImportError("libfailsafe_b200 ABI version mismatch")
    return lib


lib = _load()


def check(rc, what=""):
    """Map a C-ABI status to the reference's exception classes."""
    if rc == FS_OK:
        return
    msg = (lib.fs_last_error() or b"").decode(errors="replace")
    if what:
        msg = f"{what}: {msg}"
    if rc == FS_EVALIDATION:
        raise ValidationError(msg)
    raise SimulationError(msg)


def i32_array(values):
    vals = [int(v) for v in values]
    return (C.c_int32 * max(1, len(vals)))(*vals), len(vals)


def i64_array(values):
    vals = [int(v) for v in values]
    return (C.c_int64 * max(1, len(vals)))(*vals), len(vals)


def ptr(t):
    """Raw device/host pointer of a torch tensor (None-safe)."""
    return None if t is None else C.c_void_p(t.data_ptr())
