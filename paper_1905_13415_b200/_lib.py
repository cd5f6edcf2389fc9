"""ctypes declarations for libparpa.so (include/parpa.h).  Argument marshalling only."""
from __future__ import annotations

import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PARPA_LIB") or os.path.join(HERE, "libparpa.so")  # PARPA_LIB: A/B builds

c_u8p = ctypes.POINTER(ctypes.c_uint8)


class Schema_t(ctypes.Structure):
    _fields_ = [("num_columns", ctypes.c_uint32), ("types", c_u8p), ("has_default", c_u8p),
                ("default_bits", ctypes.POINTER(ctypes.c_int64)), ("strict", ctypes.c_uint32)]


class Column_t(ctypes.Structure):
    _fields_ = [("offset", ctypes.c_void_p), ("length", ctypes.c_void_p), ("value", ctypes.c_void_p),
                ("valid", ctypes.c_void_p)]


class Stats_t(ctypes.Structure):
    _fields_ = [("records", ctypes.c_uint64), ("fields", ctypes.c_uint64), ("first_invalid", ctypes.c_uint64),
                ("missing_records", ctypes.c_uint64), ("extra_fields", ctypes.c_uint64),
                ("deferred_fields", ctypes.c_uint64), ("status", ctypes.c_int32), ("final_state", ctypes.c_uint32),
                ("block_fields", ctypes.c_uint32), ("device_fields", ctypes.c_uint32)]


class Tau_t(ctypes.Structure):
    _fields_ = [("tau", ctypes.c_uint8 * 16)]


class Counts_t(ctypes.Structure):
    _fields_ = [("records", ctypes.c_uint64), ("fields", ctypes.c_uint64), ("open_first", ctypes.c_uint64),
                ("open_last", ctypes.c_uint64), ("column", ctypes.c_uint32), ("flags", ctypes.c_uint32),
                ("first_invalid", ctypes.c_uint64)]


class Context_t(ctypes.Structure):
    _fields_ = [("entry_state", ctypes.c_uint32), ("_pad", ctypes.c_uint32), ("base", ctypes.c_uint64),
                ("prefix", Counts_t)]


STATS_BYTES = ctypes.sizeof(Stats_t)
assert STATS_BYTES == 64

_lock = threading.Lock()
_lib = None

EXPORTS = [
    "parpa_create_dfa", "parpa_destroy_dfa", "parpa_parse", "parpa_result_stats", "parpa_result_column",
    "parpa_result_records", "parpa_result_status", "parpa_set_allocator",
    "parpa_workspace_create", "parpa_workspace_destroy", "parpa_parse_into_ws",
    "parpa_result_copy_column", "parpa_result_free", "parpa_plan_create", "parpa_plan_records", "parpa_plan_emit", "parpa_plan_destroy",
    "parpa_parse_into", "parpa_parse_host", "parpa_summarize", "parpa_count", "parpa_compose_tau",
    "parpa_compose_counts", "parpa_parse_range", "parpa_range_begin", "parpa_range_count", "parpa_range_emit",
    "parpa_range_state_at", "parpa_range_emit_halo", "parpa_parse_into_skip",
    "parpa_compact_rows",
    "parpa_strings_size", "parpa_strings_copy", "parpa_plan_strings_size", "parpa_plan_strings_copy",
    "parpa_css_index", "parpa_infer_columns", "parpa_infer_types",
    "parpa_debug_trace", "parpa_debug_masks", "parpa_chunk_bytes", "parpa_tile_bytes",
    "parpa_set_profiling", "parpa_last_kernel_times", "parpa_status_string", "parpa_version",
    "parpa_last_error",
]


def load(build_if_missing: bool = True):
    """Load libparpa.so (building it in-tree with nvcc if missing).  Raises if it cannot be loaded:
    there is no CPU fallback."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if build_if_missing and not os.environ.get("PARPA_LIB"):
            from . import build as _build
            try:
                _build.build()
            except Exception:
                if not os.path.exists(LIB_PATH):
                    raise
        lib = ctypes.CDLL(LIB_PATH)
        P = ctypes.c_void_p
        pp = ctypes.POINTER(ctypes.c_void_p)
        u32, u64 = ctypes.c_uint32, ctypes.c_uint64
        lib.parpa_create_dfa.argtypes = [u32, u32, u32, u32, c_u8p, c_u8p, c_u8p, c_u8p, pp]
        lib.parpa_destroy_dfa.argtypes = [P]
        lib.parpa_destroy_dfa.restype = None
        lib.parpa_parse.argtypes = [P, ctypes.POINTER(Schema_t), P, u64, P, pp]
        lib.parpa_result_stats.argtypes = [P, ctypes.POINTER(Stats_t)]
        lib.parpa_result_records.argtypes = [P, ctypes.POINTER(u64)]
        lib.parpa_result_status.argtypes = [P, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(u64), ctypes.POINTER(u64),
                                            ctypes.POINTER(u64)]
        lib.parpa_set_allocator.argtypes = [P, P, P]
        lib.parpa_workspace_create.argtypes = [u64, P, pp]
        lib.parpa_workspace_destroy.argtypes = [P]
        lib.parpa_workspace_destroy.restype = None
        lib.parpa_parse_into_ws.argtypes = [P, P, ctypes.POINTER(Schema_t), P, u64, ctypes.POINTER(Column_t), u64, P, P,
                                            ctypes.POINTER(u32)]
        lib.parpa_result_column.argtypes = [P, u32, ctypes.POINTER(Column_t)]
        lib.parpa_result_copy_column.argtypes = [P, u32, ctypes.POINTER(Column_t), P]
        lib.parpa_result_free.argtypes = [P]
        lib.parpa_result_free.restype = None
        lib.parpa_plan_create.argtypes = [P, P, u64, P, pp]
        lib.parpa_plan_records.argtypes = [P, ctypes.POINTER(u64)]
        lib.parpa_plan_emit.argtypes = [P, ctypes.POINTER(Schema_t), ctypes.POINTER(Column_t), P, P]
        lib.parpa_plan_destroy.argtypes = [P]
        lib.parpa_plan_destroy.restype = None
        lib.parpa_parse_into.argtypes = [P, ctypes.POINTER(Schema_t), P, u64, ctypes.POINTER(Column_t), u64, P, P,
                                         ctypes.POINTER(u32)]
        lib.parpa_parse_host.argtypes = [P, ctypes.POINTER(Schema_t), P, u64, ctypes.POINTER(Column_t), u64,
                                         ctypes.POINTER(Stats_t), P]
        lib.parpa_summarize.argtypes = [P, P, u64, P, ctypes.POINTER(Tau_t)]
        lib.parpa_count.argtypes = [P, P, u64, u64, u32, P, ctypes.POINTER(Counts_t), ctypes.POINTER(Tau_t)]
        lib.parpa_compose_tau.argtypes = [P, ctypes.POINTER(Tau_t), ctypes.POINTER(Tau_t), ctypes.POINTER(Tau_t)]
        lib.parpa_compose_counts.argtypes = [ctypes.POINTER(Counts_t), ctypes.POINTER(Counts_t),
                                             ctypes.POINTER(Counts_t)]
        lib.parpa_infer_columns.argtypes = [P, P, u64, P, ctypes.POINTER(u32), ctypes.POINTER(u32), ctypes.POINTER(u64)]
        lib.parpa_infer_types.argtypes = [P, P, u64, u32, P, P, P, ctypes.POINTER(u64)]
        lib.parpa_strings_size.argtypes = [P, P, u64, ctypes.POINTER(Column_t), u64, P, ctypes.POINTER(u64), P]
        lib.parpa_strings_copy.argtypes = [P, P, u64, ctypes.POINTER(Column_t), u64, P, P, P]
        lib.parpa_plan_strings_size.argtypes = [P, ctypes.POINTER(Column_t), u64, u32, P, ctypes.POINTER(u64), P]
        lib.parpa_plan_strings_copy.argtypes = [P, ctypes.POINTER(Column_t), u64, u32, u32, P, P, P, P]
        lib.parpa_css_index.argtypes = [u32, u32, P, P, u64, P, ctypes.POINTER(u64), P]
        lib.parpa_range_begin.argtypes = [P, P, u64, u64, P, pp, ctypes.POINTER(Tau_t)]
        lib.parpa_range_count.argtypes = [P, u32, ctypes.POINTER(Counts_t)]
        lib.parpa_range_emit.argtypes = [P, ctypes.POINTER(Schema_t), ctypes.POINTER(Context_t), P, u64,
                                         ctypes.c_int, ctypes.POINTER(Column_t), u64, P, P]
        lib.parpa_range_state_at.argtypes = [P, u64, ctypes.POINTER(u32)]
        lib.parpa_compact_rows.argtypes = [P, u64, P, u64, P, ctypes.POINTER(u64), P]
        lib.parpa_parse_into_skip.argtypes = [P, ctypes.POINTER(Schema_t), P, u64, P, u64, ctypes.POINTER(Column_t),
                                              u64, P, P, ctypes.POINTER(u32)]
        lib.parpa_range_emit_halo.argtypes = [P, ctypes.POINTER(Schema_t), ctypes.POINTER(Context_t), P, u64, u32,
                                              ctypes.c_int, ctypes.POINTER(Column_t), u64, P, P]
        lib.parpa_parse_range.argtypes = [P, ctypes.POINTER(Schema_t), P, u64, ctypes.POINTER(Context_t), P, u64,
                                          ctypes.c_int, ctypes.POINTER(Column_t), u64, P, P]
        lib.parpa_debug_trace.argtypes = [P, P, u64, P, P, P, P]
        lib.parpa_debug_masks.argtypes = [P, P, u64, P, P]
        lib.parpa_chunk_bytes.restype = u32
        lib.parpa_tile_bytes.restype = u32
        lib.parpa_set_profiling.argtypes = [ctypes.c_int]
        lib.parpa_last_kernel_times.argtypes = [ctypes.POINTER(ctypes.c_char_p), ctypes.POINTER(ctypes.c_float),
                                                ctypes.c_int]
        lib.parpa_status_string.restype = ctypes.c_char_p
        lib.parpa_status_string.argtypes = [ctypes.c_int]
        lib.parpa_version.restype = ctypes.c_char_p
        lib.parpa_last_error.restype = ctypes.c_char_p
        _lib = lib
        return lib
