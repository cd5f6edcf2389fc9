"""Seeded synthetic inputs shaped like the paper's workloads (input generator only).

This module is the one piece both sides of the parity tests share: it produces
bytes and workload descriptions (dialect name, column types) and holds none of the
method's arithmetic.  See ``parpa_gen.c`` for the record recipes and DESIGN.md
§Inputs for the distributions.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "parpa_gen.c")
_LIB = os.path.join(_HERE, "libparpa_gen.so")
_lock = threading.Lock()
_lib = None
MAX_INT_COLS = 8

SPAN, INT64, FLOAT64 = 0, 1, 2
I, F, S = INT64, FLOAT64, SPAN


@dataclass(frozen=True)
class Workload:
    name: str
    gen_id: int
    seed: int
    target_bytes: int
    dialect: str          # "csv" | "csv_comment" | "clf"
    types: tuple          # column types
    description: str

    @property
    def C(self) -> int:
        return len(self.types)


WORKLOADS = {
    "cfg1": Workload("cfg1", 0, 1, 1_000_000, "csv", (I, I, F, S, F, S, I, S),
                     "1 MB RFC-4180 CSV, 8 int/float/string columns, ~10% quoted fields with "
                     "embedded commas/newlines/\"\" escapes"),
    "taxi": Workload("taxi", 1, 2, 4_800_000_000, "csv",
                     (I, S, S, I, F, I, S, I, I, I, F, F, F, F, F, F, F, F),
                     "NYC-taxi-shaped CSV, 4.8 GB, 18 numeric/datetime columns, unquoted"),
    "yelp": Workload("yelp", 2, 3, 4_823_000_000, "csv", (S, S, S, I, I, I, I, S, S),
                     "Yelp-reviews-shaped CSV, 4.823 GB, all fields quoted, long multi-line text "
                     "with escaped quotes"),
    "clf": Workload("clf", 3, 4, 8_000_000_000, "clf", (S, S, S, S, S, I, I),
                    "Common-Log-Format-shaped logs, 8 GB, bracketed timestamps, quoted requests, "
                    "'#' directive lines (9-state DFA)"),
    "taxi64": Workload("taxi64", 1, 5, 64_000_000_000, "csv",
                       (I, S, S, I, F, I, S, I, I, I, F, F, F, F, F, F, F, F),
                       "64 GB taxi-shaped CSV sharded across GPUs"),
}


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=gnu11", "-shared", "-fPIC", "-pthread", "-o", tmp, _SRC,
                               "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            lib.gen_fill.restype = ctypes.c_uint64
            lib.gen_fill.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                     ctypes.c_uint64, ctypes.c_void_p, ctypes.c_int,
                                     ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_int64)]
            lib.gen_one.restype = ctypes.c_uint64
            lib.gen_one.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_void_p]
            _lib = lib
    return _lib


@dataclass
class Generated:
    nbytes: int
    records: int
    int_sums: list      # wrapping int64 sum per int64 column, in column order
    int_nulls: list     # null count per int64 column


def fill(workload, out_ptr: int, capacity: int, first_record: int = 0, threads: int | None = None,
         max_records: int | None = None, seed: int | None = None) -> Generated:
    """Generate records first_record, first_record+1, ... into ``capacity`` bytes at ``out_ptr``
    (truncated at the last whole record).  Returns the exact size and ground truth (pin G1)."""
    w = WORKLOADS[workload] if isinstance(workload, str) else workload
    lib = _load()
    threads = threads or min(32, os.cpu_count() or 1)
    R = ctypes.c_uint64(0)
    gt = (ctypes.c_int64 * (2 * MAX_INT_COLS))()
    n = lib.gen_fill(w.gen_id, w.seed if seed is None else seed, first_record, capacity,
                     max_records if max_records is not None else (1 << 62), out_ptr, threads,
                     ctypes.byref(R), gt)
    nint = sum(1 for t in w.types if t == INT64)
    return Generated(int(n), int(R.value), [int(gt[i]) for i in range(nint)],
                     [int(gt[MAX_INT_COLS + i]) for i in range(nint)])


def generate(workload, nbytes: int | None = None, first_record: int = 0, threads: int | None = None,
             max_records: int | None = None, seed: int | None = None):
    """Generate into a fresh numpy array; returns (array[N], Generated)."""
    w = WORKLOADS[workload] if isinstance(workload, str) else workload
    cap = w.target_bytes if nbytes is None else nbytes
    buf = np.empty(max(cap, 1), np.uint8)
    g = fill(w, buf.ctypes.data, cap, first_record, threads, max_records, seed)
    return buf[:g.nbytes], g


def record(workload, index: int, seed: int | None = None) -> bytes:
    w = WORKLOADS[workload] if isinstance(workload, str) else workload
    lib = _load()
    buf = np.empty(1 << 17, np.uint8)
    n = lib.gen_one(w.gen_id, w.seed if seed is None else seed, index, buf.ctypes.data)
    return bytes(buf[:n])
