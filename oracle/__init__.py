"""Sequential CPU oracle for the ParPaRaw hot path (arXiv 1905.13415).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  It shares no code with ``paper_1905_13415_b200`` (the CUDA path) and
never imports it.

* ``parpa_oracle.c`` — the sequential parse ("A sequential approach would
  simply set the starting state of its DFA and read the symbols of the input
  beginning to end") for three dialects written as explicit control flow, plus a
  generic table walker for random DFAs.  Loaded through ctypes; compiled with gcc
  on first use (``build()``).
* ``primitives.py`` — plain-Python statements of the paper's primitives (the
  SWAR matcher of tab:twiddling, MFIRA layout of fig:multifrag, prefix scans of §2,
  the composite operator ∘ of §3.1 and the column-offset operator ⊕ of §3.2).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "parpa_oracle.c")
_LIB = os.path.join(_HERE, "libparpa_oracle.so")
_lock = threading.Lock()
_lib = None

# dialect ids (parpa_oracle.c)
CSV, CSV_COMMENT, CLF = 0, 1, 2
DIALECTS = {"csv": CSV, "csv_comment": CSV_COMMENT, "clf": CLF}
# emission kinds, EOI actions, column types, status codes (mirrors the paper's readings)
DATA, CTRL, FIELD, RECORD = 0, 1, 2, 3
EOI_NONE, EOI_RECORD, EOI_ERROR = 0, 1, 2
SPAN, INT64, FLOAT64, TIMESTAMP = 0, 1, 2, 3
OK, EFORMAT, ECOLUMNS, EUNSUPPORTED = 0, -4, -5, -6
NONE64 = 0xFFFFFFFFFFFFFFFF
MISSING_LEN = 0xFFFFFFFF


def build(force: bool = False) -> str:
    """Compile parpa_oracle.c into libparpa_oracle.so (plain gcc -O2)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            P = ctypes.c_void_p
            u8p = ctypes.POINTER(ctypes.c_uint8)
            lib.oracle_parse.restype = P
            lib.oracle_parse.argtypes = [ctypes.c_int, u8p, ctypes.c_uint64, ctypes.c_uint32, u8p, u8p,
                                         ctypes.POINTER(ctypes.c_int64), ctypes.c_int, u8p, u8p]
            lib.oracle_parse_tables.restype = P
            lib.oracle_parse_tables.argtypes = [u8p, ctypes.c_uint32, ctypes.c_uint32, u8p, u8p, u8p,
                                                ctypes.c_uint32, ctypes.c_uint32, u8p, ctypes.c_uint64,
                                                ctypes.c_uint32, u8p, u8p, ctypes.POINTER(ctypes.c_int64),
                                                ctypes.c_int, u8p, u8p]
            lib.oracle_stats.argtypes = [P, ctypes.POINTER(ctypes.c_uint64)]
            lib.oracle_column.argtypes = [P, ctypes.c_uint32, P, P, P, P]
            lib.oracle_free.argtypes = [P]
            lib.oracle_conv_int64.argtypes = [u8p, ctypes.c_uint64, ctypes.POINTER(ctypes.c_int64)]
            lib.oracle_conv_float64.argtypes = [u8p, ctypes.c_uint64, ctypes.POINTER(ctypes.c_int64)]
            lib.oracle_conv_timestamp.argtypes = [u8p, ctypes.c_uint64, ctypes.POINTER(ctypes.c_int64)]
            lib.oracle_parse_strings.argtypes = [ctypes.c_int, u8p, ctypes.c_uint64, ctypes.c_uint32, u8p, ctypes.c_uint32]
            lib.oracle_parse_strings.restype = ctypes.c_void_p
            lib.oracle_strings_size.argtypes = [ctypes.c_void_p]
            lib.oracle_strings_size.restype = ctypes.c_uint64
            lib.oracle_strings.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
            _lib = lib
    return _lib


def _u8(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))


def _as_bytes(data) -> np.ndarray:
    if isinstance(data, (bytes, bytearray, memoryview)):
        return np.frombuffer(bytes(data), dtype=np.uint8)
    a = np.ascontiguousarray(data, dtype=np.uint8)
    return a.reshape(-1)


class OracleResult:
    """Columns of one sequential parse (R rows each), plus scalar stats."""

    def __init__(self, R, nfields, first_invalid, n_missing, n_extra, status, final_state, eoi_action,
                 offset, length, value, valid, types, trace_state=None, trace_kind=None):
        self.R = R
        self.nfields = nfields
        self.first_invalid = first_invalid
        self.n_missing = n_missing
        self.n_extra = n_extra
        self.status = status
        self.final_state = final_state
        self.eoi_action = eoi_action
        self.offset = offset      # list[C] of uint64[R]
        self.length = length      # list[C] of uint32[R]
        self.value = value        # list[C] of int64[R] (float64 columns: IEEE bits) or None for spans
        self.valid = valid        # list[C] of uint8[R] or None for spans
        self.types = types
        self.trace_state = trace_state
        self.trace_kind = trace_kind

    def fields(self, data, c):
        """Raw span bytes of column c (None for missing fields)."""
        d = _as_bytes(data)
        out = []
        for o, n in zip(self.offset[c].tolist(), self.length[c].tolist()):
            out.append(None if n == MISSING_LEN else bytes(d[o:o + n]))
        return out

    def floats(self, c):
        return self.value[c].view(np.float64)


def _schema_arrays(C, types, defaults):
    types = [SPAN] * C if types is None else list(types)
    assert len(types) == C
    has_def = np.zeros(max(C, 1), np.uint8)
    def_bits = np.zeros(max(C, 1), np.int64)
    if defaults is not None:
        for c, d in enumerate(defaults):
            if d is None:
                continue
            has_def[c] = 1
            if types[c] == FLOAT64:
                def_bits[c] = np.array([float(d)], np.float64).view(np.int64)[0]
            else:
                def_bits[c] = int(d)
    return np.array(types + [0], np.uint8), has_def, def_bits, types


def _collect(lib, h, C, types, trace_state, trace_kind):
    st = (ctypes.c_uint64 * 8)()
    lib.oracle_stats(h, st)
    R = int(st[0])
    offs, lens, vals, valids = [], [], [], []
    for c in range(C):
        o = np.empty(R, np.uint64)
        n = np.empty(R, np.uint32)
        v = np.empty(R, np.int64)
        ok = np.empty(R, np.uint8)
        if R:
            lib.oracle_column(h, c, o.ctypes.data, n.ctypes.data, v.ctypes.data, ok.ctypes.data)
        offs.append(o)
        lens.append(n)
        vals.append(v if types[c] != SPAN else None)
        valids.append(ok if types[c] != SPAN else None)
    lib.oracle_free(h)
    status = ctypes.c_int64(st[5]).value
    return OracleResult(R, int(st[1]), int(st[2]), int(st[3]), int(st[4]), status, int(st[6]), int(st[7]),
                        offs, lens, vals, valids, types, trace_state, trace_kind)


def parse(dialect, data, C: int, types=None, defaults=None, strict=False, trace=False) -> OracleResult:
    """Sequential parse of ``data`` under a hand-written dialect ("csv", "csv_comment", "clf")."""
    lib = _load()
    d = _as_bytes(data)
    dialect = DIALECTS[dialect] if isinstance(dialect, str) else int(dialect)
    t, hd, db, types = _schema_arrays(C, types, defaults)
    ts = np.empty(len(d), np.uint8) if trace else None
    tk = np.empty(len(d), np.uint8) if trace else None
    dd = d if len(d) else np.zeros(1, np.uint8)
    h = lib.oracle_parse(dialect, _u8(dd), len(d), C, _u8(t), _u8(hd),
                         db.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), int(strict),
                         _u8(ts) if trace else None, _u8(tk) if trace else None)
    return _collect(lib, h, C, types, ts, tk)


def parse_tables(tables, data, C: int, types=None, defaults=None, strict=False, trace=False) -> OracleResult:
    """Sequential parse driven by explicit DFA tables (the generic table walker).

    ``tables``: dict with group_of_byte[256], transition[G][S], emit[G][S], eoi[S], start, invalid.
    """
    lib = _load()
    d = _as_bytes(data)
    gob = np.ascontiguousarray(tables["group_of_byte"], np.uint8)
    tr = np.ascontiguousarray(tables["transition"], np.uint8)
    em = np.ascontiguousarray(tables["emit"], np.uint8)
    eoi = np.ascontiguousarray(tables["eoi"], np.uint8)
    G, S = tr.shape
    t, hd, db, types = _schema_arrays(C, types, defaults)
    ts = np.empty(len(d), np.uint8) if trace else None
    tk = np.empty(len(d), np.uint8) if trace else None
    dd = d if len(d) else np.zeros(1, np.uint8)
    h = lib.oracle_parse_tables(_u8(gob), S, G, _u8(tr), _u8(em), _u8(eoi), int(tables["start"]),
                                int(tables["invalid"]), _u8(dd), len(d), C, _u8(t), _u8(hd),
                                db.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), int(strict),
                                _u8(ts) if trace else None, _u8(tk) if trace else None)
    return _collect(lib, h, C, types, ts, tk)


def conv_int64(s: bytes):
    """R14: (ok, value)."""
    lib = _load()
    a = np.frombuffer(s + b"\0", np.uint8)
    v = ctypes.c_int64(0)
    ok = lib.oracle_conv_int64(_u8(a), len(s), ctypes.byref(v))
    return bool(ok), v.value if ok else 0


def strings(dialect, data, C: int, col: int, types=None):
    """SURVEY N3 (the paper's CSS): the DATA bytes of every field of column ``col``
    concatenated in row order (control bytes dropped; missing fields empty).  Returns
    (offsets int64[R + 1], data bytes)."""
    lib = _load()
    d = _as_bytes(data)
    dialect = DIALECTS[dialect] if isinstance(dialect, str) else int(dialect)
    t, _, _, _ = _schema_arrays(C, types, None)
    dd = d if len(d) else np.zeros(1, np.uint8)
    h = lib.oracle_parse_strings(dialect, _u8(dd), len(d), C, _u8(t), col)
    st = (ctypes.c_uint64 * 8)()
    lib.oracle_stats(h, st)
    R = int(st[0])
    n = int(lib.oracle_strings_size(h))
    offs = np.zeros(R + 1, np.int64)
    buf = np.zeros(max(n, 1), np.uint8)
    lib.oracle_strings(h, offs.ctypes.data, buf.ctypes.data)
    lib.oracle_free(h)
    return offs, bytes(buf[:n])


CSS_ARROW, CSS_INLINE, CSS_VECTOR = 0, 1, 2


def css(dialect, data, C: int, col: int, types=None, mode=CSS_ARROW, terminator=0x1F):
    """The column's CSS in one of the paper's layouts (alternative tagging modes P:493-502),
    written out from ``strings`` (the DATA bytes of each field, in row order):
      CSS_ARROW  -> (offsets, data)
      CSS_INLINE -> (offsets, data): "replaces delimiters with a terminator": every field's bytes
                    followed by the terminator; offsets[r] = start of field r (its terminator at
                    offsets[r + 1] - 1)
      CSS_VECTOR -> (offsets, data, aux): "its own auxiliary boolean vector that delimits the fields"
                    (P:499): the ARROW bytes, aux = 1 at the last symbol of every non-empty field
    Plain Python loops over the fields."""
    offs, buf = strings(dialect, data, C, col, types)
    R = len(offs) - 1
    if mode == CSS_ARROW:
        return offs, buf
    if mode == CSS_INLINE:
        out, o2 = bytearray(), [0]
        for r in range(R):
            out += buf[offs[r]:offs[r + 1]]
            out.append(terminator)
            o2.append(len(out))
        return np.array(o2, np.int64), bytes(out)
    aux = bytearray(len(buf))
    for r in range(R):
        if offs[r + 1] > offs[r]:
            aux[offs[r + 1] - 1] = 1
    return offs, buf, bytes(aux)


def css_index(mode, buf: bytes, terminator=0x1F):
    """The CSS index as P:497 / P:501-502 generate it: the positions of all terminators (CSS_INLINE) or of
    the nonzero auxiliary entries (CSS_VECTOR), in order."""
    if mode == CSS_INLINE:
        return np.array([k for k, c in enumerate(buf) if c == terminator], np.int64)
    return np.array([k for k, c in enumerate(buf) if c != 0], np.int64)


def conv_timestamp(s: bytes):
    """R29: (ok, seconds since 1970-01-01T00:00:00Z) for ISO or CLF datetimes."""
    lib = _load()
    a = np.frombuffer(s + b"\0", np.uint8)
    v = ctypes.c_int64(0)
    ok = lib.oracle_conv_timestamp(_u8(a), len(s), ctypes.byref(v))
    return bool(ok), v.value if ok else 0


def conv_float64(s: bytes):
    """R15: (ok, IEEE-754 bits as int64)."""
    lib = _load()
    a = np.frombuffer(s + b"\0", np.uint8)
    v = ctypes.c_int64(0)
    ok = lib.oracle_conv_float64(_u8(a), len(s), ctypes.byref(v))
    return bool(ok), v.value if ok else 0


# ---- type inference (reading R31) ------------------------------------------------
CLASSES = ("empty", "int8", "int16", "int32", "int64", "float64", "timestamp", "string")


def field_class(s: bytes) -> str:
    """R31: the minimal type backing one field's DATA bytes ("the minimum numerical type being
    required to back their field value"), extended to temporal types."""
    if not s:
        return "empty"
    ok, v = conv_int64(s)
    if ok:
        for name, bits in (("int8", 8), ("int16", 16), ("int32", 32)):
            if -(1 << (bits - 1)) <= v < (1 << (bits - 1)):
                return name
        return "int64"
    if conv_float64(s)[0]:
        return "float64"
    if conv_timestamp(s)[0]:
        return "timestamp"
    return "string"


def resolve_types(classes) -> str:
    """P:572 "a subsequent parallel reduction over the minimum type yields the inferred type of a
    column": the widest numeric class; timestamps only with timestamps; anything else a string."""
    present = set(classes) - {"empty"}
    if not present:
        return "empty"
    if "string" in present or ("timestamp" in present and len(present) > 1):
        return "string"
    if present == {"timestamp"}:
        return "timestamp"
    return max(present, key=CLASSES.index)


def infer_types(dialect, data, C: int):
    """Per column c < C: (type, set of field classes) from the sequential parse's DATA bytes."""
    out = []
    for c in range(C):
        offs, buf = strings(dialect, data, C, c)
        cls = {field_class(buf[offs[i]:offs[i + 1]]) for i in range(len(offs) - 1)}
        out.append((resolve_types(cls), cls - {"empty"}))
    return out
