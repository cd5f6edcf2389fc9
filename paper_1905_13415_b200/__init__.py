"""paper_1905_13415_b200 — B200-native (sm_100a) ParPaRaw hot path (arXiv 1905.13415).

Thin Python binding over the C ABI of ``libparpa.so`` (include/parpa.h).  Every step of the
path runs in the library's CUDA kernels; this module only marshals arguments.  PyTorch is
used for device memory (tensors) and streams.  There is no CPU fallback: if the extension
cannot be loaded, every entry point raises.

    import paper_1905_13415_b200 as parpa
    dfa = parpa.Dfa.dialect("csv")                              # tab:ttable
    schema = parpa.Schema([parpa.INT64, parpa.SPAN, parpa.FLOAT64])
    res = parpa.parse(dfa, schema, data)                        # data: torch.uint8 CUDA tensor
    res.records, res.columns[2].value, res.stats
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

from . import _lib
from . import dialects

SPAN, INT64, FLOAT64, TIMESTAMP = 0, 1, 2, 3
DATA, CTRL, FIELD, RECORD = 0, 1, 2, 3
OK, EINVAL, ENOMEM, ECUDA, EFORMAT, ECOLUMNS, EUNSUPPORTED, ENEEDMORE = 0, -1, -2, -3, -4, -5, -6, -7
MISSING_LENGTH = 0xFFFFFFFF
NONE = 0xFFFFFFFFFFFFFFFF


class ParpaError(RuntimeError):
    def __init__(self, code, what=""):
        lib = _lib.load()
        detail = lib.parpa_last_error().decode() if code == -3 else ""
        super().__init__(f"{what}: {lib.parpa_status_string(code).decode()} ({code}) {detail}")
        self.code = code


def _check(rc, what):
    if rc != OK:
        raise ParpaError(rc, what)


def lib():
    return _lib.load()


def _stream_handle(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _u8(buf):
    return ctypes.cast(buf, _lib.c_u8p)


class Dfa:
    """A compiled parsing DFA (parpa_create_dfa).  Row-per-group tables."""

    def __init__(self, num_states, start, invalid, group_of_byte, transition, emit, eoi, name="custom"):
        L = _lib.load()
        G = len(transition)
        S = num_states
        gob = (ctypes.c_uint8 * 256)(*group_of_byte)
        tr = (ctypes.c_uint8 * (G * S))(*[v for row in transition for v in row])
        em = (ctypes.c_uint8 * (G * S))(*[v for row in emit for v in row])
        eo = (ctypes.c_uint8 * S)(*eoi)
        h = ctypes.c_void_p()
        _check(L.parpa_create_dfa(S, start, invalid, G, _u8(gob), _u8(tr), _u8(em), _u8(eo), ctypes.byref(h)),
               "parpa_create_dfa")
        self._h = h
        self.name = name
        self.num_states = S
        self.start = start
        self.invalid = invalid
        self.tables = {"group_of_byte": list(group_of_byte), "transition": [list(r) for r in transition],
                       "emit": [list(r) for r in emit], "eoi": list(eoi), "start": start, "invalid": invalid}

    @classmethod
    def from_tables(cls, t: "dialects.DfaTables"):
        return cls(t.S, t.start, t.invalid, t.group_of_byte, t.transition, t.emit, t.eoi, name=t.name)

    @classmethod
    def dialect(cls, name: str):
        return cls.from_tables(dialects.get(name))

    @property
    def handle(self):
        return self._h

    def __del__(self):
        try:
            h = getattr(self, "_h", None)
            if h is not None and h.value and _lib._lib is not None:
                _lib._lib.parpa_destroy_dfa(h)
                self._h = None
        except Exception:  # interpreter shutdown
            pass


@dataclass
class Schema:
    """Column types (SPAN / INT64 / FLOAT64), optional defaults for empty / missing typed fields
    (P:564-568), strict column count."""
    types: list
    defaults: list | None = None
    strict: bool = False

    @property
    def C(self):
        return len(self.types)

    def struct(self):
        C = self.C
        self._t = (ctypes.c_uint8 * max(C, 1))(*self.types)
        self._hd = (ctypes.c_uint8 * max(C, 1))()
        self._db = (ctypes.c_int64 * max(C, 1))()
        if self.defaults is not None:
            import struct as _st
            for c, d in enumerate(self.defaults):
                if d is None:
                    continue
                self._hd[c] = 1
                if self.types[c] == FLOAT64:
                    self._db[c] = _st.unpack("<q", _st.pack("<d", float(d)))[0]
                else:
                    self._db[c] = int(d)
        return _lib.Schema_t(C, _u8(self._t), _u8(self._hd), ctypes.cast(self._db, ctypes.POINTER(ctypes.c_int64)),
                             int(self.strict))


class Column:
    """One output column as torch tensors: offset u64 (int64 storage), length u32 (int32 storage),
    value int64 / float64 (typed only), valid uint8 (typed only)."""

    def __init__(self, offset, length, value=None, valid=None):
        self.offset, self.length, self.value, self.valid = offset, length, value, valid

    def struct(self):
        if self.offset is None:                                   # skipped column
            return _lib.Column_t(None, None, None, None)
        return _lib.Column_t(self.offset.data_ptr(), self.length.data_ptr(),
                             self.value.data_ptr() if self.value is not None else None,
                             self.valid.data_ptr() if self.valid is not None else None)


def alloc_columns(schema: Schema, capacity: int, device="cuda"):
    import torch
    n = max(int(capacity), 1)
    cols = []
    for t in schema.types:
        off = torch.empty(n, dtype=torch.int64, device=device)
        ln = torch.empty(n, dtype=torch.int32, device=device)
        if t == SPAN:
            cols.append(Column(off, ln))
        else:
            val = torch.empty(n, dtype=torch.float64 if t == FLOAT64 else torch.int64, device=device)
            cols.append(Column(off, ln, val, torch.empty(n, dtype=torch.uint8, device=device)))
    return cols


def _col_array(cols):
    arr = (_lib.Column_t * max(len(cols), 1))()
    for i, c in enumerate(cols):
        arr[i] = c.struct()
    return arr


def stats_from_tensor(t):
    """Decode a parpa_stats written on the device into a dict (synchronises)."""
    raw = bytes(t.cpu().numpy().tobytes())
    s = _lib.Stats_t.from_buffer_copy(raw[:_lib.STATS_BYTES])
    return {"records": s.records, "fields": s.fields, "first_invalid": s.first_invalid,
            "missing_records": s.missing_records, "extra_fields": s.extra_fields,
            "deferred_fields": s.deferred_fields, "status": s.status, "final_state": s.final_state,
            "block_fields": s.block_fields, "device_fields": s.device_fields}


def new_stats_tensor(device="cuda"):
    import torch
    return torch.zeros(_lib.STATS_BYTES, dtype=torch.uint8, device=device)


class ParseResult:
    def __init__(self, columns, stats):
        self.columns = columns
        self.stats = stats
        self.records = stats["records"]
        self.status = stats["status"]


def _check_input(data):
    import torch
    if not isinstance(data, torch.Tensor) or data.dtype != torch.uint8 or not data.is_cuda:
        raise TypeError("data must be a torch.uint8 CUDA tensor")
    if not data.is_contiguous():
        raise ValueError("data must be contiguous")


def parse(dfa: Dfa, schema: Schema, data, stream=None) -> ParseResult:
    """Two-phase parse into exactly-sized torch columns (parpa_plan_create + parpa_plan_emit)."""
    L = _lib.load()
    _check_input(data)
    s = _stream_handle(stream)
    plan = ctypes.c_void_p()
    _check(L.parpa_plan_create(dfa.handle, ctypes.c_void_p(data.data_ptr()), data.numel(), s, ctypes.byref(plan)),
           "parpa_plan_create")
    try:
        R = ctypes.c_uint64()
        _check(L.parpa_plan_records(plan, ctypes.byref(R)), "parpa_plan_records")
        cols = alloc_columns(schema, R.value, data.device)
        st = new_stats_tensor(data.device)
        sch = schema.struct()
        arr = _col_array(cols)
        _check(L.parpa_plan_emit(plan, ctypes.byref(sch), arr, ctypes.c_void_p(st.data_ptr()), s), "parpa_plan_emit")
        stats = stats_from_tensor(st)
    finally:
        L.parpa_plan_destroy(plan)
    n = stats["records"]
    for c in cols:
        c.offset, c.length = c.offset[:n], c.length[:n]
        if c.value is not None:
            c.value, c.valid = c.value[:n], c.valid[:n]
    return ParseResult(cols, stats)


class Workspace:
    """A reusable parse workspace (parpa_workspace_create): parse_into(..., workspace=ws) then allocates,
    zeroes and synchronises nothing (one kernel for inputs up to 2 MB; CUDA-graph friendly)."""

    def __init__(self, max_len: int, stream=None):
        L = _lib.load()
        self._ws = ctypes.c_void_p()
        _check(L.parpa_workspace_create(int(max_len), _stream_handle(stream), ctypes.byref(self._ws)),
               "parpa_workspace_create")
        self.max_len = int(max_len)

    def close(self):
        if self._ws:
            _lib.load().parpa_workspace_destroy(self._ws)
            self._ws = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def parse_into(dfa: Dfa, schema: Schema, data, columns, capacity: int, stats_tensor, stream=None,
               skip_records=None, workspace: "Workspace" = None) -> int:
    """Parse into caller columns without a host round trip (parpa_parse_into).  Asynchronous; returns the
    number of kernels launched.  skip_records: a sorted device int64 tensor of record indices not to write
    (parpa_parse_into_skip).  workspace: a Workspace (parpa_parse_into_ws: no allocation or memset)."""
    L = _lib.load()
    _check_input(data)
    sch = schema.struct()
    arr = _col_array(columns)
    n = ctypes.c_uint32(0)
    if workspace is not None:
        assert skip_records is None, "skip_records is not combined with a workspace"
        _check(L.parpa_parse_into_ws(workspace._ws, dfa.handle, ctypes.byref(sch), ctypes.c_void_p(data.data_ptr()),
                                     data.numel(), arr, int(capacity), ctypes.c_void_p(stats_tensor.data_ptr()),
                                     _stream_handle(stream), ctypes.byref(n)), "parpa_parse_into_ws")
        return n.value
    if skip_records is not None and skip_records.numel():
        _check(L.parpa_parse_into_skip(dfa.handle, ctypes.byref(sch), ctypes.c_void_p(data.data_ptr()), data.numel(),
                                       ctypes.c_void_p(skip_records.data_ptr()), skip_records.numel(), arr,
                                       int(capacity), ctypes.c_void_p(stats_tensor.data_ptr()),
                                       _stream_handle(stream), ctypes.byref(n)), "parpa_parse_into_skip")
        return n.value
    _check(L.parpa_parse_into(dfa.handle, ctypes.byref(sch), ctypes.c_void_p(data.data_ptr()), data.numel(), arr,
                              int(capacity), ctypes.c_void_p(stats_tensor.data_ptr()), _stream_handle(stream),
                              ctypes.byref(n)), "parpa_parse_into")
    return n.value


def parse_c_owned(dfa: Dfa, schema: Schema, data, stream=None) -> ParseResult:
    """parpa_parse (library-allocated result), columns copied into torch tensors, result freed."""
    import torch
    L = _lib.load()
    _check_input(data)
    sch = schema.struct()
    s = _stream_handle(stream)
    res = ctypes.c_void_p()
    _check(L.parpa_parse(dfa.handle, ctypes.byref(sch), ctypes.c_void_p(data.data_ptr()), data.numel(), s,
                         ctypes.byref(res)), "parpa_parse")
    try:
        st = _lib.Stats_t()
        _check(L.parpa_result_stats(res, ctypes.byref(st)), "parpa_result_stats")
        stats = {f: getattr(st, f) for f, _ in _lib.Stats_t._fields_}
        R = stats["records"]
        cols = alloc_columns(schema, R, data.device)
        for c in range(schema.C):
            dst = cols[c].struct()
            _check(L.parpa_result_copy_column(res, c, ctypes.byref(dst), s), "parpa_result_copy_column")
        torch.cuda.current_stream().synchronize() if stream is None else stream.synchronize()
    finally:
        L.parpa_result_free(res)
    for c in cols:
        c.offset, c.length = c.offset[:R], c.length[:R]
        if c.value is not None:
            c.value, c.valid = c.value[:R], c.valid[:R]
    return ParseResult(cols, stats)


def parse_host(dfa: Dfa, schema: Schema, host_bytes, capacity: int, stream=None):
    """End to end from host memory (parpa_parse_host): returns (stats, numpy columns)."""
    import numpy as np
    L = _lib.load()
    if isinstance(host_bytes, (bytes, bytearray, memoryview)):
        buf = np.frombuffer(bytes(host_bytes), np.uint8)
    else:
        buf = np.ascontiguousarray(host_bytes, dtype=np.uint8).reshape(-1)
    cap = max(int(capacity), 1)
    cols_np = []
    arr = (_lib.Column_t * max(schema.C, 1))()
    for i, t in enumerate(schema.types):
        off = np.empty(cap, np.uint64)
        ln = np.empty(cap, np.uint32)
        val = np.empty(cap, np.float64 if t == FLOAT64 else np.int64) if t != SPAN else None
        ok = np.empty(cap, np.uint8) if t != SPAN else None
        cols_np.append((off, ln, val, ok))
        arr[i] = _lib.Column_t(off.ctypes.data, ln.ctypes.data, val.ctypes.data if val is not None else None,
                               ok.ctypes.data if ok is not None else None)
    sch = schema.struct()
    st = _lib.Stats_t()
    _check(L.parpa_parse_host(dfa.handle, ctypes.byref(sch), ctypes.c_void_p(buf.ctypes.data), buf.size, arr, cap,
                              ctypes.byref(st), _stream_handle(stream)), "parpa_parse_host")
    stats = {f: getattr(st, f) for f, _ in _lib.Stats_t._fields_}
    R = min(stats["records"], cap)
    return stats, [(o[:R], n[:R], v[:R] if v is not None else None, k[:R] if k is not None else None)
                   for o, n, v, k in cols_np]


def parse_host_into(dfa: Dfa, schema: Schema, host_data, host_columns, capacity: int, stream=None):
    """End to end from host tensors (pinned for full PCIe bandwidth): parpa_parse_host copies the input
    to the device, parses it and copies every column back into ``host_columns``.  Returns stats."""
    L = _lib.load()
    sch = schema.struct()
    arr = _col_array(host_columns)
    st = _lib.Stats_t()
    _check(L.parpa_parse_host(dfa.handle, ctypes.byref(sch), ctypes.c_void_p(host_data.data_ptr()), host_data.numel(),
                              arr, int(capacity), ctypes.byref(st), _stream_handle(stream)), "parpa_parse_host")
    return {f: getattr(st, f) for f, _ in _lib.Stats_t._fields_}


def debug_trace(dfa: Dfa, data, per_byte=True, stream=None):
    """GPU per-chunk entry states (S2-S3 path) and, optionally, per-byte kinds / states."""
    import torch
    L = _lib.load()
    _check_input(data)
    n = data.numel()
    cb = L.parpa_chunk_bytes()
    nch = (n + cb - 1) // cb
    cs = torch.empty(max(nch, 1), dtype=torch.uint8, device=data.device)
    kinds = torch.empty(max(n, 1), dtype=torch.uint8, device=data.device) if per_byte else None
    states = torch.empty(max(n, 1), dtype=torch.uint8, device=data.device) if per_byte else None
    _check(L.parpa_debug_trace(dfa.handle, ctypes.c_void_p(data.data_ptr()), n, ctypes.c_void_p(cs.data_ptr()),
                               ctypes.c_void_p(kinds.data_ptr()) if per_byte else None,
                               ctypes.c_void_p(states.data_ptr()) if per_byte else None, _stream_handle(stream)),
           "parpa_debug_trace")
    return cs[:nch], (kinds[:n] if per_byte else None), (states[:n] if per_byte else None)


# ---- range summaries (windows / multi-GPU) -------------------------------------------------
def compact_rows(data, skip_rows, stream=None):
    """parpa_compact_rows: the input without the raw lines whose indices are in ``skip_rows`` (sorted device
    int64 tensor).  Returns a new device uint8 tensor."""
    import torch
    L = _lib.load()
    _check_input(data)
    out = torch.empty(max(data.numel(), 1) + 16, dtype=torch.uint8, device=data.device)
    n = ctypes.c_uint64(0)
    sk = skip_rows if skip_rows is not None else torch.empty(0, dtype=torch.int64, device=data.device)
    _check(L.parpa_compact_rows(ctypes.c_void_p(data.data_ptr()), data.numel(),
                                ctypes.c_void_p(sk.data_ptr()) if sk.numel() else None, sk.numel(),
                                ctypes.c_void_p(out.data_ptr()), ctypes.byref(n), _stream_handle(stream)),
           "parpa_compact_rows")
    return out[:n.value]


def debug_masks(dfa: Dfa, data, stream=None):
    """The production pass-2 masks (parpa_debug_masks) as a host uint64 array [chunks, 3] (DATA, DELIM,
    RECORD; bit i = byte i of the chunk)."""
    import numpy as np
    import torch
    L = _lib.load()
    _check_input(data)
    n = data.numel()
    tb = L.parpa_tile_bytes()
    nt = (n + tb - 1) // tb
    m = torch.empty(max(nt * 96, 1), dtype=torch.int64, device=data.device)
    _check(L.parpa_debug_masks(dfa.handle, ctypes.c_void_p(data.data_ptr()), n, ctypes.c_void_p(m.data_ptr()),
                               _stream_handle(stream)), "parpa_debug_masks")
    a = m.cpu().numpy().view(np.uint64)[:nt * 96].reshape(nt, 3, 32)
    nch = (n + L.parpa_chunk_bytes() - 1) // L.parpa_chunk_bytes()
    return a.transpose(0, 2, 1).reshape(nt * 32, 3)[:nch]


def summarize(dfa: Dfa, data, stream=None):
    L = _lib.load()
    _check_input(data)
    t = _lib.Tau_t()
    _check(L.parpa_summarize(dfa.handle, ctypes.c_void_p(data.data_ptr()), data.numel(), _stream_handle(stream),
                             ctypes.byref(t)), "parpa_summarize")
    return list(t.tau[:dfa.num_states])


def count(dfa: Dfa, data, base: int, entry_state: int, stream=None):
    L = _lib.load()
    _check_input(data)
    c = _lib.Counts_t()
    t = _lib.Tau_t()
    _check(L.parpa_count(dfa.handle, ctypes.c_void_p(data.data_ptr()), data.numel(), int(base), int(entry_state),
                         _stream_handle(stream), ctypes.byref(c), ctypes.byref(t)), "parpa_count")
    return c, list(t.tau[:dfa.num_states])


def compose_tau(dfa: Dfa, a, b):
    L = _lib.load()
    ta, tb, out = _lib.Tau_t(), _lib.Tau_t(), _lib.Tau_t()
    for i in range(16):
        ta.tau[i] = a[i] if i < len(a) else 0xFF
        tb.tau[i] = b[i] if i < len(b) else 0xFF
    _check(L.parpa_compose_tau(dfa.handle, ctypes.byref(ta), ctypes.byref(tb), ctypes.byref(out)), "compose_tau")
    return list(out.tau[:dfa.num_states])


def compose_counts(a, b):
    L = _lib.load()
    out = _lib.Counts_t()
    _check(L.parpa_compose_counts(ctypes.byref(a), ctypes.byref(b), ctypes.byref(out)), "compose_counts")
    return out


def identity_counts():
    return _lib.Counts_t(0, 0, NONE, NONE, 0, 0, NONE)


def counts_to_bytes(c) -> bytes:
    return bytes(c)


def counts_from_bytes(b: bytes):
    return _lib.Counts_t.from_buffer_copy(b)


def parse_range(dfa: Dfa, schema: Schema, data, entry_state: int, base: int, prefix, columns, capacity: int,
                stats_tensor, left=None, is_last=True, stream=None):
    L = _lib.load()
    _check_input(data)
    ctx = _lib.Context_t(int(entry_state), 0, int(base), prefix)
    sch = schema.struct()
    arr = _col_array(columns)
    lptr = ctypes.c_void_p(left.data_ptr()) if left is not None and left.numel() else None
    llen = left.numel() if left is not None else 0
    _check(L.parpa_parse_range(dfa.handle, ctypes.byref(sch), ctypes.c_void_p(data.data_ptr()), data.numel(),
                               ctypes.byref(ctx), lptr, llen, int(bool(is_last)), arr, int(capacity),
                               ctypes.c_void_p(stats_tensor.data_ptr()), _stream_handle(stream)), "parpa_parse_range")


def infer_columns(dfa: Dfa, data, stream=None):
    """(records, min fields per record, max fields per record) of the device bytes (parpa_infer_columns)."""
    L = _lib.load()
    _check_input(data)
    mn, mx, r = ctypes.c_uint32(0), ctypes.c_uint32(0), ctypes.c_uint64(0)
    _check(L.parpa_infer_columns(dfa.handle, ctypes.c_void_p(data.data_ptr()), data.numel(), _stream_handle(stream),
                                 ctypes.byref(mn), ctypes.byref(mx), ctypes.byref(r)), "parpa_infer_columns")
    return int(r.value), int(mn.value), int(mx.value)


CLASS_NAMES = ("empty", "int8", "int16", "int32", "int64", "float64", "timestamp", "string")


def infer_types(dfa: Dfa, data, num_columns: int, stream=None):
    """Type inference of the first ``num_columns`` columns (parpa_infer_types): returns
    (types, class_masks, records) — types[c] a class name of CLASS_NAMES, class_masks[c] the OR of
    1 << class over the column's fields."""
    import numpy as np
    L = _lib.load()
    _check_input(data)
    n = int(num_columns)
    masks = np.zeros(max(n, 1), np.uint32)
    types = np.zeros(max(n, 1), np.uint8)
    r = ctypes.c_uint64(0)
    _check(L.parpa_infer_types(dfa.handle, ctypes.c_void_p(data.data_ptr()), data.numel(), n, _stream_handle(stream),
                               ctypes.c_void_p(masks.ctypes.data), ctypes.c_void_p(types.ctypes.data), ctypes.byref(r)),
           "parpa_infer_types")
    return [CLASS_NAMES[t] for t in types[:n]], [int(m) for m in masks[:n]], int(r.value)


def strings(dfa: Dfa, data, column, rows: int, stream=None):
    """String materialisation of one parsed column (parpa_strings_size / _copy): returns
    (offsets int64[rows + 1], data uint8[total]) on the GPU — the DATA bytes of every field with
    control bytes dropped, Arrow layout."""
    import torch
    L = _lib.load()
    _check_input(data)
    offs = torch.empty(int(rows) + 1, dtype=torch.int64, device=data.device)
    total = ctypes.c_uint64(0)
    col = column.struct()
    _check(L.parpa_strings_size(dfa.handle, ctypes.c_void_p(data.data_ptr()), data.numel(), ctypes.byref(col),
                                int(rows), ctypes.c_void_p(offs.data_ptr()), ctypes.byref(total),
                                _stream_handle(stream)), "parpa_strings_size")
    buf = torch.empty(max(int(total.value), 1), dtype=torch.uint8, device=data.device)
    _check(L.parpa_strings_copy(dfa.handle, ctypes.c_void_p(data.data_ptr()), data.numel(), ctypes.byref(col),
                                int(rows), ctypes.c_void_p(offs.data_ptr()), ctypes.c_void_p(buf.data_ptr()),
                                _stream_handle(stream)), "parpa_strings_copy")
    return offs, buf[:int(total.value)]


_ALLOC_FN = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p)
_FREE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p)
_ALLOC_KEEP = []


def use_torch_allocator(enable: bool = True):
    """Route result-owned buffers (parpa_parse / parse_c_owned) through torch's caching allocator
    (parpa_set_allocator); enable=False restores the library default (cudaMallocAsync)."""
    import torch
    L = _lib.load()
    if not enable:
        _check(L.parpa_set_allocator(None, None, None), "parpa_set_allocator")
        return

    def _alloc(n, stream, ctx):
        try:
            return torch.cuda.caching_allocator_alloc(int(n), stream=int(stream or 0))
        except Exception:
            return None

    def _free(ptr, stream, ctx):
        torch.cuda.caching_allocator_delete(int(ptr))

    fa, ff = _ALLOC_FN(_alloc), _FREE_FN(_free)
    _ALLOC_KEEP[:] = [fa, ff]                      # the C side keeps raw pointers to these thunks
    _check(L.parpa_set_allocator(ctypes.cast(fa, ctypes.c_void_p), ctypes.cast(ff, ctypes.c_void_p), None),
           "parpa_set_allocator")


CSS_ARROW, CSS_INLINE, CSS_VECTOR = 0, 1, 2     # CSS layouts


class Plan:
    """A two-phase parse kept open (parpa_plan_create ... parpa_plan_destroy): ``emit(schema)`` writes the
    columns; ``strings(column, rows, mode)`` materialises a string column from the plan's chunk masks
    (parpa_plan_strings_size / _copy: no second scan half)."""

    def __init__(self, dfa: Dfa, data, stream=None):
        L = _lib.load()
        _check_input(data)
        self._data, self._stream = data, stream
        self._dfa = dfa                                  # the plan's kernels read the DFA: keep it alive
        self._plan = ctypes.c_void_p()
        _check(L.parpa_plan_create(dfa.handle, ctypes.c_void_p(data.data_ptr()), data.numel(), _stream_handle(stream),
                                   ctypes.byref(self._plan)), "parpa_plan_create")
        R = ctypes.c_uint64()
        _check(L.parpa_plan_records(self._plan, ctypes.byref(R)), "parpa_plan_records")
        self.records = R.value

    def emit(self, schema: Schema):
        cols = alloc_columns(schema, self.records, self._data.device)
        st = new_stats_tensor(self._data.device)
        _check(_lib.load().parpa_plan_emit(self._plan, ctypes.byref(schema.struct()), _col_array(cols),
                                           ctypes.c_void_p(st.data_ptr()), _stream_handle(self._stream)),
               "parpa_plan_emit")
        stats = stats_from_tensor(st)
        n = stats["records"]
        for c in cols:
            c.offset, c.length = c.offset[:n], c.length[:n]
            if c.value is not None:
                c.value, c.valid = c.value[:n], c.valid[:n]
        return ParseResult(cols, stats)

    def strings(self, column, rows: int, mode: int = CSS_ARROW, terminator: int = 0x1F):
        """(offsets int64[rows + 1], data uint8[total]) — plus aux uint8[total] for CSS_VECTOR."""
        import torch
        L = _lib.load()
        dev = self._data.device
        offs = torch.empty(int(rows) + 1, dtype=torch.int64, device=dev)
        total = ctypes.c_uint64(0)
        col = column.struct()
        s = _stream_handle(self._stream)
        _check(L.parpa_plan_strings_size(self._plan, ctypes.byref(col), int(rows), int(mode),
                                         ctypes.c_void_p(offs.data_ptr()), ctypes.byref(total), s),
               "parpa_plan_strings_size")
        n = int(total.value)
        buf = torch.empty(max(n, 1), dtype=torch.uint8, device=dev)
        aux = torch.empty(max(n, 1), dtype=torch.uint8, device=dev) if mode == CSS_VECTOR else None
        _check(L.parpa_plan_strings_copy(self._plan, ctypes.byref(col), int(rows), int(mode), int(terminator),
                                         ctypes.c_void_p(offs.data_ptr()), ctypes.c_void_p(buf.data_ptr()),
                                         ctypes.c_void_p(aux.data_ptr() if aux is not None else 0), s),
               "parpa_plan_strings_copy")
        return (offs, buf[:n]) if aux is None else (offs, buf[:n], aux[:n])

    def close(self):
        if self._plan:
            _lib.load().parpa_plan_destroy(self._plan)
            self._plan = ctypes.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def css_index(mode: int, buf, terminator: int = 0x1F, stream=None):
    """The CSS index as the paper generates it (parpa_css_index): positions of the terminators in an
    inline-terminated CSS (mode CSS_INLINE, buf = data) or of the nonzero entries of the auxiliary vector
    (CSS_VECTOR, buf = aux).  Returns an int64 tensor on buf's device."""
    import torch
    L = _lib.load()
    n = buf.numel()
    idx = torch.empty(max(n, 1), dtype=torch.int64, device=buf.device)
    cnt = ctypes.c_uint64(0)
    p = ctypes.c_void_p(buf.data_ptr() if n else 0)
    _check(L.parpa_css_index(int(mode), int(terminator), p if mode == CSS_INLINE else None,
                             p if mode == CSS_VECTOR else None, n, ctypes.c_void_p(idx.data_ptr()), ctypes.byref(cnt),
                             _stream_handle(stream)), "parpa_css_index")
    return idx[:int(cnt.value)]


STATE_UNKNOWN = 0xFFFFFFFF


class RangePlan:
    """Staged parse of one byte range (the multi-GPU exchange with every pass run once):
    ``begin`` -> the range's transition vector, ``count(entry_state)`` -> its counts,
    ``emit(...)`` -> its columns (parpa_range_begin / _count / _emit)."""

    def __init__(self, dfa: Dfa, data, base: int, stream=None):
        L = _lib.load()
        _check_input(data)
        self._dfa, self._data, self._stream = dfa, data, stream
        self.handle = ctypes.c_void_p()
        t = _lib.Tau_t()
        _check(L.parpa_range_begin(dfa.handle, ctypes.c_void_p(data.data_ptr()), data.numel(), int(base),
                                   _stream_handle(stream), ctypes.byref(self.handle), ctypes.byref(t)),
               "parpa_range_begin")
        self.tau = list(t.tau[:dfa.num_states])
        self.base = int(base)

    def count(self, entry_state: int):
        c = _lib.Counts_t()
        _check(_lib.load().parpa_range_count(self.handle, int(entry_state), ctypes.byref(c)), "parpa_range_count")
        self.entry_state = int(entry_state)
        return c

    def state_at(self, pos: int) -> int:
        """DFA state before the byte at global offset ``pos`` (chunk-aligned, within the range; after
        ``count``) — the state a halo sender attaches to bytes sent from ``pos`` on."""
        st = ctypes.c_uint32(0)
        _check(_lib.load().parpa_range_state_at(self.handle, int(pos), ctypes.byref(st)), "parpa_range_state_at")
        return st.value

    def emit(self, schema: Schema, prefix, columns, capacity: int, stats_tensor, left=None, is_last=True,
             left_state=None):
        """left: device bytes just before the range (the halo); left_state: the DFA state before left[0]
        (None: unknown — straddling typed fields with inner control bytes are then unsupported)."""
        L = _lib.load()
        ctx = _lib.Context_t(self.entry_state, 0, self.base, prefix)
        sch = schema.struct()
        arr = _col_array(columns)
        lptr = ctypes.c_void_p(left.data_ptr()) if left is not None and left.numel() else None
        llen = left.numel() if left is not None else 0
        ls = STATE_UNKNOWN if left_state is None or not llen else int(left_state)
        _check(L.parpa_range_emit_halo(self.handle, ctypes.byref(sch), ctypes.byref(ctx), lptr, llen, ls,
                                       int(bool(is_last)), arr, int(capacity),
                                       ctypes.c_void_p(stats_tensor.data_ptr()), _stream_handle(self._stream)),
               "parpa_range_emit_halo")

    def close(self):
        if getattr(self, "handle", None) and self.handle.value:
            try:
                _lib.load().parpa_plan_destroy(self.handle)
            except Exception:
                pass
            self.handle = ctypes.c_void_p()

    def __del__(self):
        self.close()


def set_profiling(enable: bool):
    _lib.load().parpa_set_profiling(int(enable))


def last_kernel_times():
    L = _lib.load()
    names = (ctypes.c_char_p * 4096)()
    ms = (ctypes.c_float * 4096)()
    n = L.parpa_last_kernel_times(names, ms, 4096)
    return [(names[i].decode(), ms[i]) for i in range(n)]


def chunk_bytes() -> int:
    return _lib.load().parpa_chunk_bytes()


def tile_bytes() -> int:
    return _lib.load().parpa_tile_bytes()


def version() -> str:
    return _lib.load().parpa_version().decode()
