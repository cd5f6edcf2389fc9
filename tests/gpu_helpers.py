"""Shared helpers for the GPU parity tests (compare the CUDA path with the oracle element by element)."""
import numpy as np

import oracle


def to_np(t):
    return t.detach().cpu().numpy()


def compare(res, ora, types, label=""):
    """res: paper_1905_13415_b200.ParseResult; ora: oracle.OracleResult.  Bit-exact on every array."""
    st = res.stats
    assert st["status"] == ora.status, (label, st, ora.status)
    if ora.status == oracle.EFORMAT:
        assert st["first_invalid"] == ora.first_invalid, (label, st["first_invalid"], ora.first_invalid)
        return
    assert st["records"] == ora.R, (label, st["records"], ora.R)
    assert st["missing_records"] == ora.n_missing, label
    assert st["extra_fields"] == ora.n_extra, label
    assert st["fields"] == ora.nfields, (label, st["fields"], ora.nfields)
    for c, t in enumerate(types):
        col = res.columns[c]
        off = to_np(col.offset).view(np.uint64)[:ora.R]
        ln = to_np(col.length).view(np.uint32)[:ora.R]
        bad = np.flatnonzero(off != ora.offset[c])
        assert bad.size == 0, (label, "offset", c, bad[:5], off[bad[:5]], ora.offset[c][bad[:5]])
        bad = np.flatnonzero(ln != ora.length[c])
        assert bad.size == 0, (label, "length", c, bad[:5], ln[bad[:5]], ora.length[c][bad[:5]])
        if t != oracle.SPAN:
            ok = to_np(col.valid)[:ora.R]
            bad = np.flatnonzero(ok != ora.valid[c])
            assert bad.size == 0, (label, "valid", c, bad[:5])
            v = to_np(col.value).view(np.int64)[:ora.R]
            bad = np.flatnonzero(v != ora.value[c])
            assert bad.size == 0, (label, "value", c, bad[:5], v[bad[:5]], ora.value[c][bad[:5]])
