"""Pins for the oracle's string materialisation (the paper's CSS P:439-457): the DATA
bytes of every field of a column, control bytes dropped.  For RFC-4180 CSV this is exactly what
Python's csv module returns (an independent implementation); for the Common Log Format the SURVEY
Appendix A.3 fixture fixes the request string."""
import csv
import io

import pytest

import datagen
import oracle


def split(offs, data):
    return [data[offs[i]:offs[i + 1]] for i in range(len(offs) - 1)]


@pytest.mark.parametrize("col", range(8))
def test_cfg1_strings_equal_python_csv(col):
    data, g = datagen.generate("cfg1", 300_000)
    raw = bytes(data)
    ref = [row for row in csv.reader(io.StringIO(raw.decode("latin-1"), newline=""), strict=True)]
    offs, s = oracle.strings("csv", raw, 8, col)
    got = split(offs, s)
    assert len(got) == len(ref) == g.records
    for r, row in enumerate(ref):
        want = row[col].encode("latin-1") if col < len(row) else b""
        assert got[r] == want, (r, col)


def test_escapes_and_missing():
    data = b'a,"x""y",z\n"p,q"\n,,\n"multi\nline",""\n'
    offs, s = oracle.strings("csv", data, 3, 1)
    assert split(offs, s) == [b'x"y', b"", b"", b""]
    offs, s = oracle.strings("csv", data, 3, 0)
    assert split(offs, s) == [b"a", b"p,q", b"", b"multi\nline"]


def test_clf_fixture_request_string():
    data = (b'#Version: 1.0\n#Fields: host ident "req" [t]\n'
            b'10.0.0.1 - frank [10/Oct/2000:13:55:36 -0700] "GET /a#b?q=\\"x\\" HTTP/1.0" 200 2326\n'
            b'1.2.3.4 - - [11/Oct/2000:00:00:01 +0000] "HEAD / HTTP/1.1" 304 -')
    offs, s = oracle.strings("clf", data, 7, 4)
    assert split(offs, s) == [b'GET /a#b?q=\\"x\\" HTTP/1.0', b"HEAD / HTTP/1.1"]
    offs, s = oracle.strings("clf", data, 7, 3)
    assert split(offs, s) == [b"10/Oct/2000:13:55:36 -0700", b"11/Oct/2000:00:00:01 +0000"]


def test_css_layouts_hand_derived():
    """P:494-502 on the fixture above, column 1 (fields x"y, "", "", ""), written out by hand: the
    inline-terminated CSS puts the terminator after every field (empty ones too); the vector-delimited CSS
    keeps the Arrow bytes and marks the last symbol of each non-empty field."""
    data = b'a,"x""y",z\n"p,q"\n,,\n"multi\nline",""\n'
    offs, s = oracle.css("csv", data, 3, 1, mode=oracle.CSS_INLINE, terminator=0x1F)
    assert s == b'x"y\x1f\x1f\x1f\x1f' and list(offs) == [0, 4, 5, 6, 7]
    offs, s, aux = oracle.css("csv", data, 3, 0, mode=oracle.CSS_VECTOR)
    assert s == b"ap,qmulti\nline" and list(offs) == [0, 1, 4, 4, 14]
    assert aux == bytes([1, 0, 0, 1] + [0] * 9 + [1])
    # the index: terminator / flag positions = one past each field's last byte - 1
    assert list(oracle.css_index(oracle.CSS_INLINE, b'x"y\x1f\x1f\x1f\x1f')) == [3, 4, 5, 6]
    assert list(oracle.css_index(oracle.CSS_VECTOR, aux)) == [0, 3, 13]


@pytest.mark.parametrize("col", [0, 3, 5])
def test_css_inline_splits_back_to_python_csv(col):
    """Splitting the inline-terminated CSS at its terminators gives Python csv's fields (cfg1 text has no
    0x1F byte, so the terminator is unambiguous)."""
    data, g = datagen.generate("cfg1", 100_000)
    raw = bytes(data)
    ref = [row for row in csv.reader(io.StringIO(raw.decode("latin-1"), newline=""), strict=True)]
    offs, s = oracle.css("csv", raw, 8, col, mode=oracle.CSS_INLINE)
    parts = s.split(b"\x1f")
    assert parts[-1] == b"" and len(parts) - 1 == len(ref)
    for r, row in enumerate(ref):
        assert parts[r] == (row[col].encode("latin-1") if col < len(row) else b""), r
    idx = oracle.css_index(oracle.CSS_INLINE, s)
    assert list(idx) == [int(o) - 1 for o in offs[1:]]
