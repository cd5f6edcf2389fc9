"""Pins of the oracle's type inference ("Type inference", reading R31).

Every field class is checked against an independent classification written here with Python's own
int() / float() / datetime and regular expressions for the R14 / R15 / R29 grammars, and columns built
with a known type (by construction: values drawn from one width's range, including its endpoints) must
resolve to that type.  CPU only."""
import calendar
import datetime
import random
import re

import oracle

INT_RE = re.compile(rb"[+-]?[0-9]+\Z")
FLOAT_RE = re.compile(rb"[+-]?([0-9]+(\.[0-9]*)?|\.[0-9]+)([eE][+-]?[0-9]+)?\Z")
ISO_RE = re.compile(rb"(\d{4})-(\d{2})-(\d{2})[ T](\d{2}):(\d{2}):(\d{2})\Z")
CLF_RE = re.compile(rb"(\d{2})/([A-Z][a-z]{2})/(\d{4}):(\d{2}):(\d{2}):(\d{2}) ([+-])(\d{2})(\d{2})\Z")
MONTHS = [calendar.month_abbr[i].encode() for i in range(1, 13)]


def valid_datetime(s: bytes) -> bool:
    m = ISO_RE.match(s)
    if m:
        Y, M, D, h, mi, sec = (int(x) for x in m.groups())
    else:
        m = CLF_RE.match(s)
        if not m or m.group(2) not in MONTHS or int(m.group(8)) > 23 or int(m.group(9)) > 59:
            return False
        D, Y, h, mi, sec = int(m.group(1)), int(m.group(3)), int(m.group(4)), int(m.group(5)), int(m.group(6))
        M = MONTHS.index(m.group(2)) + 1
    if Y < 1:
        return False
    try:
        datetime.datetime(Y, M, D, h, mi, sec)
    except ValueError:
        return False
    return True


def reference_class(s: bytes) -> str:
    if not s:
        return "empty"
    if INT_RE.match(s):
        v = int(s)
        for name, bits in (("int8", 8), ("int16", 16), ("int32", 32), ("int64", 64)):
            if -(1 << (bits - 1)) <= v < (1 << (bits - 1)):
                return name
        return "float64"                     # digits beyond int64 are still the float grammar
    if FLOAT_RE.match(s):
        float(s)                             # Python accepts every R15 string
        return "float64"
    if valid_datetime(s):
        return "timestamp"
    return "string"


def sample_fields(rng, n):
    out = []
    for _ in range(n):
        k = rng.randrange(9)
        if k == 0:
            bits = rng.choice([8, 16, 32, 64])
            lo, hi = -(1 << (bits - 1)), (1 << (bits - 1)) - 1
            v = rng.choice([lo, hi, lo - 1, hi + 1, rng.randint(lo, hi)])
            out.append(str(v).encode())
        elif k == 1:
            out.append(rng.choice([b"+", b"-", b""]) + b"0" * rng.randint(0, 3) + str(rng.randint(0, 10**rng.randint(1, 25))).encode())
        elif k == 2:
            out.append(f"{rng.uniform(-1e6, 1e6):.{rng.randint(0, 6)}f}".encode())
        elif k == 3:
            out.append(f"{rng.uniform(-1, 1):.3e}".encode().replace(b"e", rng.choice([b"e", b"E"])))
        elif k == 4:
            out.append(rng.choice([b".5", b"5.", b".", b"-.", b"1e", b"1e+", b"+.e1", b"1.2.3", b"--1", b"0x10", b"inf", b"1_0"]))
        elif k == 5:
            y, mo, d = rng.randint(1, 9999), rng.randint(1, 12), rng.randint(1, 31)
            out.append(f"{y:04d}-{mo:02d}-{d:02d}{rng.choice(' T')}{rng.randint(0, 24):02d}:{rng.randint(0, 59):02d}:{rng.randint(0, 60):02d}".encode())
        elif k == 6:
            mon = rng.choice(MONTHS + [b"Foo"])
            out.append(b"%02d/%s/%04d:%02d:%02d:%02d %s%02d%02d" % (rng.randint(1, 31), mon, rng.randint(1, 9999), rng.randint(0, 23),
                                                                    rng.randint(0, 59), rng.randint(0, 59), rng.choice([b"+", b"-"]),
                                                                    rng.randint(0, 24), rng.randint(0, 60)))
        elif k == 7:
            out.append(bytes(rng.choice(b"abcXYZ 12-:.") for _ in range(rng.randint(1, 12))))
        else:
            out.append(b"")
    return out


def test_field_class_matches_python_reference():
    rng = random.Random(31)
    for s in sample_fields(rng, 20000):
        assert oracle.field_class(s) == reference_class(s), s


def test_columns_of_known_type_resolve_to_it():
    """Columns generated from one type's range (endpoints included) infer exactly that type."""
    rng = random.Random(7)
    R = 300
    cols = {
        "int8": [str(v).encode() for v in [-128, 127] + [rng.randint(-128, 127) for _ in range(R - 2)]],
        "int16": [str(v).encode() for v in [-129, 32767] + [rng.randint(-128, 127) for _ in range(R - 2)]],
        "int32": [str(v).encode() for v in [40000, -2**31] + [rng.randint(0, 9) for _ in range(R - 2)]],
        "int64": [str(v).encode() for v in [2**63 - 1, -2**31 - 1] + [rng.randint(-5, 5) for _ in range(R - 2)]],
        "float64": [b"%.2f" % rng.uniform(0, 99) for _ in range(R - 1)] + [b"7"],
        "timestamp": [b"2019-%02d-%02d 12:00:00" % (rng.randint(1, 12), rng.randint(1, 28)) for _ in range(R)],
        "string": [b"x%d" % i for i in range(R - 1)] + [b"12"],
        "empty": [b""] * R,
    }
    for i in range(0, R, 7):                                  # empty fields never change a type
        for k in cols:
            cols[k][i] = b""
    names = list(cols)
    data = b"".join(b",".join(cols[k][r] for k in names) + b"\n" for r in range(R))
    got = oracle.infer_types("csv", data, len(names))
    assert [t for t, _ in got] == names
    # mixing timestamps with numbers gives a string column; quoted numbers are numbers (DATA bytes)
    got = oracle.infer_types("csv", b'1,"12"\n2019-01-01 00:00:00,"3.5"\n', 2)
    assert [t for t, _ in got] == ["string", "float64"]


def test_resolve_types_lattice():
    r = oracle.resolve_types
    assert r(set()) == "empty" and r({"empty"}) == "empty"
    assert r({"int8", "int32"}) == "int32" and r({"int64", "float64"}) == "float64"
    assert r({"timestamp"}) == "timestamp" and r({"timestamp", "int8"}) == "string"
    assert r({"string", "int8"}) == "string"
