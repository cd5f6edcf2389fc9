"""Pins for the oracle's type conversion (readings R14/R15) against Python's int()/float()."""
import random
import re
import struct

import pytest

import oracle

FLOAT_RE = re.compile(rb"^[+-]?([0-9]+(\.[0-9]*)?|\.[0-9]+)([eE][+-]?[0-9]+)?$")
INT_RE = re.compile(rb"^[+-]?[0-9]+$")


def bits(x: float) -> int:
    return struct.unpack("<q", struct.pack("<d", x))[0]


@pytest.mark.parametrize("s,ok,val", [
    (b"0", True, 0), (b"-0", True, 0), (b"+17", True, 17), (b"007", True, 7),
    (b"9223372036854775807", True, 2**63 - 1), (b"-9223372036854775808", True, -2**63),
    (b"9223372036854775808", False, 0), (b"-9223372036854775809", False, 0),
    (b"", False, 0), (b"+", False, 0), (b"-", False, 0), (b"1 ", False, 0), (b" 1", False, 0),
    (b"1.0", False, 0), (b"1e3", False, 0), (b"0x10", False, 0), (b"00000000000000000000000001", True, 1),
])
def test_int64_cases(s, ok, val):
    assert oracle.conv_int64(s) == (ok, val)


def test_int64_random_vs_python():
    rng = random.Random(5)
    for _ in range(20000):
        n = rng.randint(1, 21)
        s = (rng.choice([b"", b"+", b"-"]) + bytes(rng.choice(b"0123456789") for _ in range(n)))
        v = int(s)
        ok = -2**63 <= v < 2**63
        assert oracle.conv_int64(s) == (ok, v if ok else 0), s


@pytest.mark.parametrize("s,expect", [
    (b"0.3", 0.3), (b"-0.00", -0.0), (b"9007199254740993", 9007199254740992.0),
    (b"2.2250738585072011e-308", 2.2250738585072011e-308), (b"1e23", 1e23),
    (b"4.9406564584124654e-324", 5e-324), (b"1e400", float("inf")), (b"-1e400", float("-inf")),
    (b"1e-400", 0.0), (b".5", 0.5), (b"5.", 5.0), (b"12.5", 12.5), (b"4.217e-01", 0.4217),
    (b"0.1e0000000000000000000000000001", 1.0),
])
def test_float64_hard_cases(s, expect):
    ok, b = oracle.conv_float64(s)
    assert ok and b == bits(expect)


@pytest.mark.parametrize("s", [b"", b"1e", b"e5", b".", b"-", b"+.", b"inf", b"nan", b"0x1p3", b" 1", b"1 ",
                               b"1_0", b"1e+", b"--1", b"1.2.3"])
def test_float64_grammar_rejects(s):
    assert oracle.conv_float64(s) == (False, 0)


def test_float64_random_vs_python():
    # Python float() is correctly rounded (round-half-even), the reading R15 requires the same.
    rng = random.Random(9)
    for _ in range(30000):
        ip = bytes(rng.choice(b"0123456789") for _ in range(rng.randint(0, 20)))
        fp = bytes(rng.choice(b"0123456789") for _ in range(rng.randint(0, 20)))
        s = rng.choice([b"", b"-", b"+"]) + ip + (b"." + fp if rng.random() < 0.7 else b"")
        if rng.random() < 0.4:
            s += rng.choice([b"e", b"E"]) + rng.choice([b"", b"+", b"-"]) + str(rng.randint(0, 340)).encode()
        ok, b = oracle.conv_float64(s)
        if FLOAT_RE.match(s):
            assert ok and b == bits(float(s)), s
        else:
            assert not ok, s


def test_float64_taxi_like_decimals():
    rng = random.Random(1)
    for _ in range(20000):
        cents = rng.randint(0, 10**7)
        s = f"{cents // 100}.{cents % 100:02d}".encode()
        assert oracle.conv_float64(s)[1] == bits(float(s))
