"""Pins for the oracle's timestamp conversion (reading R29) against Python's own
calendar arithmetic (calendar.timegm / datetime with a fixed UTC offset), which shares nothing with
the oracle's era/day-of-year formula: random dates over four centuries, every day boundary of
leap-year Februaries, invalid calendar dates and malformed shapes."""
import calendar
import datetime as dt
import random

import pytest

import oracle

MON = ["Jan", "Feb", "Mar", "Apr", "May", "Jun", "Jul", "Aug", "Sep", "Oct", "Nov", "Dec"]


def iso(Y, M, D, h, m, s, sep=" "):
    return f"{Y:04d}-{M:02d}-{D:02d}{sep}{h:02d}:{m:02d}:{s:02d}".encode()


def test_iso_random_against_timegm():
    rng = random.Random(1)
    for _ in range(20000):
        Y = rng.randint(1, 9999)
        M = rng.randint(1, 12)
        D = rng.randint(1, calendar.monthrange(Y, M)[1])
        h, m, s = rng.randint(0, 23), rng.randint(0, 59), rng.randint(0, 59)
        ok, v = oracle.conv_timestamp(iso(Y, M, D, h, m, s, rng.choice(" T")))
        assert ok and v == calendar.timegm((Y, M, D, h, m, s)), (Y, M, D, h, m, s)


def test_epoch_and_leap_days():
    assert oracle.conv_timestamp(b"1970-01-01 00:00:00") == (True, 0)
    assert oracle.conv_timestamp(b"1969-12-31 23:59:59") == (True, -1)
    assert oracle.conv_timestamp(b"2038-01-19 03:14:08") == (True, 2 ** 31)
    for Y in (1600, 1900, 2000, 2019, 2020, 2100, 2400):
        leap = calendar.isleap(Y)
        assert oracle.conv_timestamp(iso(Y, 2, 29, 0, 0, 0))[0] == leap, Y
        ok, v = oracle.conv_timestamp(iso(Y, 3, 1, 0, 0, 0))
        assert ok and v == calendar.timegm((Y, 3, 1, 0, 0, 0))


@pytest.mark.parametrize("bad", [b"2019-13-01 00:00:00", b"2019-00-10 00:00:00", b"2019-04-31 00:00:00",
                                 b"2019-01-01 24:00:00", b"2019-01-01 00:60:00", b"2019-01-01 00:00:60",
                                 b"2019-01-01 00:00", b"2019/01/01 00:00:00", b"2019-01-01x00:00:00",
                                 b"201a-01-01 00:00:00", b"", b"2019-01-01 00:00:00 ", b"+019-01-01 00:00:00"])
def test_iso_invalid(bad):
    assert oracle.conv_timestamp(bad) == (False, 0)


def test_clf_random_against_datetime():
    rng = random.Random(2)
    for _ in range(5000):
        Y = rng.randint(1970, 2100)
        M = rng.randint(1, 12)
        D = rng.randint(1, calendar.monthrange(Y, M)[1])
        h, m, s = rng.randint(0, 23), rng.randint(0, 59), rng.randint(0, 59)
        zh, zm, sign = rng.randint(0, 14), rng.choice([0, 30, 45]), rng.choice("+-")
        txt = f"{D:02d}/{MON[M - 1]}/{Y:04d}:{h:02d}:{m:02d}:{s:02d} {sign}{zh:02d}{zm:02d}".encode()
        off = dt.timedelta(hours=zh, minutes=zm) * (1 if sign == "+" else -1)
        ref = int(dt.datetime(Y, M, D, h, m, s, tzinfo=dt.timezone(off)).timestamp())
        ok, v = oracle.conv_timestamp(txt)
        assert ok and v == ref, txt


@pytest.mark.parametrize("bad", [b"10/Oct/2000:13:55:36 0700", b"10/Okt/2000:13:55:36 -0700",
                                 b"31/Apr/2000:13:55:36 -0700", b"10/Oct/2000:13:55:36 -0760",
                                 b"10-Oct-2000:13:55:36 -0700", b"10/Oct/2000 13:55:36 -0700"])
def test_clf_invalid(bad):
    assert oracle.conv_timestamp(bad) == (False, 0)


def test_paper_clf_fixture_timestamp_column():
    # SURVEY Appendix A.3 fixture: the %t field of the first record, as a typed column
    data = (b'10.0.0.1 - frank [10/Oct/2000:13:55:36 -0700] "GET / HTTP/1.0" 200 2326\n')
    r = oracle.parse("clf", data, 7, [0, 0, 0, oracle.TIMESTAMP, 0, 1, 1])
    assert r.status == 0 and r.R == 1
    assert int(r.valid[3][0]) == 1 and int(r.value[3][0]) == 971211336     # 2000-10-10T20:55:36Z
