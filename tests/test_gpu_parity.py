"""GPU parity: the CUDA path (through the C ABI) against the sequential oracle, element by element.

Bar: bit-exact for states, emission kinds, offsets, lengths, counts and int64 values; 0 ulp
(bitwise) for float64 values (BASELINE north_star).
"""
import itertools
import json
import os
import random

import numpy as np
import pytest

import datagen
import oracle
from tests.gpu_helpers import compare, to_np

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
import paper_1905_13415_b200 as parpa  # noqa: E402

GOLD = os.path.join(os.path.dirname(__file__), "golden")
DIALECT_OF = {"cfg1": "csv", "taxi": "csv", "yelp": "csv", "clf": "clf"}
_DFA = {}


def dfa(name):
    if name not in _DFA:
        _DFA[name] = parpa.Dfa.dialect(name)
    return _DFA[name]


def dev(data):
    a = np.frombuffer(bytes(data), np.uint8) if isinstance(data, (bytes, bytearray)) else np.asarray(data, np.uint8)
    t = torch.empty(max(a.size, 1), dtype=torch.uint8, device="cuda")
    if a.size:
        t[:a.size].copy_(torch.from_numpy(a.copy()))
    return t[:a.size]


def run_all_paths(dialect, data, types, defaults=None, strict=False, label=""):
    schema = parpa.Schema(list(types), defaults, strict)
    ora = oracle.parse(dialect, data, len(types), list(types), defaults, strict)
    d = dev(data)
    res = parpa.parse(dfa(dialect), schema, d)                 # two-phase (scan + emit)
    compare(res, ora, types, label + "/plan")
    cap = max(ora.R, 1) + 3
    cols = parpa.alloc_columns(schema, cap)
    st = parpa.new_stats_tensor()
    parpa.parse_into(dfa(dialect), schema, d, cols, cap, st)   # parse_into: no host round trip
    compare(parpa.ParseResult(cols, parpa.stats_from_tensor(st)), ora, types, label + "/into")
    res3 = parpa.parse_c_owned(dfa(dialect), schema, d)        # library-owned result
    compare(res3, ora, types, label + "/owned")
    return ora


def test_smoke_cfg1_small():
    data, g = datagen.generate("cfg1", 50_000)
    w = datagen.WORKLOADS["cfg1"]
    ora = run_all_paths("csv", data, w.types, label="cfg1-50k")
    assert ora.R == g.records


@pytest.mark.parametrize("name", ["cfg1", "taxi", "yelp", "clf"])
def test_workload_slices_full_compare(name):
    w = datagen.WORKLOADS[name]
    data, g = datagen.generate(name, 3_000_000 if name != "cfg1" else 1_000_000)
    ora = run_all_paths(w.dialect, data, w.types, label=name)
    assert ora.R == g.records


@pytest.mark.parametrize("unit", ["1", "4"])
@pytest.mark.parametrize("name", ["cfg1", "taxi", "yelp", "clf"])
def test_emission_units_forced(name, unit, monkeypatch):
    """Both emission kernels on every workload, whatever its field density: k_emit's 2 KB warp tiles
    (PARPA_EMIT_K=1) and k_emit_sparse's 8 KB super tiles (PARPA_EMIT_K=4), staged path (> 2 MB), plus ragged
    tails of the last super tile."""
    monkeypatch.setenv("PARPA_EMIT_K", unit)
    w = datagen.WORKLOADS[name]
    data, g = datagen.generate(name, 2_600_000)
    for n in (len(data), len(data) - 2047, len(data) - 6000):
        d = data[:n]
        ora = oracle.parse(w.dialect, d, w.C, list(w.types))
        res = parpa.parse(dfa(w.dialect), parpa.Schema(list(w.types)), dev(d))
        compare(res, ora, w.types, f"{name}-K{unit}-{n}")


@pytest.mark.parametrize("n", [0, 1, 2, 63, 64, 65, 127, 4095, 16383, 16384, 16385, 16384 * 3 + 17, 200_003])
def test_ragged_sizes(n):
    data, _ = datagen.generate("cfg1", 400_000)
    run_all_paths("csv", data[:n], datagen.WORKLOADS["cfg1"].types, label=f"n={n}")


def test_golden_fixtures_on_gpu():
    fx = json.load(open(os.path.join(GOLD, "fixtures.json")))
    for key, cases in fx.items():
        if key == "source":
            continue
        dialect = key.replace("_extra", "")              # the hand-derived extra fixtures of a dialect
        for case in cases:
            C = case["C"]
            types = [oracle.SPAN] * C
            if dialect == "clf" and C == 7:
                types[5] = types[6] = oracle.INT64
            run_all_paths(dialect, case["input"].encode(), types, label=case["cite"][:30])


ALPH = [b"\n", b'"', b",", b"a"]


def test_bruteforce_corpus_trace_and_outputs():
    # every string of length <= 6 over {\n, ", ",", a}, each closed with '\n' and concatenated into one
    # corpus (so chunk and tile boundaries fall everywhere); per-chunk entry states and per-byte kinds
    # and states must equal the oracle's sequential trace.
    parts = []
    for n in range(7):
        for t in itertools.product(ALPH, repeat=n):
            parts.append(b"".join(t) + b"\n")
    data = b"".join(parts)
    ora = oracle.parse("csv", data, 4, trace=True)
    cs, kinds, states = parpa.debug_trace(dfa("csv"), dev(data))
    cb = parpa.chunk_bytes()
    starts = np.arange(0, len(data), cb)
    assert np.array_equal(to_np(cs), ora.trace_state[starts])
    assert np.array_equal(to_np(kinds), ora.trace_kind)
    assert np.array_equal(to_np(states), ora.trace_state)


@pytest.mark.parametrize("name", ["cfg1", "yelp", "clf"])
def test_trace_on_workloads(name):
    w = datagen.WORKLOADS[name]
    data, _ = datagen.generate(name, 2_000_000)
    ora = oracle.parse(w.dialect, data, w.C, trace=True)
    cs, kinds, states = parpa.debug_trace(dfa(w.dialect), dev(data))
    cb = parpa.chunk_bytes()
    assert np.array_equal(to_np(cs), ora.trace_state[np.arange(0, len(data), cb)])
    assert np.array_equal(to_np(kinds), ora.trace_kind)
    assert np.array_equal(to_np(states), ora.trace_state)


def random_dfa(rng, S):
    inv = S - 1
    G = rng.randint(2, 8)
    trans = [[rng.randrange(S) for _ in range(S - 1)] + [inv] for _ in range(G)]
    emit = [[rng.randrange(4) for _ in range(S - 1)] + [1] for _ in range(G)]
    eoi = [rng.randrange(3) for _ in range(S)]
    gob = [rng.randrange(G) for _ in range(256)]
    return {"group_of_byte": gob, "transition": trans, "emit": emit, "eoi": eoi,
            "start": rng.randrange(S - 1), "invalid": inv}


@pytest.mark.parametrize("seed", range(40))
def test_random_dfas(seed):
    # random DFAs (|S| <= 9 with an absorbing invalid state), random start state.
    rng = random.Random(seed)
    S = rng.randint(2, 9)
    t = random_dfa(rng, S)
    d = parpa.Dfa(S, t["start"], t["invalid"], t["group_of_byte"], t["transition"], t["emit"], t["eoi"])
    n = rng.choice([100, 5000, 70_000])
    # bias bytes towards a few values so that every group occurs
    vals = [rng.randrange(256) for _ in range(6)]
    data = bytes(rng.choice(vals) if rng.random() < 0.7 else rng.randrange(256) for _ in range(n))
    ora = oracle.parse_tables(t, data, 3, trace=True)
    cs, kinds, states = parpa.debug_trace(d, dev(data))
    cb = parpa.chunk_bytes()
    assert np.array_equal(to_np(cs), ora.trace_state[np.arange(0, len(data), cb)])
    assert np.array_equal(to_np(kinds), ora.trace_kind)
    assert np.array_equal(to_np(states), ora.trace_state)
    schema = parpa.Schema([parpa.SPAN] * 3)
    res = parpa.parse(d, schema, dev(data))
    compare(res, ora, [0, 0, 0], f"rand{seed}")


def test_float_and_int_hard_cases_device_tier():
    # the fast path defers these to the exact decimal algorithm (k_deferred)
    vals = [b"0.3", b"-0.00", b"9007199254740993", b"2.2250738585072011e-308", b"1e23",
            b"4.9406564584124654e-324", b"1e400", b"-1e400", b"1e-400", b".5", b"5.", b"12.5",
            b"123456789012345678901234567890", b"0.1e0000000000000000000000000001", b"1" + b"0" * 400,
            b"0." + b"0" * 300 + b"1", b"179769313486231580793728971405301e276", b"2.4703282292062327e-324",
            b"2.4703282292062328e-324", b"1.7976931348623157e308", b"1.7976931348623158e308", b"3.14159265358979323846",
            b"1e", b"e5", b"--1", b"", b"nan", b"1_0"]
    ints = [b"9223372036854775807", b"-9223372036854775808", b"9223372036854775808", b"00000000000000000000007",
            b"+5", b"-", b"1.0", b"-0"]
    rows = []
    rng = random.Random(4)
    for i in range(3000):
        f = vals[i % len(vals)] if i < 600 else (str(rng.randint(0, 10**25)).encode() + b"." +
                                                 str(rng.randint(0, 10**12)).encode() +
                                                 (b"e" + str(rng.randint(-340, 310)).encode() if i % 3 else b""))
        rows.append(f + b"," + ints[i % len(ints)] + b"\n")
    data = b"".join(rows)
    run_all_paths("csv", data, [oracle.FLOAT64, oracle.INT64], label="numbers")


def test_quoted_numbers_with_inner_quotes():
    # a typed field whose raw span holds control bytes ('""' inside quotes) goes through the
    # re-simulating device tier; DATA bytes '1"2' are not a number -> null, same as the oracle
    data = b'"1""2",3\n"4",""\n"-7","8e1"\n5,"""6"""\n'
    run_all_paths("csv", data, [oracle.INT64, oracle.FLOAT64], label="inner-quotes")


def test_defaults_strict_and_columns():
    data = b"1,\n,2.5\n7\n1,2,3\n"
    run_all_paths("csv", data, [oracle.INT64, oracle.FLOAT64], defaults=[-1, 0.25], label="defaults")
    run_all_paths("csv", data, [oracle.INT64, oracle.FLOAT64], strict=True, label="strict")


def test_format_errors_first_invalid():
    for s in [b'"x"y\n', b'"abc', b'"a"\r\n', b'a"b\n', b"ok,1\n" * 5000 + b'a"b\n' + b"x\n" * 100]:
        run_all_paths("csv", s, [oracle.SPAN], label=repr(s[:10]))


def test_capacity_needmore():
    data, _ = datagen.generate("cfg1", 100_000)
    w = datagen.WORKLOADS["cfg1"]
    schema = parpa.Schema(list(w.types))
    ora = oracle.parse("csv", data, w.C, w.types)
    cols = parpa.alloc_columns(schema, 10)
    st = parpa.new_stats_tensor()
    parpa.parse_into(dfa("csv"), schema, dev(data), cols, 10, st)
    s = parpa.stats_from_tensor(st)
    assert s["status"] == parpa.ENEEDMORE and s["records"] == ora.R
    assert np.array_equal(to_np(cols[0].offset).view(np.uint64)[:10], ora.offset[0][:10])


def test_misaligned_input_pointer():
    data, _ = datagen.generate("yelp", 500_000)
    buf = dev(b"x" + bytes(data))
    w = datagen.WORKLOADS["yelp"]
    schema = parpa.Schema(list(w.types))
    ora = oracle.parse("csv", data, w.C, w.types)
    res = parpa.parse(dfa("csv"), schema, buf[1:])
    compare(res, ora, w.types, "misaligned")


def test_parse_host_end_to_end():
    data, _ = datagen.generate("taxi", 1_000_000)
    w = datagen.WORKLOADS["taxi"]
    ora = oracle.parse("csv", data, w.C, w.types)
    stats, cols = parpa.parse_host(dfa("csv"), parpa.Schema(list(w.types)), data, ora.R + 1)
    assert stats["status"] == 0 and stats["records"] == ora.R
    for c, t in enumerate(w.types):
        assert np.array_equal(cols[c][0], ora.offset[c])
        assert np.array_equal(cols[c][1], ora.length[c])
        if t != oracle.SPAN:
            assert np.array_equal(cols[c][3], ora.valid[c])
            assert np.array_equal(cols[c][2].view(np.int64), ora.value[c])


@pytest.mark.parametrize("name,part", [("cfg1", 65536), ("yelp", 300_000), ("clf", 131072), ("taxi", 200_000),
                                       ("cfg1", 4096 + 17)])
def test_parse_host_streaming_partitions(name, part, monkeypatch):
    """parpa_parse_host in streaming mode: small partitions force many cuts inside
    records, quoted fields and typed values; the assembled host columns must equal the oracle."""
    monkeypatch.setenv("PARPA_STREAM_PARTITION", str(part))
    w = datagen.WORKLOADS[name]
    data, g = datagen.generate(name, 2_500_000)
    ora = oracle.parse(w.dialect, data, w.C, list(w.types))
    stats, cols = parpa.parse_host(dfa(w.dialect), parpa.Schema(list(w.types)), data, ora.R + 1)
    assert stats["status"] == 0 and stats["records"] == ora.R == g.records, stats
    assert stats["fields"] == ora.nfields and stats["missing_records"] == ora.n_missing
    for c, t in enumerate(w.types):
        assert np.array_equal(cols[c][0], ora.offset[c]), (name, c)
        assert np.array_equal(cols[c][1], ora.length[c]), (name, c)
        if t != oracle.SPAN:
            assert np.array_equal(cols[c][3], ora.valid[c]), (name, c)
            assert np.array_equal(cols[c][2].view(np.int64), ora.value[c]), (name, c)


def test_parse_host_streaming_needmore_and_format_error(monkeypatch):
    monkeypatch.setenv("PARPA_STREAM_PARTITION", "8192")
    w = datagen.WORKLOADS["cfg1"]
    data, g = datagen.generate("cfg1", 100_000)
    stats, cols = parpa.parse_host(dfa("csv"), parpa.Schema(list(w.types)), data, g.records // 2)
    assert stats["status"] == parpa.ENEEDMORE and stats["records"] == g.records
    ora = oracle.parse("csv", data, w.C, list(w.types))
    for c in range(w.C):
        assert np.array_equal(cols[c][0], ora.offset[c][:g.records // 2])
    wt = datagen.WORKLOADS["taxi"]
    tdata, tg = datagen.generate("taxi", 100_000)
    bad = bytearray(tdata)
    pos = next(i for i in range(60_000, 70_000) if chr(bad[i - 1]).isdigit() and chr(bad[i]).isdigit())
    bad[pos] = ord('"')                                        # quote inside an unquoted field -> INV
    orab = oracle.parse("csv", bytes(bad), wt.C, list(wt.types))
    stats, _ = parpa.parse_host(dfa("csv"), parpa.Schema(list(wt.types)), bytes(bad), tg.records + 1)
    assert orab.status == oracle.EFORMAT
    assert stats["status"] == parpa.EFORMAT and stats["first_invalid"] == orab.first_invalid


TS_COLS = {"taxi": [1, 2], "yelp": [8], "clf": [3]}


@pytest.mark.parametrize("name", ["taxi", "yelp", "clf"])
def test_timestamp_columns(name):
    """the workloads' datetime columns parsed as TIMESTAMP (int64 epoch seconds)."""
    w = datagen.WORKLOADS[name]
    types = list(w.types)
    for c in TS_COLS[name]:
        types[c] = oracle.TIMESTAMP
    data, g = datagen.generate(name, 1_500_000)
    ora = run_all_paths(w.dialect, data, types, label=name + "/ts")
    assert ora.R == g.records
    for c in TS_COLS[name]:
        assert ora.valid[c].mean() > 0.95, (name, c)                 # the generator writes valid datetimes


def test_timestamp_edge_cases():
    rows = [b"1970-01-01 00:00:00", b"2000-02-29 23:59:59", b"1900-02-29 00:00:00", b"2019-04-31 10:00:00",
            b"2038-01-19T03:14:08", b"0001-01-01 00:00:00", b"9999-12-31 23:59:59", b"2019-1-01 00:00:00",
            b"", b"x", b"2019-01-01 00:00:00.5", b'"2019-01-01 00:00:00"', b'"2019-01-01 ""00:00:00"']
    data = b"".join(b"%d,%s\n" % (i, r) for i, r in enumerate(rows)) * 50
    types = [oracle.INT64, oracle.TIMESTAMP]
    run_all_paths("csv", data, types, label="ts-edge")
    run_all_paths("csv", data, types, defaults=[None, 12345], label="ts-edge-default")


@pytest.mark.parametrize("name,cols", [("cfg1", range(8)), ("yelp", [0, 7, 8]), ("clf", [2, 3, 4]),
                                       ("taxi", [1, 6])])
def test_strings_materialisation(name, cols):
    """DATA bytes of every field of a column (control bytes dropped), Arrow layout."""
    w = datagen.WORKLOADS[name]
    data, g = datagen.generate(name, 2_000_000)
    d = dev(data)
    res = parpa.parse(dfa(w.dialect), parpa.Schema(list(w.types)), d)
    R = res.records
    for c in cols:
        ro, rs = oracle.strings(w.dialect, data, w.C, c, list(w.types))
        offs, buf = parpa.strings(dfa(w.dialect), d, res.columns[c], R)
        assert np.array_equal(offs.cpu().numpy(), ro), (name, c)
        assert bytes(buf.cpu().numpy()) == rs, (name, c)


def test_strings_escapes_missing_and_empty():
    data = b'a,"x""y",z\n"p,q"\n,,\n"multi\nline",""\n' * 3000 + b'"tail ""quoted"" text, with, commas",9'
    types = [oracle.SPAN] * 3
    d = dev(data)
    res = parpa.parse(dfa("csv"), parpa.Schema(types), d)
    for c in range(3):
        ro, rs = oracle.strings("csv", data, 3, c)
        offs, buf = parpa.strings(dfa("csv"), d, res.columns[c], res.records)
        assert np.array_equal(offs.cpu().numpy(), ro) and bytes(buf.cpu().numpy()) == rs, c


def _oracle_field_counts(dialect, data):
    """Fields per record from the oracle's per-byte emission kinds (a sequential walk)."""
    r = oracle.parse(dialect, data, 1, trace=True)
    counts, c = [], 0
    for k in r.trace_kind.tolist():
        if k == 2:
            c += 1
        elif k == 3:
            counts.append(c + 1)
            c = 0
    if r.eoi_action == 1:
        counts.append(c + 1)
    return counts


@pytest.mark.parametrize("name", ["cfg1", "yelp", "clf", "taxi"])
def test_infer_columns_workloads(name):
    w = datagen.WORKLOADS[name]
    data, g = datagen.generate(name, 1_200_000)
    R, mn, mx = parpa.infer_columns(dfa(w.dialect), dev(data))
    assert (R, mn, mx) == (g.records, w.C, w.C)


def test_infer_columns_ragged():
    rng = random.Random(5)
    rows = []
    for i in range(20000):
        n = rng.choice([1, 2, 3, 7, 40]) if i % 97 else rng.randint(1, 300)
        rows.append(",".join(('"a,\n"' if rng.random() < 0.1 else str(rng.randint(0, 999))) for _ in range(n)))
    data = ("\n".join(rows)).encode()                          # no trailing newline: EOI record
    counts = _oracle_field_counts("csv", data)
    R, mn, mx = parpa.infer_columns(dfa("csv"), dev(data))
    assert (R, mn, mx) == (len(counts), min(counts), max(counts))


def test_skipped_columns():
    """columns with NULL pointers are skipped; the others equal the full parse."""
    w = datagen.WORKLOADS["cfg1"]
    data, g = datagen.generate("cfg1", 400_000)
    ora = oracle.parse("csv", data, w.C, list(w.types))
    schema = parpa.Schema(list(w.types))
    cap = ora.R + 1
    cols = parpa.alloc_columns(schema, cap)
    keep = [0, 2, 5]
    cols = [c if i in keep else parpa.Column(None, None) for i, c in enumerate(cols)]
    st = parpa.new_stats_tensor()
    parpa.parse_into(dfa("csv"), schema, dev(data), cols, cap, st)
    s = parpa.stats_from_tensor(st)
    assert s["status"] == 0 and s["records"] == ora.R and s["missing_records"] == ora.n_missing
    for c in keep:
        assert np.array_equal(to_np(cols[c].offset).view(np.uint64)[:ora.R], ora.offset[c])
        assert np.array_equal(to_np(cols[c].length).view(np.uint32)[:ora.R], ora.length[c])
        if w.types[c] != oracle.SPAN:
            assert np.array_equal(to_np(cols[c].value).view(np.int64)[:ora.R], ora.value[c])


@pytest.mark.parametrize("big", [3_000_000, 9_000_001])
def test_giant_field_spanning_tiles_and_scan_blocks(big):
    """SURVEY N4 (the paper's 200 MB-record experiment, scaled): one quoted field of several MB, with
    escaped quotes and newlines inside, between ordinary records; plus a long numeric field."""
    rng = random.Random(big)
    body = bytearray()
    while len(body) < big:
        body += rng.choice([b"word ", b"x,y ", b'""q"" ', b"\n", b"zz "])
    data = (b"1,a,2.5\n" * 1000 + b'2,"' + bytes(body) + b'",3.25\n' + b"3,b,0." + b"1" * 5000 + b"\n" +
            b"4,c,7\n" * 1000)
    types = [oracle.INT64, oracle.SPAN, oracle.FLOAT64]
    run_all_paths("csv", data, types, label=f"giant-{big}")


@pytest.mark.parametrize("name", ["cfg1", "yelp", "clf", "taxi"])
def test_infer_types_workloads(name):
    """per-column inferred type and field-class set equal the oracle's."""
    w = datagen.WORKLOADS[name]
    data, g = datagen.generate(name, 600_000)
    types, masks, R = parpa.infer_types(dfa(w.dialect), dev(data), w.C)
    ora = oracle.infer_types(w.dialect, data, w.C)
    assert R == g.records
    assert types == [t for t, _ in ora], (types, ora)
    assert masks == [sum(1 << oracle.CLASSES.index(c) for c in cls) for _, cls in ora]


def test_infer_types_constructed():
    """Random fields of every class (integer widths at their endpoints, floats, exponents, bad numbers,
    ISO / CLF datetimes valid and not, strings, empties), some quoted and some with "" escapes (control
    bytes inside the span), missing fields in short records, across several warp tiles."""
    from tests.test_oracle_types import sample_fields
    rng = random.Random(77)
    C = 6
    rows = []
    for r in range(6000):
        fs = sample_fields(rng, C)
        for i, f in enumerate(fs):
            if rng.random() < 0.15:
                fs[i] = b'"' + f + b'"'
            elif rng.random() < 0.03:
                fs[i] = b'"' + f[:1] + b'""' + f[1:] + b'"'
        if rng.random() < 0.05:
            fs = fs[:rng.randint(1, C)]
        # one column per class family so that several resolve to non-string types
        rows.append(b",".join(fs))
    data = b"\n".join(rows) + b"\n"
    col_ints = b"\n".join(str(rng.randint(-30000, 30000)).encode() for _ in range(5000)) + b"\n"
    for d, n in ((data, C), (col_ints, 1)):
        types, masks, R = parpa.infer_types(dfa("csv"), dev(d), n)
        ora = oracle.infer_types("csv", d, n)
        assert types == [t for t, _ in ora], (types, ora)
        assert masks == [sum(1 << oracle.CLASSES.index(c) for c in cls) for _, cls in ora]
    assert parpa.infer_types(dfa("csv"), dev(col_ints), 1)[0] == ["int16"]


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_plain_tiles_ragged_empty_and_giant(seed):
    """Tiles without control bytes (the direct delimiter-list paths of k_emit): many short records per tile
    (column-uniform writes) with empty fields (defaults on some typed columns), records with missing and
    extra fields, numbers of every window length (1-20 characters, far more device-tier fields than the
    defer queue holds), and unquoted giant fields of 3-70 KB (field 0 of later tiles begins tiles
    earlier) in span and typed columns."""
    from tests.gpu_helpers import adversarial_plain
    data, types = adversarial_plain(seed)
    run_all_paths("csv", data, types, label=f"plain{seed}")
    run_all_paths("csv", data, types, defaults=[-7, 0.5, None, None, -0.0, None, 3, None], label=f"plain{seed}/defaults")


@pytest.mark.parametrize("seed", [4, 5])
def test_quoted_tiles_deferred_overflow(seed):
    """Tiles with control bytes and far more device-tier fields than the defer queue holds (len / 512):
    quoted numbers, numbers with "" inside (inner control bytes: invalid, decided by the device tier),
    exponents beyond the fast path, 20+ digit floats, ragged records, quoted giant fields."""
    rng = random.Random(seed)
    types = [oracle.FLOAT64, oracle.INT64, oracle.SPAN, oracle.FLOAT64]
    rows = []
    for r in range(30000):
        fs = []
        for t in types:
            k = rng.random()
            if t == oracle.SPAN:
                f = '"' + "".join(rng.choice('ab,\n ') for _ in range(rng.randint(0, 20))) + '"'
            elif k < 0.25:
                f = '"' + str(rng.randint(-999, 999)) + '"'
            elif k < 0.45:
                f = '"' + str(rng.randint(0, 99)) + '""' + str(rng.randint(0, 9)) + '"'
            elif k < 0.65 and t == oracle.FLOAT64:
                f = f"{rng.randint(1, 9)}e{rng.choice([23, 50, -30, 300, -320])}"
            elif k < 0.8 and t == oracle.FLOAT64:
                f = "".join(rng.choice("0123456789") for _ in range(rng.randint(17, 30))) + "." + str(rng.randint(0, 99))
            else:
                f = str(rng.randint(-10**6, 10**6))
            fs.append(f)
        if rng.random() < 0.05:
            fs = fs[:rng.randint(1, 3)]
        if rng.random() < 0.001:
            fs[0] = '"' + "x" * rng.randint(3000, 40000) + '""' + '"'
        rows.append(",".join(fs))
    data = ("\n".join(rows) + "\n").encode()
    ora = run_all_paths("csv", data, types, label=f"quoted{seed}")
    assert sum(1 for c in (0, 1, 3) for v in ora.valid[c] if v == 0) > 5000      # many invalid (device tier)


@pytest.mark.parametrize("seed", [1, 2])
def test_clf_adversarial(seed):
    """The 9-state CLF DFA on adversarial lines (tests/gpu_helpers.adversarial_clf): enclosed fields with
    escapes, directive lines, '#' inside tokens and at line start, ragged lines, long / quoted / '-' numbers."""
    from tests.gpu_helpers import adversarial_clf
    data, types = adversarial_clf(seed)
    ora = run_all_paths("clf", data, types, label=f"clf{seed}")
    assert ora.status == 0 and ora.n_missing > 0 and ora.n_extra > 0


def test_csv_comment_adversarial():
    """CSV + '#' comment lines (reading R19): comments with quotes, commas and brackets between records,
    '#' inside fields and quoted fields, quoted multi-line fields that contain '\\n#' (not a comment)."""
    rng = random.Random(21)
    lines = []
    for _ in range(25000):
        r = rng.random()
        if r < 0.05:
            lines.append("#" + "".join(rng.choice('a,"#[] x') for _ in range(rng.randint(0, 40))))
        else:
            fs = []
            for c in range(4):
                k = rng.random()
                if k < 0.3:
                    fs.append('"' + "".join(rng.choice('ab,#\n x') for _ in range(rng.randint(0, 15))).replace('"', '""') + '"')
                elif k < 0.5 and c > 0:                       # (a leading '#' would make the line a comment)
                    fs.append("#" + str(rng.randint(0, 99)))
                else:
                    fs.append(str(rng.randint(-10 ** 9, 10 ** 9)))
            lines.append(",".join(fs[:rng.choice([4, 4, 4, 2, 5])] if rng.random() < 0.1 else fs))
    data = ("\n".join(lines) + "\n").encode()
    types = [oracle.SPAN, oracle.INT64, oracle.SPAN, oracle.INT64]
    ora = run_all_paths("csv_comment", data, types, label="csvc")
    assert ora.status == 0


@pytest.mark.parametrize("kind", ["clf", "plain"])
def test_strings_and_types_adversarial(kind):
    """String columns (N3) and type inference (N2) on the adversarial generators: enclosed fields with
    escapes, giant fields across tiles, ragged records (missing fields give empty strings)."""
    from tests.gpu_helpers import adversarial_clf, adversarial_plain
    data, types = adversarial_clf(4, 15000) if kind == "clf" else adversarial_plain(5, 15000)
    dialect = "clf" if kind == "clf" else "csv"
    C = len(types)
    d = dev(data)
    res = parpa.parse(dfa(dialect), parpa.Schema([oracle.SPAN] * C), d)
    for c in range(C):
        ro, rs = oracle.strings(dialect, data, C, c)
        offs, buf = parpa.strings(dfa(dialect), d, res.columns[c], res.records)
        assert np.array_equal(offs.cpu().numpy(), ro), (kind, c)
        assert bytes(buf.cpu().numpy()) == rs, (kind, c)
    got, masks, R = parpa.infer_types(dfa(dialect), d, C)
    ora = oracle.infer_types(dialect, data, C)
    assert got == [t for t, _ in ora], (got, ora)
    assert masks == [sum(1 << oracle.CLASSES.index(x) for x in cls) for _, cls in ora]


def test_merged_states_exact_at_the_end():
    """Device states are classes of DFA states with identical rows (CSV: EOR and EOF differ only in their
    end-of-input action).  Inputs ending in each of them must still take the right EOI action, report
    the exact final state, and summarise to the exact transition vector (the oracle's final state)."""
    for data in [b"a,b\nc,", b",", b"x,\n", b"1,2\n3,4\n" * 40 + b"5,", b"q\n" * 70, b'"a",', b'a,"b"\n,']:
        types = [oracle.INT64, oracle.SPAN]
        ora = run_all_paths("csv", data, types, label=repr(data[-8:]))
        ro = oracle.parse("csv", data, 2, types, trace=True)
        tau = parpa.summarize(dfa("csv"), dev(data))
        assert tau[0] == ro.final_state, (data[-8:], tau, ro.final_state)
        res = parpa.parse(dfa("csv"), parpa.Schema(types), dev(data))
        assert res.stats["final_state"] == ro.final_state, (data[-8:], res.stats)


@pytest.mark.parametrize("name", ["bruteforce", "cfg1", "yelp", "clf"])
def test_production_masks_equal_oracle_kinds(name):
    """The DATA / DELIM / RECORD masks pass 2 stores for the emission kernel (not a debug re-simulation),
    bit for bit against the oracle's per-byte emission kinds (DELIM = field or record
    delimiter, RECORD ⊂ DELIM; invalid tail bits of the last chunk are zero)."""
    if name == "bruteforce":
        data = b"".join(b"".join(t) + b"\n" for n in range(7) for t in itertools.product(ALPH, repeat=n))
        dialect = "csv"
    else:
        w = datagen.WORKLOADS[name]
        data, _ = datagen.generate(name, 2_000_000)
        data, dialect = bytes(data), w.dialect
    ora = oracle.parse(dialect, data, 1, trace=True)
    m = parpa.debug_masks(dfa(dialect), dev(data))
    k = ora.trace_kind
    n = len(data)
    pad = (-n) % 64
    kk = np.concatenate([k, np.full(pad, 1, np.uint8)]).reshape(-1, 64)      # pad as CTRL (no bits)
    w64 = (1 << np.arange(64, dtype=np.uint64)).astype(np.uint64)
    exp_d = ((kk == oracle.DATA).astype(np.uint64) * w64).sum(axis=1, dtype=np.uint64)
    exp_f = ((kk >= oracle.FIELD).astype(np.uint64) * w64).sum(axis=1, dtype=np.uint64)
    exp_r = ((kk == oracle.RECORD).astype(np.uint64) * w64).sum(axis=1, dtype=np.uint64)
    assert np.array_equal(m[:, 0], exp_d)
    assert np.array_equal(m[:, 1], exp_f)
    assert np.array_equal(m[:, 2], exp_r)


@pytest.mark.parametrize("name,nbytes", [("cfg1", 600_000), ("taxi", 3_000_000), ("yelp", 3_000_000)])
def test_skip_records(name, nbytes):
    """Skipping a user-specified set of records: the records listed (the first, a run, random
    ones, the last) are not written; every other record lands in the next row, bit-exact vs the oracle's
    parse with those rows removed.  (cfg1 at 600 KB runs the one-launch k_small path, the others the
    multi-kernel path.)"""
    import torch
    w = datagen.WORKLOADS[name]
    data, g = datagen.generate(name, nbytes)
    ora = oracle.parse(w.dialect, data, w.C, list(w.types))
    rng = random.Random(7)
    R = ora.R
    skip = sorted(set([0, 1, 2, R - 1] + list(range(R // 2, R // 2 + 40)) + rng.sample(range(R), R // 10)))
    keep = np.setdiff1d(np.arange(R), np.array(skip))
    schema = parpa.Schema(list(w.types))
    cols = parpa.alloc_columns(schema, R)
    st = parpa.new_stats_tensor()
    sk = torch.tensor(skip, dtype=torch.int64, device="cuda")
    parpa.parse_into(dfa(w.dialect), schema, dev(data), cols, R, st, skip_records=sk)
    s = parpa.stats_from_tensor(st)
    assert s["status"] == 0 and s["records"] == len(keep), s
    n = len(keep)
    for c, t in enumerate(w.types):
        assert np.array_equal(to_np(cols[c].offset).view(np.uint64)[:n], ora.offset[c][keep]), c
        assert np.array_equal(to_np(cols[c].length).view(np.uint32)[:n], ora.length[c][keep]), c
        if t != oracle.SPAN:
            assert np.array_equal(to_np(cols[c].valid)[:n], ora.valid[c][keep]), c
            assert np.array_equal(to_np(cols[c].value).view(np.int64)[:n], ora.value[c][keep]), c


@pytest.mark.parametrize("name,nbytes", [("cfg1", 400_000), ("yelp", 3_000_000)])
def test_skip_rows_compaction(name, nbytes):
    """Skipping rows: raw lines (quoting ignored — yelp records span several rows) removed by
    the device stream compaction equal the plain definition (split after every '\\n', drop the listed
    indices, concatenate); the compacted input then parses exactly like the oracle's parse of it."""
    import torch
    w = datagen.WORKLOADS[name]
    data, _ = datagen.generate(name, nbytes)
    data = bytes(data) + b"tail without newline"
    lines = data.splitlines(keepends=True)
    rng = random.Random(5)
    skip = sorted(set([0, 1, len(lines) - 1, len(lines) // 3] + rng.sample(range(len(lines)), len(lines) // 7)))
    exp = b"".join(l for i, l in enumerate(lines) if i not in set(skip))
    got = parpa.compact_rows(dev(data), torch.tensor(skip, dtype=torch.int64, device="cuda"))
    assert bytes(to_np(got).tobytes()) == exp
    assert bytes(to_np(parpa.compact_rows(dev(data), None)).tobytes()) == data          # nothing skipped
    run_all_paths(w.dialect, exp, w.types, label=name + "/compacted")   # valid or not, GPU == oracle
