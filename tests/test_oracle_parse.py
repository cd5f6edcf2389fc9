"""Pins for the oracle's sequential parse (fixtures, brute force, Python csv, closed forms, G1)."""
import csv
import io
import itertools
import json
import os
import random

import numpy as np
import pytest

import datagen
import oracle
from oracle import primitives as P

GOLD = os.path.join(os.path.dirname(__file__), "golden")
with open(os.path.join(GOLD, "fixtures.json")) as f:
    FIX = json.load(f)
with open(os.path.join(GOLD, "tab_ttable.json")) as f:
    TT = json.load(f)

# tab:ttable as printed (golden), used only to drive the oracle's table walker
_ST = {n: i for i, n in enumerate(TT["states"])}
PAPER_TRANSITION = [[_ST[s] for s in TT["rows"][sym]] for sym in ["\n", '"', ",", "*"]]
PAPER_GOB = [3] * 256
PAPER_GOB[ord("\n")], PAPER_GOB[ord('"')], PAPER_GOB[ord(",")] = 0, 1, 2
ALPHABET = [b"\n", b'"', b",", b"a"]


def data_bytes(data: bytes, r, kinds, c):
    """DATA bytes of each field of column c (the paper's CSS content)."""
    out = []
    for o, n in zip(r.offset[c].tolist(), r.length[c].tolist()):
        if n == oracle.MISSING_LEN:
            out.append(None)
        else:
            out.append(bytes(data[i] for i in range(o, o + n) if kinds[i] == oracle.DATA))
    return out


@pytest.mark.parametrize("fx", FIX["csv"], ids=lambda f: f["cite"][:40])
def test_csv_fixtures(fx):
    data = fx["input"].encode()
    r = oracle.parse("csv", data, fx["C"], trace=True)
    if "status" in fx:
        assert r.status == fx["status"] and r.first_invalid == fx["first_invalid"]
        return
    assert r.status == oracle.OK
    assert r.R == fx["R"]
    if "n_missing" in fx:
        assert r.n_missing == fx["n_missing"]
    if "spans" in fx:
        for row, spans in enumerate(fx["spans"]):
            for c, (o, n) in enumerate(spans):
                assert (int(r.offset[c][row]), int(r.length[c][row])) == (o, n)
    if "data" in fx:
        got = [data_bytes(data, r, r.trace_kind, c)[0] for c in range(fx["C"])]
        assert got == [d.encode() for d in fx["data"]]


def test_context_example_naive_start_misparses():
    # fig:contextex: a chunk starting inside the quotes must enter in ENC; starting it in
    # EOR emits false delimiters.  The sequential trace gives the true entry state at every cut.
    data = b'1,"Hello, World\nHow are you?",3\n'
    r = oracle.parse("csv", data, 3, trace=True)
    assert r.trace_state[8] == _ST["ENC"]
    naive = oracle.parse("csv", data[8:], 3, trace=True)
    kinds = naive.trace_kind.tolist()
    assert kinds[0] == oracle.FIELD          # the ',' inside the quotes (byte 8)
    assert kinds[15 - 8] == oracle.RECORD    # the '\n' inside the quotes (byte 15)
    assert naive.first_invalid == 28 - 8     # the closing quote (byte 28) is then read in FLD -> INV


@pytest.mark.parametrize("dialect", ["csv_comment", "clf"])
def test_dialect_fixtures(dialect):
    for fx in FIX[dialect]:
        data = fx["input"].encode()
        types = [oracle.SPAN] * fx["C"]
        if dialect == "clf":
            types[5] = types[6] = oracle.INT64
        r = oracle.parse(dialect, data, fx["C"], types=types, trace=True)
        assert r.status == oracle.OK and r.R == fx["R"]
        got = []
        for row in range(r.R):
            for c in range(fx["C"]):
                got.append(data_bytes(data, r, r.trace_kind, c)[row])
        assert got == [d.encode() for d in fx["data"]]
        if "ints" in fx:
            for row, vals in enumerate(fx["ints"]):
                for k, c in enumerate([5, 6]):
                    if vals[k] is None:
                        assert r.valid[c][row] == 0
                    else:
                        assert r.valid[c][row] == 1 and r.value[c][row] == vals[k]


def all_strings(maxlen):
    for n in range(maxlen + 1):
        for t in itertools.product(ALPHABET, repeat=n):
            yield b"".join(t)


def test_oracle_csv_matches_paper_table_walker_bruteforce():
    # The hand-written CSV dialect == a table walker over tab:ttable as PRINTED (golden), on every
    # string of length <= 7 over {\n, ", ",", a}: pins the oracle's transitions to the paper.
    tables = {"group_of_byte": PAPER_GOB, "transition": PAPER_TRANSITION,
              "emit": [[0] * 6] * 4, "eoi": [0] * 6, "start": 0, "invalid": 5}
    for s in all_strings(7):
        a = oracle.parse("csv", s, 1, trace=True)
        b = oracle.parse_tables(tables, s, 1, trace=True)
        assert a.trace_state.tolist() == b.trace_state.tolist()
        assert a.final_state == b.final_state


def test_composition_equals_sequential_bruteforce():
    # for every string and every cut, the exclusive ∘-scan of per-chunk τ seeded with the
    # identity, read at the start state, equals the sequential state at the cut.
    for s in all_strings(6):
        r = oracle.parse("csv", s, 1, trace=True)
        seq = r.trace_state.tolist() + [r.final_state]
        for cut in range(len(s) + 1):
            ta = P.tau(PAPER_TRANSITION, PAPER_GOB, s[:cut])
            tb = P.tau(PAPER_TRANSITION, PAPER_GOB, s[cut:])
            assert ta[0] == seq[cut]
            assert P.compose(ta, tb)[0] == r.final_state


def test_chunked_scan_random_chunk_sizes():
    # SPEC S:224 / O10: entry states of every chunk are independent of the chunk size.
    rng = random.Random(11)
    for _ in range(300):
        s = b"".join(rng.choice(ALPHABET) for _ in range(rng.randint(0, 60)))
        r = oracle.parse("csv", s, 1, trace=True)
        seq = r.trace_state.tolist() + [r.final_state]
        for cs in (1, 2, 3, 7, 16, 31):
            starts = list(range(0, len(s), cs))
            taus = [P.tau(PAPER_TRANSITION, PAPER_GOB, s[i:i + cs]) for i in starts]
            pref = P.exclusive_scan(taus, P.compose, P.identity_vector(6))
            assert [p[0] for p in pref] == [seq[i] for i in starts]


def test_python_csv_crosscheck_bruteforce():
    # Library pin: on every DFA-valid LF input of length <= 8 without blank lines, the DATA bytes of
    # each field equal Python's csv.reader(strict=True) values.
    checked = 0
    for s in all_strings(8):
        r = oracle.parse("csv", s, 16, trace=True)
        if r.status != oracle.OK:
            continue
        text = s.decode()
        if text.startswith("\n") or "\n\n" in text:
            pass
        rows = list(csv.reader(io.StringIO(text, newline=""), strict=True))
        if any(len(row) == 0 for row in rows):      # csv returns [] for a blank line (reading R5)
            continue
        kinds = r.trace_kind.tolist()
        got = []
        for row in range(r.R):
            fields = []
            for c in range(16):
                if r.length[c][row] == oracle.MISSING_LEN:
                    break
                o, n = int(r.offset[c][row]), int(r.length[c][row])
                fields.append(bytes(s[i] for i in range(o, o + n) if kinds[i] == oracle.DATA).decode())
            got.append(fields)
        assert got == rows, s
        checked += 1
    assert checked > 10000


def test_quote_parity_closed_form():
    # The CSV-specific closed form the paper contrasts with: on valid CSV a non-quote byte is
    # enclosed (state ENC before it) iff an odd number of quotes precede it.
    for s in all_strings(7):
        r = oracle.parse("csv", s, 1, trace=True)
        if r.status != oracle.OK:
            continue
        q = 0
        for i, b in enumerate(s):
            if b != ord('"'):
                assert (r.trace_state[i] == _ST["ENC"]) == (q % 2 == 1)
            else:
                q += 1


def test_record_and_field_count_invariants():
    # fields per record (R*C entries = fields + missing), delimiter counts outside quotes
    data, g = datagen.generate("cfg1", 300_000)
    w = datagen.WORKLOADS["cfg1"]
    r = oracle.parse("csv", data, w.C, w.types, trace=True)
    kinds = r.trace_kind
    assert r.status == 0 and r.R == g.records
    assert int((kinds == oracle.RECORD).sum()) == r.R
    assert int(((kinds == oracle.FIELD) | (kinds == oracle.RECORD)).sum()) == r.nfields == r.R * w.C
    # every '\n' that is not a record delimiter sits inside quotes
    nl = np.flatnonzero(data == ord("\n"))
    inside = nl[kinds[nl] != oracle.RECORD]
    assert (r.trace_state[inside] == _ST["ENC"]).all()


@pytest.mark.parametrize("name", ["cfg1", "taxi", "yelp", "clf"])
def test_generator_ground_truth(name):
    # pin G1: records and int64 column sums / null counts as printed by the generator
    w = datagen.WORKLOADS[name]
    data, g = datagen.generate(name, 2_000_000)
    r = oracle.parse(w.dialect, data, w.C, w.types)
    assert r.status == 0 and r.R == g.records and r.n_missing == 0 and r.n_extra == 0
    ints = [c for c, t in enumerate(w.types) if t == datagen.INT64]
    sums = [int(np.where(r.valid[c] == 1, r.value[c], 0).astype(np.int64).sum()) for c in ints]
    nulls = [int((r.valid[c] == 0).sum()) for c in ints]
    assert sums == g.int_sums and nulls == g.int_nulls


def test_defaults_for_empty_and_missing():
    # P:564-568 (reading R16): empty and missing typed fields take the column default when given.
    r = oracle.parse("csv", b"1,\n,2.5\n7\n", 2, types=[oracle.INT64, oracle.FLOAT64], defaults=[-1, 0.25])
    assert r.R == 3
    assert r.value[0].tolist() == [1, -1, 7] and r.valid[0].tolist() == [1, 1, 1]
    assert r.floats(1).tolist() == [0.25, 2.5, 0.25] and r.valid[1].tolist() == [1, 1, 1]
    r2 = oracle.parse("csv", b"1,\n,2.5\n7\n", 2, types=[oracle.INT64, oracle.FLOAT64])
    assert r2.valid[0].tolist() == [1, 0, 1] and r2.valid[1].tolist() == [0, 1, 0]


def test_strict_columns():
    r = oracle.parse("csv", b"1,Apples\n2\n", 2, strict=True)
    assert r.status == oracle.ECOLUMNS and r.n_missing == 1
    r = oracle.parse("csv", b"1,2,3\n", 2)
    assert r.status == oracle.OK and r.n_extra == 1


@pytest.mark.parametrize("dialect", ["csv_comment", "clf"])
def test_dialect_fixtures_hand_derived(dialect):
    """Transitions of the two invented dialects not covered by the SURVEY Appendix A fixtures, each
    expected value derived by hand from the printed tables (A.2 / A.3), not from the oracle."""
    for fx in FIX[dialect + "_extra"]:
        data = fx["input"].encode()
        r = oracle.parse(dialect, data, fx["C"], types=[oracle.SPAN] * fx["C"], trace=True)
        if fx.get("status") == "EFORMAT":
            assert r.status == oracle.EFORMAT and r.first_invalid == fx["first_invalid"], fx["cite"]
            continue
        assert r.status == oracle.OK and r.R == fx["R"], fx["cite"]
        got = [data_bytes(data, r, r.trace_kind, c)[row] for row in range(r.R) for c in range(fx["C"])]
        assert got == [x.encode() for x in fx["data"]], fx["cite"]
