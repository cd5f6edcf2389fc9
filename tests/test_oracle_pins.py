"""Pins for the oracle's primitives against values the paper prints (tests/golden/*.json)."""
import itertools
import json
import os
import random

import pytest

import oracle
from oracle import primitives as P

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def test_prefix_sum_example():
    g = gold("prefix_sum.json")
    add = lambda a, b: a + b
    assert P.inclusive_scan(g["x"], add, 0) == g["inclusive"]
    assert P.exclusive_scan(g["x"], add, 0) == g["exclusive"]


def test_tab_twiddling_rows():
    g = gold("tab_twiddling.json")
    lu = bytes(g["lookup_bytes"])
    rows = P.swar_trace(lu, g["read_symbol"])
    assert [f"{c:08X}" for c, _, _ in rows] == g["c_words_hex"]
    assert f"{rows[0][1]:08X}" == g["swar_low_word_hex"]
    assert f"{rows[1][1]:08X}" == g["swar_high_word_hex"]
    assert [r[2] for r in rows] == g["bfind_shift3"]
    idx = P.swar_match_paper(lu, g["read_symbol"], 0xFFFFFFFF)
    assert idx == g["idx"]
    assert min(idx, g["catch_all_position"]) == g["min_idx_5"]
    assert g["position_groups"][idx] == 2  # ',' is in symbol group 2 (tab:twiddling "symbol group" row)


def test_H_definition_examples():
    assert P.H(0x50000E26) == 0x00800000   # tab:twiddling
    assert P.H(0x00000000) == 0x80808080
    assert P.H(0x01010101) == 0x00000000


def test_swar_bfind_hazard_and_lsb_fix():
    # Reading R9: with LU = '"' '#' '[' ']' and s = '"', Mycroft's borrow flags lane 1 too.
    lu = b'"#[]'
    rows = P.swar_trace(lu, ord('"'))
    assert rows[0][1] == 0x00008080
    assert P.swar_match_paper(lu, ord('"'), 4) == 1          # MSB pick: wrong lane ('#')
    assert P.swar_match_lsb(lu, ord('"'), 4) == 0            # LSB pick: right lane


@pytest.mark.parametrize("lookup", [b"\n\",", b"\n\",#", b"\n \"[]\\#", b"\n\",|\t", b'"#[]'])
def test_swar_lsb_equals_linear_scan_all_bytes(lookup):
    # brute-force equivalence over all 256 byte values.
    for s in range(256):
        assert P.swar_match_lsb(lookup, s, len(lookup)) == P.naive_match(lookup, s, len(lookup))


def test_mfira_table():
    g = gold("mfira.json")                 # fig:multifrag P:645-649
    assert P.mfira_layout(g["c"], g["b"]) == (g["a"], g["k"], g["fragments"])
    # c=6 items of 3 bits (CSV tau) fit one register; c=9 of 4 bits (CLF tau) need two.
    assert P.mfira_layout(6, 3) == (5, 4, 1)
    assert P.mfira_layout(9, 4) == (3, 2, 2)


def test_tab_ttable_compose_example():
    g = gold("tab_ttable.json")
    st = {n: i for i, n in enumerate(g["states"])}
    row = {k: [st[s] for s in v] for k, v in g["rows"].items()}
    # (a∘b)_i = b_{a_i}: ',' then '\n' from every state
    assert P.compose(row[","], row["\n"]) == [0, 1, 0, 0, 0, 5]
    ident = P.identity_vector(6)
    for r in row.values():
        assert P.compose(ident, r) == r and P.compose(r, ident) == r


def test_compose_associative_random():
    rng = random.Random(7)
    for _ in range(3000):
        S = rng.randint(1, 16)
        a, b, c = ([rng.randrange(S) for _ in range(S)] for _ in range(3))
        assert P.compose(P.compose(a, b), c) == P.compose(a, P.compose(b, c))


def test_combine_offset_examples_and_assoc():
    assert P.combine_offset(("rel", 4), ("abs", 2)) == ("abs", 2)
    assert P.combine_offset(("abs", 3), ("rel", 0)) == ("abs", 3)       # identity
    assert P.exclusive_scan([("rel", 1), ("abs", 2), ("rel", 3)], P.combine_offset, ("rel", 0)) == \
        [("rel", 0), ("rel", 1), ("abs", 2)]
    rng = random.Random(3)
    for _ in range(5000):
        a, b, c = ((rng.choice(["abs", "rel"]), rng.randrange(10)) for _ in range(3))
        assert P.combine_offset(P.combine_offset(a, b), c) == P.combine_offset(a, P.combine_offset(b, c))


def test_fig_parser_two_column_offsets():
    # fig:parser_two: 'a,b,c\nd,e\n' chunked as ["a,b", ",c\nd", ",e\n"]
    data = b"a,b,c\nd,e\n"
    r = oracle.parse("csv", data, 3, trace=True)
    kinds = r.trace_kind.tolist()
    chunks = [(0, 3), (3, 7), (7, 10)]
    per_chunk = [P.chunk_column_offset(kinds[a:b]) for a, b in chunks]
    assert per_chunk == [("rel", 1), ("abs", 0), ("abs", 0)]
    # exclusive ⊕-scan seeded with the stream start (column 0 of record 0)
    entry = P.exclusive_scan(per_chunk, P.combine_offset, ("rel", 0))
    assert entry == [("rel", 0), ("rel", 1), ("abs", 0)]


def test_chunk_column_offset_spec_examples():
    # SPEC S:306-308 in per-byte form (bit j = byte j); corrected prose reading R8
    def kinds(n, rec, col):
        k = [0] * n
        for j in col:
            k[j] = 2
        for j in rec:
            k[j] = 3
        return k
    assert P.chunk_column_offset(kinds(8, [], [1, 5])) == ("rel", 2)
    assert P.chunk_column_offset(kinds(8, [3], [1, 3, 6])) == ("abs", 1)
    assert P.chunk_column_offset(kinds(8, [7], [7])) == ("abs", 0)


def test_blsmsk_formula_disagrees_with_prose():
    # Reading R8: the printed POPCNT((~BLSMSK(rec)) & col) with byte 0 at bit 0 counts field
    # delimiters after the FIRST record delimiter; the prose says after the LAST one.
    rec, col = (1 << 2) | (1 << 5), (1 << 2) | (1 << 4) | (1 << 5) | (1 << 7)
    blsmsk = rec ^ (rec - 1)
    formula = bin(~blsmsk & col & 0xFF).count("1")
    prose = bin(col & ~((1 << 6) - 1) & 0xFF).count("1")
    assert formula == 3 and prose == 1
