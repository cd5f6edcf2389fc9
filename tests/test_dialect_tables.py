"""The tables the GPU consumes (paper_1905_13415_b200.dialects) encode exactly the oracle's languages.

The oracle's dialects are hand-written control flow; its generic table walker is fed the
product's tables; per-byte states, emissions and all outputs must coincide on fuzz and on
the generated workloads.  Also: random DFAs — the ∘-scan of per-chunk τ
equals the sequential walk for every chunking.
"""
import random

import numpy as np
import pytest

import datagen
import oracle
from oracle import primitives as P
from paper_1905_13415_b200 import dialects

ALPH = {
    "csv": b'\n",ab1',
    "csv_comment": b'\n",#ab1',
    "clf": b'\n "[]\\#a1',
}


def same(a, b):
    assert a.status == b.status and a.R == b.R and a.first_invalid == b.first_invalid
    assert a.trace_state.tolist() == b.trace_state.tolist()
    assert a.trace_kind.tolist() == b.trace_kind.tolist()
    for c in range(len(a.offset)):
        assert a.offset[c].tolist() == b.offset[c].tolist()
        assert a.length[c].tolist() == b.length[c].tolist()


@pytest.mark.parametrize("name", ["csv", "csv_comment", "clf"])
def test_tables_equal_handwritten_fuzz(name):
    t = dialects.get(name)
    rng = random.Random(hash(name) & 0xFFFF)
    alph = ALPH[name]
    for _ in range(3000):
        s = bytes(rng.choice(alph) for _ in range(rng.randint(0, 40)))
        same(oracle.parse(name, s, 4, trace=True), oracle.parse_tables(t.as_dict(), s, 4, trace=True))


@pytest.mark.parametrize("name,wl", [("csv", "cfg1"), ("csv", "yelp"), ("clf", "clf"), ("csv_comment", "taxi")])
def test_tables_equal_handwritten_workloads(name, wl):
    t = dialects.get(name)
    data, _ = datagen.generate(wl, 300_000)
    w = datagen.WORKLOADS[wl]
    same(oracle.parse(name, data, w.C, trace=True), oracle.parse_tables(t.as_dict(), data, w.C, trace=True))


@pytest.mark.parametrize("name", ["csv", "csv_comment", "clf"])
def test_invalid_state_absorbing_and_catch_all_idempotent(name):
    t = dialects.get(name)
    for g in range(t.G):
        assert t.transition[g][t.invalid] == t.invalid
    ca = t.transition[t.G - 1]
    assert [ca[s] for s in ca] == ca          # r∘r = r: the catch-all row is idempotent


def random_dfa(rng):
    S = rng.randint(2, 16)
    G = rng.randint(2, 8)
    trans = [[rng.randrange(S) for _ in range(S)] for _ in range(G)]
    gob = [rng.randrange(G) for _ in range(256)]
    return S, G, trans, gob


def test_random_dfa_chunked_scan_equals_sequential():
    # 1,000 random DFAs, random start state, chunk sizes 1-17.
    rng = random.Random(2024)
    for _ in range(1000):
        S, G, trans, gob = random_dfa(rng)
        start = rng.randrange(S)
        tables = {"group_of_byte": gob, "transition": trans, "emit": [[0] * S] * G, "eoi": [0] * S,
                  "start": start, "invalid": S - 1}
        s = bytes(rng.randrange(256) for _ in range(rng.randint(0, 120)))
        r = oracle.parse_tables(tables, s, 1, trace=True)
        seq = r.trace_state.tolist() + [r.final_state]
        cs = rng.randint(1, 17)
        starts = list(range(0, len(s), cs))
        taus = [P.tau(trans, gob, s[i:i + cs]) for i in starts]
        pref = P.exclusive_scan(taus, P.compose, P.identity_vector(S))
        assert [p[start] for p in pref] == [seq[i] for i in starts]
