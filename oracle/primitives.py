"""Plain-Python statements of the paper's primitives (TEST INFRASTRUCTURE ONLY).

Each function restates one passage of PAPER.md; none is used by the CUDA path.

* ``H`` / ``swar_match_paper`` — tab:twiddling and its prose P:873-884.
* ``swar_match_lsb`` — the same matcher with the lowest-set-bit lane pick (reading R9:
  the paper's bfind (MSB) pick is wrong when a matching lane is followed by a lane
  equal to LU^0x01, because of Mycroft's borrow).
* ``mfira_layout`` — fig:multifrag table: a=floor(32/c), k=2^floor(log2 a),
  fragments=ceil(b/k).
* ``exclusive_scan`` / ``inclusive_scan`` — §2 definitions.
* ``compose`` — the composite operator (a∘b)_i = b_{a_i}.
* ``combine_offset`` — ⊕ on (type, offset) column offsets.
* ``tau`` — the state-transition vector of a chunk: simulate one DFA instance per
  start state.
* ``chunk_column_offset`` — "count field delimiters after the last record delimiter"
  (prose P:400; reading R8), by per-byte replay.
"""
from __future__ import annotations

M32 = 0xFFFFFFFF


def H(x: int) -> int:
    """Mycroft null-byte test as printed under tab:twiddling: ((x-0x01010101) & ~x & 0x80808080)."""
    return ((x - 0x01010101) & (~x) & 0x80808080) & M32


def bfind(x: int) -> int:
    """Position of the most significant set bit; 0xFFFFFFFF if none."""
    return x.bit_length() - 1 if x else 0xFFFFFFFF


def lowest_set(x: int) -> int:
    return (x & -x).bit_length() - 1 if x else 0xFFFFFFFF


def _lu_words(lookup: bytes):
    """Pack lookup bytes four per 32-bit LU-register, byte j of word w = lookup[4w+j]."""
    words = []
    for w in range(0, max(len(lookup), 1), 4):
        part = lookup[w:w + 4]
        v = 0
        for j, b in enumerate(part):
            v |= b << (8 * j)
        words.append((v, len(part)))
    return words


def swar_trace(lookup: bytes, s: int):
    """Per LU-register rows of tab:twiddling: (c = LU xor s-register, H(c), bfind(H(c)) >> 3)."""
    sreg = (s * 0x01010101) & M32                     # "replicate that symbol in every byte"
    rows = []
    for v, _n in _lu_words(lookup):
        c = v ^ sreg
        h = H(c)
        rows.append((c, h, (bfind(h) >> 3) & 0x1FFFFFFF))
    return rows


def swar_match_paper(lookup: bytes, s: int, catch_all_pos: int) -> int:
    """Matching index exactly as P:876-883: min over registers of bfind(H)>>3 (+4 per word), min with catch-all."""
    idx = 0xFFFFFFFF
    for w, (c, h, pos) in enumerate(swar_trace(lookup, s)):
        if pos != 0x1FFFFFFF:
            pos += 4 * w                          # second LU register holds positions 4..7 (reading R9 ii)
        idx = min(idx, pos)
    return min(idx, catch_all_pos)


def swar_match_lsb(lookup: bytes, s: int, catch_all_pos: int) -> int:
    """Reading R9: pick the lowest flagged lane (borrows only propagate upwards)."""
    sreg = (s * 0x01010101) & M32
    idx = 0xFFFFFFFF
    for w, (v, _n) in enumerate(_lu_words(lookup)):
        h = H(v ^ sreg)
        pos = (lowest_set(h) >> 3) & 0x1FFFFFFF
        if pos != 0x1FFFFFFF:
            pos += 4 * w
        idx = min(idx, pos)
    return min(idx, catch_all_pos)


def naive_match(lookup: bytes, s: int, catch_all_pos: int) -> int:
    """Linear scan with catch-all fallback."""
    for i, b in enumerate(lookup):
        if b == s:
            return i
    return catch_all_pos


def mfira_layout(c: int, b: int):
    """fig:multifrag: (a, k, fragments) for c items of b bits in 32-bit registers."""
    a = 32 // c
    k = 1 << (a.bit_length() - 1)
    return a, k, -(-b // k)


def exclusive_scan(xs, op, identity):
    out, acc = [], identity
    for x in xs:
        out.append(acc)
        acc = op(acc, x)
    return out


def inclusive_scan(xs, op, identity):
    out, acc = [], identity
    for x in xs:
        acc = op(acc, x)
        out.append(acc)
    return out


def compose(a, b):
    """(a∘b)_i = b_{a_i}: apply a's chunk first, then b's."""
    return [b[ai] for ai in a]


def identity_vector(S: int):
    return list(range(S))


def combine_offset(a, b):
    """⊕ of P:408-414 on (kind, value) with kind in {"abs", "rel"}."""
    return b if b[0] == "abs" else (a[0], a[1] + b[1])


def tau(transition, group_of_byte, chunk: bytes):
    """State-transition vector of a chunk: one DFA instance per start state.

    ``transition[g][s]`` is the row-per-group table of P:728.
    """
    S = len(transition[0])
    vec = []
    for s0 in range(S):
        s = s0
        for b in chunk:
            s = transition[group_of_byte[b]][s]
        vec.append(s)
    return vec


def chunk_column_offset(kinds):
    """Column offset a chunk hands to its successor (prose reading R8).

    ``kinds``: per-byte emission kinds (0 DATA, 1 CTRL, 2 FIELD, 3 RECORD).  abs(#field
    delimiters strictly after the last record delimiter) if the chunk holds a record
    delimiter, else rel(#field delimiters).  Record delimiters are field delimiters too.
    """
    last_rec = None
    for i, k in enumerate(kinds):
        if k == 3:
            last_rec = i
    if last_rec is None:
        return ("rel", sum(1 for k in kinds if k in (2, 3)))
    return ("abs", sum(1 for k in kinds[last_rec + 1:] if k in (2, 3)))
