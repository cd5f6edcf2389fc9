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


def adversarial_plain(seed, nrows=40000):
    """CSV without control bytes: 8 columns (int / float / span), 90% complete records, the rest short or
    long; 8% empty fields; numbers of 1-20 characters (signs, '.' anywhere in floats); ~0.15% of records with
    one unquoted giant field of 3-70 KB (digits in typed columns, letters in spans)."""
    import random
    rng = random.Random(seed)
    types = [oracle.INT64, oracle.FLOAT64, oracle.SPAN, oracle.INT64, oracle.FLOAT64, oracle.SPAN, oracle.INT64,
             oracle.FLOAT64]
    C = len(types)

    def num(t):
        L = rng.choice([1, 1, 2, 3, 4, 5, 6, 7, 8, 9, 12, 16, 20])
        s = rng.choice(["", "", "-", "+"]) + "".join(rng.choice("0123456789") for _ in range(L))
        if t == oracle.FLOAT64 and rng.random() < 0.6:
            q = rng.randint(0, len(s))
            s = s[:q] + "." + s[q:]
        return s

    rows = []
    for _ in range(nrows):
        n = C if rng.random() < 0.9 else rng.choice([1, 3, C - 1, C + 1, C + 3])
        fs = []
        for c in range(n):
            t = types[c % C]
            if rng.random() < 0.08:
                fs.append("")
            elif t == oracle.SPAN:
                fs.append("".join(rng.choice("abcxyz XYZ-:.") for _ in range(rng.randint(0, 12))))
            else:
                fs.append(num(t))
        if rng.random() < 0.0015:
            c = rng.randrange(len(fs))
            big = rng.randint(3000, 70000)
            fs[c] = "".join(rng.choice("0123456789") for _ in range(big)) if types[c % C] != oracle.SPAN else "g" * big
        rows.append(",".join(fs))
    return ("\n".join(rows) + ("\n" if seed % 2 else "")).encode(), types


def adversarial_clf(seed, nlines=30000):
    """Common-Log-Format-like lines (reading R20): space-delimited tokens, [..] and "..." enclosed fields with
    spaces, \\" and \\\\ escapes inside quotes, '#' directive lines (with quotes and brackets) and '#' inside
    tokens, ragged token counts, typed columns holding long numbers, '-', empties and quoted numbers."""
    import random
    rng = random.Random(seed)
    types = [oracle.SPAN, oracle.SPAN, oracle.SPAN, oracle.SPAN, oracle.SPAN, oracle.INT64, oracle.INT64]
    lines = []
    for _ in range(nlines):
        if rng.random() < 0.01:
            lines.append("#" + "".join(rng.choice('ab "[]x #') for _ in range(rng.randint(0, 30))))
            continue
        n = 7 if rng.random() < 0.9 else rng.choice([1, 2, 5, 8, 9])
        fs = []
        for c in range(n):
            k = rng.random()
            if c == 3 or (c > 6 and k < 0.3):
                fs.append("[" + "".join(rng.choice("0123456789/:+- abc") for _ in range(rng.randint(0, 26))) + "]")
            elif c == 4 or (c > 6 and k < 0.6):
                body = ""
                for _ in range(rng.randint(0, 30)):
                    r = rng.random()
                    body += '\\"' if r < 0.05 else "\\\\" if r < 0.08 else rng.choice("GET /a?b=1 HTTP/1.0#")
                fs.append('"' + body + '"')
            elif c in (5, 6):
                fs.append(rng.choice(["-", "", str(rng.randint(0, 999)), str(rng.randint(0, 10 ** 12)),
                                      "".join(rng.choice("0123456789") for _ in range(rng.randint(15, 25))),
                                      '"' + str(rng.randint(0, 99)) + '"']))
            else:
                fs.append("".join(rng.choice("0123456789.-abc#") for _ in range(rng.randint(1, 15))))
        lines.append(" ".join(fs))
    return ("\n".join(lines) + "\n").encode(), types
