"""Skewed input (the paper's E4, fig:tagskew right: one 200 MB record): yelp-shaped input with
one record whose text field is SKEW bytes of quoted text (commas, newlines, "" escapes), against the same
input without it.  Checks: one more record; the giant field's span is exactly the constructed one; every
other row equals the plain parse's row (offsets after the insertion shifted by the inserted bytes).
usage: python scripts/skew_probe.py [base_bytes] [skew_bytes]"""
import json
import statistics
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

import datagen
import paper_1905_13415_b200 as parpa

base_n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 2e9
skew = int(float(sys.argv[2])) if len(sys.argv) > 2 else 200e6
w = datagen.WORKLOADS["yelp"]
data, g = datagen.generate("yelp", base_n)
R0 = g.records
cut_rec = R0 // 2
# byte offset of record cut_rec: parse once and take column 0's first DATA byte - 1 (the opening quote)
dfa = parpa.Dfa.dialect("csv")
schema = parpa.Schema(list(w.types))


def parse_timed(buf):
    d = torch.from_numpy(buf).cuda()
    res = parpa.parse(dfa, schema, d)
    cap = res.records + 1
    cols = parpa.alloc_columns(schema, cap)
    st = parpa.new_stats_tensor()
    for _ in range(2):
        parpa.parse_into(dfa, schema, d, cols, cap, st)
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        parpa.parse_into(dfa, schema, d, cols, cap, st)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    s = parpa.stats_from_tensor(st)
    assert s["status"] == 0, s
    out = [(c.offset[:s["records"]].cpu().numpy().view(np.uint64), c.length[:s["records"]].cpu().numpy().view(np.uint32),
            None if c.value is None else c.value[:s["records"]].cpu().numpy().view(np.int64)) for c in cols]
    return s["records"], statistics.median(ts), out


R_plain, ms_plain, cols_plain = parse_timed(data)
assert R_plain == R0
pos = int(cols_plain[0][0][cut_rec]) - 1                       # the opening quote of record cut_rec
rng = np.random.default_rng(9)
words = rng.integers(ord("a"), ord("z") + 1, size=skew, dtype=np.uint8)
words[rng.random(skew) < 0.15] = ord(" ")
words[rng.random(skew) < 0.01] = ord(",")
words[rng.random(skew) < 0.002] = ord("\n")
text = words.tobytes().replace(b"q", b'""')[:skew]             # "" escapes (CTRL + DATA inside the span)
trail = len(text) - len(text.rstrip(b'"'))
if trail % 2:                                                  # truncation split a "" pair
    text = text[:-1]
prefix = b'"skewskewskewskewskew00","u","b","5","0","0","0","'
rec = prefix + text + b'","2020-01-01 00:00:00"\n'
ins = np.frombuffer(rec, np.uint8)
skewed = np.concatenate([data[:pos], ins, data[pos:]])
R_skew, ms_skew, cols_skew = parse_timed(skewed)
assert R_skew == R0 + 1, (R_skew, R0)
# the giant record is row cut_rec: its text field (column 7) spans the constructed bytes
t_off, t_len = int(cols_skew[7][0][cut_rec]), int(cols_skew[7][1][cut_rec])
exp_off = pos + len(prefix)
exp_len = len(text)
assert (t_off, t_len) == (exp_off, exp_len), ((t_off, t_len), (exp_off, exp_len))
for c in range(w.C):                                           # every other row is the plain parse's row
    o_p, l_p, v_p = cols_plain[c]
    o_s, l_s, v_s = cols_skew[c]
    assert np.array_equal(o_s[:cut_rec], o_p[:cut_rec]) and np.array_equal(l_s[:cut_rec], l_p[:cut_rec])
    assert np.array_equal(o_s[cut_rec + 1:], o_p[cut_rec:] + np.uint64(len(rec))), c
    assert np.array_equal(l_s[cut_rec + 1:], l_p[cut_rec:]), c
    if v_p is not None:
        assert np.array_equal(v_s[:cut_rec], v_p[:cut_rec]) and np.array_equal(v_s[cut_rec + 1:], v_p[cut_rec:]), c
print(json.dumps({"experiment": "E4 skewed input (one giant record)", "base_bytes": int(data.size), "records": R0,
                  "skew_record_bytes": len(rec), "plain_ms": round(ms_plain, 3), "plain_GBps": round(data.size / ms_plain / 1e6, 1),
                  "skewed_ms": round(ms_skew, 3), "skewed_GBps": round(skewed.size / ms_skew / 1e6, 1),
                  "checks": "R+1, giant span exact, all other rows equal (shifted)"}))
