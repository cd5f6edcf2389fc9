"""Attribute ncu per-instruction metrics (SASS csv) to CUDA source lines via nvdisasm -g line info.
usage: sass_lines.py <ncu_sass.csv> <nvdisasm -g output> <mangled kernel name> [topN]"""
import csv
import re
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
num = lambda x: float(x.replace(",", "")) if x.strip() else 0.0
lines = {}
cur = None
infn = False
for ln in open(sys.argv[2]):
    if ln.startswith(".text.") or "--- .text." in ln:
        infn = sys.argv[3] in ln
    if not infn:
        continue
    m = re.search(r'File "(.*?)", line (\d+)', ln)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
    if m and cur:
        lines[int(m.group(1), 16)] = cur
base = min(int(d["Address"], 16) for d in data)
ex, st = Counter(), Counter()
te = ts = 0
for d in data:
    off = int(d["Address"], 16) - base
    key = lines.get(off, ("?", 0))
    e, s = num(d["Instructions Executed"]), num(d["Warp Stall Sampling (All Samples)"])
    ex[key] += e
    st[key] += s
    te += e
    ts += s
src = {}
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
print(f"{'file:line':34s} {'exec%':>7s} {'stall%':>7s}")
for key, v in sorted(ex.items(), key=lambda kv: -(kv[1] / te + st[kv[0]] / ts))[:top]:
    print(f"{key[0]+':'+str(key[1]):34s} {100*v/te:7.2f} {100*st[key]/ts:7.2f}")
