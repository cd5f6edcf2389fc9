"""Per-function / per-line instruction and stall breakdown of an ncu SASS source csv (k_scan<2>)."""
import csv, re, sys
from collections import Counter
sass_csv, disasm, kern = sys.argv[1], sys.argv[2], sys.argv[3]
rows = list(csv.reader(open(sass_csv))); hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr) and r[0] != 'Address']
num = lambda x: float(x.replace(',', '')) if x.strip() else 0.0
lines = {}; cur = None; infn = False
for ln in open(disasm):
    if '.text.' in ln: infn = kern in ln
    if not infn: continue
    m = re.search(r'File "(.*?)", line (\d+)', ln)
    if m: cur = (m.group(1).split('/')[-1], int(m.group(2))); continue
    m = re.match(r'\s*/\*([0-9a-f]{4,})\*/', ln)
    if m and cur: lines[int(m.group(1), 16)] = cur
base = min(int(d['Address'], 16) for d in data)
srcs = {}
def fn_of(f, l):
    if f not in srcs:
        try:
            srcs[f] = open('/root/repo/paper_1905_13415_b200/csrc/' + f).read().split('\n')
        except Exception:
            return f
    src = srcs[f]; i = min(l - 1, len(src) - 1)
    while i >= 0:
        m = re.match(r'(?:template <[^>]*>\s*)?(?:__device__|__global__)[^(]*?\b([a-zA-Z_0-9]+)\s*\(', src[i])
        if m: return f + ':' + m.group(1)
        i -= 1
    return f
ex = Counter(); st = Counter(); te = ts = 0
for d in data:
    k = lines.get(int(d['Address'], 16) - base, ('?', 0))
    e = num(d['Instructions Executed']); sm = num(d['Warp Stall Sampling (All Samples)'])
    fn = fn_of(*k); ex[fn] += e; st[fn] += sm; te += e; ts += sm
print(f"{'function':45s} {'exec%':>7s} {'stall%':>7s}")
for f, v in sorted(ex.items(), key=lambda kv: -(kv[1] / te + st[kv[0]] / ts))[:int(sys.argv[4]) if len(sys.argv) > 4 else 25]:
    print(f"{f:45s} {100*v/te:7.2f} {100*st[f]/ts:7.2f}")
