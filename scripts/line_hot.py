"""Per-source-line instruction count, active threads and stall share (ncu SASS csv + nvdisasm -g)."""
import csv, re, sys
from collections import defaultdict
sass_csv, disasm, kern = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
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
ex = defaultdict(float); th = defaultdict(float); st = defaultdict(float); te = ts = 0
for d in data:
    k = lines.get(int(d['Address'], 16) - base, ('?', 0))
    e = num(d['Instructions Executed']); s = num(d['Warp Stall Sampling (All Samples)'])
    ex[k] += e; th[k] += num(d['Thread Instructions Executed']); st[k] += s; te += e; ts += s
srcs = {}
def src(f, l):
    if f not in srcs:
        try: srcs[f] = open('/root/repo/paper_1905_13415_b200/csrc/' + f).read().split('\n')
        except Exception: srcs[f] = []
    return srcs[f][l - 1].strip()[:70] if 0 < l <= len(srcs[f]) else ''
print(f"{'line':28s} {'exec%':>6s} {'thr':>5s} {'stall%':>6s}  source")
for k in sorted(ex, key=lambda k: -(ex[k] / te + st[k] / ts))[:top]:
    print(f"{k[0][:18]+':'+str(k[1]):28s} {100*ex[k]/te:6.2f} {th[k]/max(ex[k],1):5.1f} {100*st[k]/ts:6.2f}  {src(*k)}")
