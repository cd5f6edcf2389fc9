"""Which source lines execute with few active threads (SIMT efficiency) — ncu SASS csv + nvdisasm -g."""
import csv, re, sys
from collections import Counter
sass_csv, disasm, kern = sys.argv[1], sys.argv[2], sys.argv[3]
lo, hi = float(sys.argv[4]), float(sys.argv[5])
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
c = Counter(); tot = 0
for d in data:
    e = num(d['Instructions Executed']); tot += e
    t = num(d['Avg. Threads Executed'])
    if lo <= t < hi: c[lines.get(int(d['Address'], 16) - base)] += e
for k, v in c.most_common(int(sys.argv[6]) if len(sys.argv) > 6 else 30):
    print(f"{100 * v / tot:6.2f}%  {k}")
