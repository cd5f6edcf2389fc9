"""k_emit instruction share by phase (E1a / E1b / E2 / conversion ...) from an ncu SASS csv + nvdisasm -g."""
import csv, re, sys
from collections import defaultdict
sass_csv, disasm = sys.argv[1], sys.argv[2]
rows = list(csv.reader(open(sass_csv))); hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr) and r[0] != 'Address']
num = lambda x: float(x.replace(',', '')) if x.strip() else 0.0
lines = {}; cur = None; infn = False
for ln in open(disasm):
    if '.text.' in ln: infn = '_ZN5parpa6k_emit' in ln
    if not infn: continue
    m = re.search(r'File "(.*?)", line (\d+)', ln)
    if m: cur = (m.group(1).split('/')[-1], int(m.group(2))); continue
    m = re.match(r'\s*/\*([0-9a-f]{4,})\*/', ln)
    if m and cur: lines[int(m.group(1), 16)] = cur
base = min(int(d['Address'], 16) for d in data)
src = open('/root/repo/paper_1905_13415_b200/csrc/parpa_kernels.cuh').read().split('\n')
def find(pat):
    for i, l in enumerate(src):
        if pat in l: return i + 1
    return 10 ** 9
marks = sorted([(find('__device__ __forceinline__ void write_value'), 'write_value'),
                (find('__device__ void emit_tile'), 'emit_tile head'), (find('// ---- E1a'), 'E1a'),
                (find('// ---- E1b'), 'E1b'), (find('// ---- E2 ----'), 'E2'),
                (find('__global__ void __launch_bounds__(EMIT_WARPS'), 'k_emit loop'),
                (find('// ---- finalize'), 'after')])
agg = defaultdict(float); tot = 0; st = defaultdict(float); sttot = 0
for d in data:
    f, l = lines.get(int(d['Address'], 16) - base, ('?', 0))
    e = num(d['Instructions Executed']); s = num(d['Warp Stall Sampling (All Samples)']); tot += e; sttot += s
    if f == 'parpa_kernels.cuh':
        ph = 'other kernels.cuh'
        for ln0, name in marks:
            if l >= ln0: ph = name
    else:
        ph = f
    agg[ph] += e; st[ph] += s
for k, v in sorted(agg.items(), key=lambda kv: -kv[1]):
    print(f"{k:28s} exec {100 * v / tot:6.2f}%  stall {100 * st[k] / sttot:6.2f}%")
