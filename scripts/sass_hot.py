"""Summarise an ncu --page source --print-source=sass CSV: hottest instructions and opcode mix."""
import csv
import sys
from collections import Counter, defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr) and r[0] != 'Address']


def num(x):
    try:
        return float(x.replace(",", ""))
    except Exception:
        return 0.0


tot_s = sum(num(d["Warp Stall Sampling (All Samples)"]) for d in data)
tot_i = sum(num(d["Instructions Executed"]) for d in data)
print(f"instructions {len(data)}  samples {tot_s:.0f}  warp-instr executed {tot_i:.3e}")
op_i, op_s = Counter(), Counter()
for d in data:
    op = d["Source"].split()[0] if d["Source"].split() else "?"
    if op.startswith("@"):
        op = d["Source"].split()[1]
    op = op.split(".")[0]
    op_i[op] += num(d["Instructions Executed"])
    op_s[op] += num(d["Warp Stall Sampling (All Samples)"])
print("opcode mix (exec %, stall %):")
for op, v in op_i.most_common(25):
    print(f"  {op:10s} {100*v/tot_i:6.2f}%  {100*op_s[op]/tot_s:6.2f}%")
stall_cols = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
agg = Counter()
for d in data:
    for c in stall_cols:
        agg[c] += num(d[c])
print("stall reasons:", ", ".join(f"{k[6:]}={100*v/tot_s:.1f}%" for k, v in agg.most_common(8)))
top = sorted(data, key=lambda d: -num(d["Warp Stall Sampling (All Samples)"]))[:int(sys.argv[2]) if len(sys.argv) > 2 else 30]
for d in top:
    print(f"{d['Address']:>6} {100*num(d['Warp Stall Sampling (All Samples)'])/tot_s:5.2f}% exec={num(d['Instructions Executed']):.2e} thr={d['Avg. Threads Executed']:>6} {d['Source'][:70]}")
