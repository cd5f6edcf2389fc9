"""Stall-sample breakdown per CUDA source line of one kernel in an ncu report.
usage: python scripts/stall_lines.py <report> <kernel-regex> [top]"""
import csv, io, subprocess, collections, os, sys
rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", "regex:" + kre],
                     capture_output=True, text=True).stdout
hdr = None; fname = None
agg = collections.defaultdict(collections.Counter); src = {}
for row in csv.reader(io.StringIO(out)):
    if not row: continue
    if row[0] == "File Path": fname = os.path.basename(row[1]); continue
    if row[0] == "Line No": hdr = row; continue
    if hdr is None or row[0] == "Function Name": continue
    if row[0] != "":
        k = (fname, int(row[0])); src[k] = row[1].strip()[:60]
        for i, h in enumerate(hdr):
            if h.startswith("stall_") and "Not Issued" not in h:
                try: agg[k][h] += int(row[i] or 0)
                except ValueError: pass
tot = sum(sum(c.values()) for c in agg.values()) or 1
allc = collections.Counter()
for c in agg.values(): allc.update(c)
print("total samples", tot, " overall:", ", ".join(f"{n[6:]}={100*v/tot:.1f}%" for n, v in allc.most_common(8)))
for k, c in sorted(agg.items(), key=lambda kv: -sum(kv[1].values()))[:top]:
    s = sum(c.values()); t3 = ", ".join(f"{n[6:]}={v}" for n, v in c.most_common(3))
    print(f"{k[0]}:{k[1]} {100*s/tot:5.1f}%  {t3}  | {src[k]}")
