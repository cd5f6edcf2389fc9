"""Per-source-line hot spots of one kernel in an ncu report (needs -lineinfo + --import-source).

usage: python scripts/src_hot.py <report.ncu-rep> <kernel-regex> [top]
Prints, per CUDA source line, warp-instructions executed, thread-instructions, stall samples, and the
share of the kernel's instructions, sorted by instructions."""
import csv, io, subprocess, sys, collections, os

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", "regex:" + kre],
                     capture_output=True, text=True).stdout
fname = None
agg = collections.defaultdict(lambda: [0, 0, 0, ""])
hdr = None
for row in csv.reader(io.StringIO(out)):
    if not row:
        continue
    if row[0] == "File Path":
        fname = os.path.basename(row[1]); continue
    if row[0] == "Line No":
        hdr = row; continue
    if row[0] in ("Function Name",) or hdr is None:
        continue
    if row[0] != "":                      # a CUDA line with aggregated metrics
        try:
            ins = int(row[hdr.index("Instructions Executed")].replace(",", "") or 0)
            thr = int(row[hdr.index("Thread Instructions Executed")].replace(",", "") or 0)
            smp = int(row[hdr.index("Warp Stall Sampling (All Samples)")].replace(",", "") or 0)
        except ValueError:
            continue
        k = (fname, int(row[0]))
        a = agg[k]; a[0] += ins; a[1] += thr; a[2] += smp; a[3] = row[1].strip()[:70]
tot_i = sum(v[0] for v in agg.values()) or 1
tot_s = sum(v[2] for v in agg.values()) or 1
print(f"total warp-instr {tot_i:.4e}  samples {tot_s}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{k[0]:>20s}:{k[1]:<5d} {v[0]:>12d} {100*v[0]/tot_i:5.1f}%  thr/w {v[1]/max(v[0],1):5.1f}  stall {100*v[2]/tot_s:5.1f}%  {v[3]}")
