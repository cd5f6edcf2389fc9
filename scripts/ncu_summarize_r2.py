"""Per-kernel summaries of the round-2 final ncu captures (gpurun_out/final/raw_<workload>_<kernel>.csv) into
profiles/r02_ncu_kernels.jsonl and the emission kernel's DRAM bytes per input byte into profiles/ncu_traffic.json.
Input bytes per capture = its record count x the workload's bytes per record in the bench line."""
import csv
import json
import sys

B = {"yelp": (1_000_000, 4824048489 / 6645853, "k_emit_sparse"), "taxi": (8_000_000, 4797042681 / 48900000, "k_emit"),
     "clf": (8_000_000, 7547654818 / 78000000, "k_emit")}
SC = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "ms": 1.0, "nsecond": 1e-6,
      "usecond": 1e-3, "msecond": 1.0}
src = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/final"
out = []
traffic = {"_note": "emission-kernel DRAM bytes per input byte, (dram__bytes_read.sum + dram__bytes_write.sum) / input "
                    "bytes from one ncu --set full capture of bench.py per workload at reduced record counts "
                    "(profiles/r02_ncu_kernels.jsonl); bench.py scales it to the launch"}
for wl, (recs, bpr, ke) in B.items():
    nin = recs * bpr
    for k in ["k_pass1", "k_pass2", ke]:
        rows = list(csv.reader(open(f"{src}/raw_{wl}_{k}.csv")))
        h, u, r = rows[0], rows[1], rows[2]

        def g(m):
            i = h.index(m)
            return float(r[i].replace(",", "")) * SC.get(u[i], 1)
        t = g("gpu__time_duration.sum")
        rd, wr = g("dram__bytes_read.sum"), g("dram__bytes_write.sum")
        d = dict(workload=wl, kernel=k, records=recs, input_bytes=int(nin), ms_under_ncu=round(t, 4),
                 dram_B_per_B=round((rd + wr) / nin, 3), warp_instr_per_B=round(g("smsp__inst_executed.sum") / nin, 4),
                 ipc=round(g("sm__inst_executed.avg.per_cycle_active"), 2),
                 issue_pct=round(g("smsp__issue_active.avg.pct_of_peak_sustained_active"), 1),
                 alu_pct=round(g("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"), 1),
                 fma_pct=round(g("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"), 1),
                 lsu_pct=round(g("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"), 1),
                 thr_per_instr=round(g("smsp__thread_inst_executed_per_inst_executed.ratio"), 1),
                 dram_GBps=round((rd + wr) / t / 1e6, 1))
        out.append(d)
        if k == ke:
            traffic[wl] = {"kernel": ke, "dram_bytes_per_input_byte": d["dram_B_per_B"],
                           "source": "profiles/r02_ncu_kernels.jsonl"}
with open("profiles/r02_ncu_kernels.jsonl", "w") as f:
    for d in out:
        f.write(json.dumps(d) + "\n")
with open("profiles/ncu_traffic.json", "w") as f:
    json.dump(traffic, f, indent=1)
print(f"{'wl':5s} {'kernel':14s} {'B/B':>6s} {'wi/B':>6s} {'ipc':>5s} {'iss%':>5s} {'alu%':>5s} {'fma%':>5s} {'thr':>5s} {'GB/s':>7s}")
for d in out:
    print(f"{d['workload']:5s} {d['kernel']:14s} {d['dram_B_per_B']:6.3f} {d['warp_instr_per_B']:6.3f} {d['ipc']:5.2f} "
          f"{d['issue_pct']:5.1f} {d['alu_pct']:5.1f} {d['fma_pct']:5.1f} {d['thr_per_instr']:5.1f} {d['dram_GBps']:7.1f}")
