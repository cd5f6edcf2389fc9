"""Summarise every kernel launch of an ncu --set full report (raw page) as a compact table.
usage: python scripts/ncu_multi.py <report.ncu-rep> <input_bytes> [alg_bytes_of_k_emit] [label]"""
import csv
import io
import subprocess
import sys

M = {
    "gpu__time_duration.sum": "ms",
    "dram__bytes_read.sum": "dram_rd",
    "dram__bytes_write.sum": "dram_wr",
    "smsp__inst_executed.sum": "warp_instr",
    "sm__inst_executed.avg.per_cycle_active": "ipc",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue%",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occ%",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "alu%",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma%",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "lsu%",
    "smsp__thread_inst_executed_per_inst_executed.ratio": "thr/inst",
    "launch__registers_per_thread": "regs",
    "sm__cycles_active.avg": "cycles",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0,
         "second": 1e3}


def main():
    rep, n = sys.argv[1], float(sys.argv[2])
    alg = float(sys.argv[3]) if len(sys.argv) > 3 else None
    label = sys.argv[4] if len(sys.argv) > 4 else rep
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    print(f"# {label}: input {n:.4e} B" + (f", k_emit algorithmic bytes {alg:.4e}" if alg else ""))
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        name = d.get("Kernel Name", "?").split("(")[0].replace("void ", "")
        g = {}
        for k, short in M.items():
            if k in hdr:
                u = units[hdr.index(k)]
                g[short] = float(d[k].replace(",", "")) * (SCALE.get(u, 1) if short in ("ms", "dram_rd", "dram_wr") else 1)
        tot = g["dram_rd"] + g["dram_wr"]
        line = (f"{name:28s} {g['ms']:8.3f} ms  dram {tot / 1e9:6.2f} GB ({tot / n:5.2f} B/in-B, {tot / g['ms'] / 1e6:6.0f} GB/s)"
                f"  in {n / g['ms'] / 1e6:6.0f} GB/s  warp-instr/B {g['warp_instr'] / n:5.3f}  ipc {g['ipc']:4.2f}"
                f"  issue {g['issue%']:4.1f}%  alu {g.get('alu%', 0):4.1f}%  fma {g.get('fma%', 0):4.1f}%"
                f"  lsu {g.get('lsu%', 0):4.1f}%  occ {g['occ%']:4.1f}%  thr {g['thr/inst']:4.1f}  regs {g['regs']:.0f}")
        if alg and "k_emit" in name:
            line += f"  traffic/alg {tot / alg:5.3f}"
        print(line)


if __name__ == "__main__":
    main()
