"""Summarise an ncu --set full report (one kernel launch) into the numbers DESIGN.md / bench.py use.

usage: python scripts/ncu_summary.py <report.ncu-rep> [input_bytes] [alg_bytes]
Prints a compact text block (duration, DRAM bytes, throughputs, issue, occupancy, stall mix) and,
when input/alg bytes are given, bytes-per-input-byte and the algorithmic vs actual traffic ratio.
"""
import csv
import io
import subprocess
import sys

WANT = {
    "Duration": "duration",
    "DRAM Throughput": "dram_pct",
    "Memory Throughput": "mem_pct",
    "L2 Cache Throughput": "l2_pct",
    "Compute (SM) Throughput": "sm_pct",
    "Executed Ipc Active": "ipc",
    "Issue Slots Busy": "issue_pct",
    "Achieved Occupancy": "occupancy_pct",
    "Registers Per Thread": "regs",
    "Avg. Active Threads Per Warp": "active_threads",
    "Executed Instructions": "instructions",
    "L1/TEX Hit Rate": "l1_hit",
    "L2 Hit Rate": "l2_hit",
    "Block Size": "block",
    "Grid Size": "grid",
}


def details(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    res = {}
    kernel = None
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        kernel = d.get("Kernel Name", kernel)
        name = d.get("Metric Name")
        if name in WANT and WANT[name] not in res:
            res[WANT[name]] = (d.get("Metric Value"), d.get("Metric Unit"))
    return kernel, res


def raw(rep, metrics):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    res = {}
    for m in metrics:
        if m in hdr:
            i = hdr.index(m)
            res[m] = (vals[i], units[i])
    return res


def num(v):
    return float(str(v).replace(",", ""))


def main():
    rep = sys.argv[1]
    kernel, d = details(rep)
    r = raw(rep, ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
                  "smsp__inst_executed.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed"])
    print(f"kernel: {kernel}")
    for k, (v, u) in d.items():
        print(f"  {k:16s} {v} {u}")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rb = num(r["dram__bytes_read.sum"][0]) * scale.get(r["dram__bytes_read.sum"][1], 1)
    wb = num(r["dram__bytes_write.sum"][0]) * scale.get(r["dram__bytes_write.sum"][1], 1)
    tu = r["gpu__time_duration.sum"][1]
    t = num(r["gpu__time_duration.sum"][0]) * {"nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6,
                                                "msecond": 1e-3, "ms": 1e-3, "s": 1.0}.get(tu, 1e-9)
    print(f"  dram_read_bytes  {rb:.4e}\n  dram_write_bytes {wb:.4e}\n  dram_total_bytes {rb + wb:.4e}")
    print(f"  dram_gbs         {(rb + wb) / t / 1e9:.1f}")
    if len(sys.argv) > 2:
        n = float(sys.argv[2])
        print(f"  input_gbs        {n / t / 1e9:.1f}")
        print(f"  dram_bytes_per_input_byte {(rb + wb) / n:.3f}")
        ins = num(r["smsp__inst_executed.sum"][0])
        print(f"  warp_instr_per_input_byte {ins / n:.3f}")
    if len(sys.argv) > 3:
        alg = float(sys.argv[3])
        print(f"  algorithmic_bytes {alg:.4e}  traffic/alg {(rb + wb) / alg:.3f}")


if __name__ == "__main__":
    main()
