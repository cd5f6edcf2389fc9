"""Summarise `ncu --page raw --csv` exports (one or more launches per file) as a compact table.
usage: python scripts/raw_summary.py <raw.csv>... (input bytes per launch from the launch's own DRAM/time
is not known here: the table reports per-launch absolute values and per-input-byte figures when the file
name carries the workload and `--bytes N` is given)"""
import csv
import sys

M = [("gpu__time_duration.sum", "time"), ("dram__bytes_read.sum", "dram_rd"), ("dram__bytes_write.sum", "dram_wr"),
     ("smsp__inst_executed.sum", "warp_instr"), ("sm__inst_executed.avg.per_cycle_active", "ipc"),
     ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
     ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
     ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "alu%"),
     ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma%"),
     ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu%"),
     ("smsp__thread_inst_executed_per_inst_executed.ratio", "thr/inst"),
     ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem_conf"),
     ("lts__t_sector_hit_rate.pct", "l2hit%"),
     ("launch__registers_per_thread", "regs")]


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    for f in args:
        rows = list(csv.reader(open(f)))
        if len(rows) < 3:
            print(f, "empty"); continue
        hdr, units = rows[0], rows[1]
        for r in rows[2:]:
            name = r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
            out = []
            for m, lab in M:
                if m not in hdr:
                    continue
                i = hdr.index(m)
                out.append(f"{lab}={r[i]}{units[i] if lab in ('time', 'dram_rd', 'dram_wr') else ''}")
            print(f.split("/")[-1], name.split("(")[0][:40], " ".join(out))


if __name__ == "__main__":
    main()
