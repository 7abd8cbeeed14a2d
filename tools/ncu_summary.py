"""Summarise an `ncu --page raw --csv` export into a markdown table (one row
per kernel launch): duration, DRAM bytes and rate, shared-memory wavefronts,
pipe utilisation, occupancy — the figures DESIGN.md and profiles/ quote.

    python tools/ncu_summary.py gpurun_out/p8_ncu_v4_raw.csv [--algo-bytes 536870912]
"""
import argparse
import csv

METRICS = [
    ("gpu__time_duration.sum", "us"),
    ("dram__bytes_read.sum", "MB rd"),
    ("dram__bytes_write.sum", "MB wr"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wf"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem wf %"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "bank confl"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--algo-bytes", type=float, default=None,
                    help="algorithmic bytes per launch -> GB/s column")
    a = ap.parse_args()
    rows = list(csv.reader(open(a.csv)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}
    keys = [(m, lbl) for m, lbl in METRICS if m in col]
    print("| kernel | " + " | ".join(lbl for _, lbl in keys) +
          (" | algo GB/s |" if a.algo_bytes else " |"))
    print("|---" * (len(keys) + 1 + (1 if a.algo_bytes else 0)) + "|")
    for r in data:
        name = r[col["Kernel Name"]].split("(")[0].split("::")[-1]
        vals = []
        for m, _ in keys:
            v = r[col[m]].replace(",", "")
            vals.append(v)
        line = f"| {name} | " + " | ".join(vals)
        if a.algo_bytes:
            us = float(r[col["gpu__time_duration.sum"]].replace(",", ""))
            line += f" | {a.algo_bytes / (us * 1e-6) / 1e9:.0f}"
        print(line + " |")


if __name__ == "__main__":
    main()
