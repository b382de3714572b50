#!/usr/bin/env python
"""Summarise an ncu --set full report (raw page) per kernel: time, DRAM bytes/throughput, pipes,
issue activity and the top warp-stall reasons. Usage: ncu_summary.py REPORT.ncu-rep"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma_type_fp16.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__inst_executed.sum", "sm__cycles_elapsed.avg", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        print(f"== {name}")
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"   {k:70s} {r[i]} {units[i]}")
        st = [(float(r[i]), h.replace("smsp__pcsamp_warps_issue_stalled_", ""))
              for i, h in enumerate(hdr) if h.startswith("smsp__pcsamp_warps_issue_stalled_")
              and not h.endswith("not_issued") and r[i] not in ("", "n/a")]
        tot = sum(v for v, _ in st) or 1
        print("   stalls:", ", ".join(f"{n} {100 * v / tot:.0f}%" for v, n in sorted(st, reverse=True)[:7]))


if __name__ == "__main__":
    main(sys.argv[1])
