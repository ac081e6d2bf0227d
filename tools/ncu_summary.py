#!/usr/bin/env python
"""Key metrics of one ncu --set full capture, in the profiles/*_full.txt format.

    python tools/ncu_summary.py REPORT.ncu-rep "title line" "command line" > profiles/X_full.txt
"""
import csv
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "launch__grid_size", "launch__block_size",
    "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers", "smsp__inst_executed.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__cycles_elapsed.avg.per_second",
]


def main():
    rep, title, cmd = sys.argv[1], sys.argv[2], sys.argv[3]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], dict(zip(rows[0], rows[1]))
    for row in rows[2:]:
        d = dict(zip(hdr, row))
        print(f"# {title}")
        print(f"# command: {cmd}")
        print(f"{'Kernel Name':70} {d['Kernel Name']}")
        for k in KEYS:
            if k in d:
                print(f"{k:70} {d[k]} {units.get(k, '')}")
        print("# top stall reasons (warps per issue-active cycle)")
        st = [(k, float(d[k].replace(",", ""))) for k in hdr
              if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")
              and d[k] not in ("", "n/a")]
        for k, v in sorted(st, key=lambda x: -x[1])[:8]:
            print(f"{k:70} {v:.3f}")


if __name__ == "__main__":
    main()
