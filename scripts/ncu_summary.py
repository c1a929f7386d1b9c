#!/usr/bin/env python
"""Summarise an ncu --set full report: per kernel time, DRAM bytes, throughput, occupancy,
top stall reasons.  Usage: python scripts/ncu_summary.py report.ncu-rep [...]"""
import csv
import io
import subprocess
import sys

KEYS = [("gpu__time_duration.sum", "time"), ("dram__bytes_read.sum", "dram_rd"),
        ("dram__bytes_write.sum", "dram_wr"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_%"),
        ("launch__registers_per_thread", "regs"), ("launch__grid_size", "grid"),
        ("lts__t_sector_hit_rate.pct", "l2_hit_%"), ("l1tex__t_sector_hit_rate.pct", "l1_hit_%")]


def main():
    for rep in sys.argv[1:]:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        hdr, units = rows[0], rows[1]
        print(f"== {rep}")
        for r in rows[2:]:
            d = dict(zip(hdr, r))
            u = dict(zip(hdr, units))
            name = d["Kernel Name"].split("(")[0]
            parts = []
            for k, short in KEYS:
                if k in d:
                    parts.append(f"{short}={d[k]}{u.get(k, '')}")
            stalls = []
            for h, v in d.items():
                if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                    try:
                        stalls.append((float(v), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                    except ValueError:
                        pass
            stalls.sort(reverse=True)
            print(f"  {name}: " + " ".join(parts))
            print("     stalls/issue: " + ", ".join(f"{n} {v:.2f}" for v, n in stalls[:5]))


if __name__ == "__main__":
    main()
