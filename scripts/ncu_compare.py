"""Side-by-side key metrics of the first kernel in several .ncu-rep files.
Usage: python scripts/ncu_compare.py a.ncu-rep b.ncu-rep ..."""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio",
        "smsp__pcsamp_warps_issue_stalled_long_scoreboard",
        "smsp__pcsamp_warps_issue_stalled_membar",
        "smsp__pcsamp_warps_issue_stalled_lg_throttle",
        "smsp__pcsamp_warps_issue_stalled_wait",
        "smsp__pcsamp_warps_issue_stalled_selected",
        "smsp__pcsamp_warps_issue_stalled_short_scoreboard",
        "smsp__pcsamp_warps_issue_stalled_sleeping",
        "smsp__pcsamp_sample_count"]


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, v = rows[0], rows[1], rows[2]
    return {k: (x, u) for k, u, x in zip(h, units, v)}, v[h.index("Kernel Name")]


if __name__ == "__main__":
    reps = [raw(p) for p in sys.argv[1:]]
    for p, (_, name) in zip(sys.argv[1:], reps):
        print(p, name[:90])
    for k in KEYS:
        vals = [r[0].get(k, ("-", ""))[0] for r in reps]
        unit = next((r[0][k][1] for r in reps if k in r[0]), "")
        print(f"{k:70s} {unit:8s} " + "  ".join(f"{x:>16s}" for x in vals))
