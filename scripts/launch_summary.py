#!/usr/bin/env python
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): per kernel the
launch count, total and mean time, and share of all kernel time.
Usage: python scripts/launch_summary.py launches.csv"""
import collections
import csv
import sys


def main(path):
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0].strip()
        t = float(r["Metric Value"]) * (1e-3 if r["Metric Unit"] == "ns" else 1.0)
        tot[name] += t
        cnt[name] += 1
    allt = sum(tot.values())
    print(f"{'kernel':60s} {'launches':>8s} {'total_us':>12s} {'mean_us':>10s} {'share':>6s}")
    for k in sorted(tot, key=tot.get, reverse=True):
        print(f"{k[:60]:60s} {cnt[k]:8d} {tot[k]:12.1f} {tot[k] / cnt[k]:10.2f} "
              f"{tot[k] / allt:6.1%}")
    print(f"{'TOTAL':60s} {sum(cnt.values()):8d} {allt:12.1f}")


if __name__ == "__main__":
    main(sys.argv[1])
