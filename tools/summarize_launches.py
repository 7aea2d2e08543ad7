"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel:
launches, total and mean device time, share. Usage: summarize_launches.py launches.csv"""
import csv
import re
import sys
from collections import defaultdict


def short(name):
    name = re.sub(r"\(.*$", "", name)
    name = name.replace("pcr::<unnamed>::", "").replace("pcr::", "")
    return name


def main(path):
    tot = defaultdict(float)
    cnt = defaultdict(int)
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for row in csv.DictReader(lines):
        if row.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = short(row["Kernel Name"])
        v = float(row["Metric Value"].replace(",", ""))
        unit = row.get("Metric Unit", "ns")
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}.get(unit, 1e-6)
        tot[k] += v * scale
        cnt[k] += 1
    grand = sum(tot.values())
    print(f"{'kernel':32s} {'launches':>9s} {'total ms':>11s} {'mean us':>10s} {'share':>7s}")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"{k:32s} {cnt[k]:9d} {v:11.3f} {1e3 * v / cnt[k]:10.2f} {100 * v / grand:6.2f}%")
    print(f"{'TOTAL':32s} {sum(cnt.values()):9d} {grand:11.3f}")


if __name__ == "__main__":
    main(sys.argv[1])
