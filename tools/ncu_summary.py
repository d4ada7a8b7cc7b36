"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel:
launches, total / mean device time and share.  Times are cold-cache and
serialised (ncu), so compare SHARES, not absolutes.

usage: python tools/ncu_summary.py gpurun_out/launches.csv [steps]
"""
import csv
import re
import sys
from collections import defaultdict


def short(name):
    name = re.sub(r"\(.*", "", name)
    name = name.replace("hexconv::", "")
    return name


def main():
    path = sys.argv[1]
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        unit = r.get("Metric Unit", "")
        v = float(r["Metric Value"].replace(",", ""))
        if v != v:  # nan: a launch ncu could not time (e.g. cut off at process exit)
            continue
        scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "s": 1e6, "second": 1e6}.get(unit, 1.0)
        rows.append((short(r["Kernel Name"]), v * scale))
    agg = defaultdict(lambda: [0, 0.0])
    for k, us in rows:
        agg[k][0] += 1
        agg[k][1] += us
    total = sum(v[1] for v in agg.values())
    print(f"{'kernel':60s} {'launches':>8s} {'per step':>9s} {'total us':>10s} {'mean us':>9s} {'share':>7s}")
    for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k[:60]:60s} {n:8d} {n / steps:9.1f} {us:10.1f} {us / n:9.1f} {us / total * 100:6.1f}%")
    print(f"{'total':60s} {len(rows):8d} {len(rows) / steps:9.1f} {total:10.1f}")


if __name__ == "__main__":
    main()
