"""Compact per-launch summary of an ncu --set full report (the metrics the round reports quote):
time, DRAM bytes, tensor-pipe activity, L2 and DRAM throughput, grid size, registers.

usage: python tools/ncu_full_summary.py REPORT.ncu-rep OUT.csv [kernel-regex]
"""
import csv
import io
import re
import subprocess
import sys

COLS = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__grid_size", "launch__registers_per_thread"]


def main():
    rep, out = sys.argv[1], sys.argv[2]
    pat = re.compile(sys.argv[3] if len(sys.argv) > 3 else ".")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    idx = [hdr.index(c) if c in hdr else None for c in COLS]
    with open(out, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(COLS)
        w.writerow([units[i] if i is not None else "" for i in idx])
        for r in rows[2:]:
            if not pat.search(r[hdr.index("Kernel Name")]):
                continue
            w.writerow([(r[i][:40] if c == "Kernel Name" else r[i]) if i is not None else "" for c, i in zip(COLS, idx)])


if __name__ == "__main__":
    main()
