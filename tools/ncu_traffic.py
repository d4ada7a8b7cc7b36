"""Per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) of the
kernels in an ncu report, averaged over launches -> JSON for bench.py's
roofline.traffic.

usage: python tools/ncu_traffic.py REPORT.ncu-rep OUT.json [kernel-regex]
"""
import csv
import io
import json
import re
import subprocess
import sys


def main():
    rep, out = sys.argv[1], sys.argv[2]
    pat = re.compile(sys.argv[3] if len(sys.argv) > 3 else ".")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    col = {h: i for i, h in enumerate(hdr)}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    launches = []
    for r in rows[2:]:
        name = r[col["Kernel Name"]]
        if not pat.search(name):
            continue
        rd = float(r[col["dram__bytes_read.sum"]].replace(",", "")) * scale[units[col["dram__bytes_read.sum"]]]
        wr = float(r[col["dram__bytes_write.sum"]].replace(",", "")) * scale[units[col["dram__bytes_write.sum"]]]
        t = float(r[col["gpu__time_duration.sum"]].replace(",", ""))
        launches.append({"kernel": name[:80], "dram_read": rd, "dram_write": wr, "time": t,
                         "time_unit": units[col["gpu__time_duration.sum"]]})
    avg = sum(l["dram_read"] + l["dram_write"] for l in launches) / max(len(launches), 1)
    json.dump({"source": rep, "launches": len(launches), "bytes_per_launch": avg, "per_launch": launches},
              open(out, "w"), indent=1)
    print(f"{len(launches)} launches, {avg / 1e6:.1f} MB per launch")


if __name__ == "__main__":
    main()
