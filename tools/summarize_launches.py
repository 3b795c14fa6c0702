"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per
kernel: launches and median duration (serialized, cold-cache).

  python tools/summarize_launches.py launches.csv "<command it came from>" > out.txt"""
import csv
import statistics
import sys
from collections import OrderedDict


def main(path, cmd=""):
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hdr_i]
    kn, mv, unit, bs = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit"), hdr.index("Block Size")
    per = OrderedDict()
    for r in rows[hdr_i + 1:]:
        if len(r) <= mv or not r[mv]:
            continue
        v = float(r[mv].replace(",", ""))
        v *= {"nsecond": 1e-3, "ns": 1e-3, "msecond": 1e3, "ms": 1e3}.get(r[unit], 1.0)
        per.setdefault((r[kn][:60], r[bs]), []).append(v)
    if cmd:
        print(f"ncu --metrics gpu__time_duration.sum --clock-control none: {cmd}")
        print("(serialized, cold-cache per-launch durations)\n")
    for (name, block), ts in per.items():
        print(f"{name:60s} {block:12s} launches={len(ts):4d} median_us={statistics.median(ts):9.1f}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
