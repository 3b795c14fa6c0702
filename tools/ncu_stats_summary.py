"""Summarise an ncu --csv metrics log (tools/gpu_r02bc.sh) of the statistics passes
into JSON: per kernel, the median duration, DRAM bytes, achieved GB/s against the
measured HBM peak (MEASURED_PEAKS.json) and the algorithmic bytes."""
import csv
import json
import statistics
import sys
from collections import defaultdict

ALG = {  # algorithmic bytes per launch at 4096^2 / 4096^3 (DESIGN: kernels and their rooflines)
    "bside_kernel<0": 4096 * 4096 * 2,            # B read once (BF16)
    "bside_kernel<2": 4096 * 4096 * 4 * 3,        # B read once + TF32 hi / lo written (FP32)
    "wide_apart_kernel": 4096 * 4096 * 4,          # A read once (FP32)
    "wide_combine_kernel": 4096 * 32 * 48 + 4096 * 32 * 8,  # partials + C-row partials read once
}


def main(path, out):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, mi, vi, ui = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    vals = defaultdict(lambda: defaultdict(list))
    for r in rows[1:]:
        name = r[ki]
        key = next((k for k in ALG if k in name.replace(" ", "")), None)
        if key is None:
            continue
        v = float(r[vi].replace(",", ""))
        u = r[ui]
        v *= {"nsecond": 1e-3, "ns": 1e-3, "us": 1.0, "usecond": 1.0, "msecond": 1e3, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6,
              "Gbyte": 1e9}.get(u, 1.0)
        vals[key][r[mi]].append(v)
    peaks = json.load(open("MEASURED_PEAKS.json")) if len(sys.argv) < 4 else {}
    hbm = None
    for k, v in peaks.items():
        if "hbm" in k.lower() and isinstance(v, (int, float)):
            hbm = v
            break
    res = {"source": "ncu --metrics (see tools/gpu_r02bc.sh) --clock-control none python tools/stats_once.py",
           "hbm_peak_GBps": hbm, "kernels": {}}
    for key, m in vals.items():
        d = {k: statistics.median(v) for k, v in m.items()}
        t_us = d.get("gpu__time_duration.sum")
        dram = d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
        e = {"launches": len(m.get("gpu__time_duration.sum", [])), "us": t_us, "dram_bytes": dram,
             "algorithmic_bytes": ALG[key],
             "dram_GBps": dram / (t_us * 1e3) if t_us else None,
             "algorithmic_GBps": ALG[key] / (t_us * 1e3) if t_us else None}
        if hbm and t_us:
            e["frac_of_hbm_peak"] = e["algorithmic_GBps"] / hbm
        for k, v in d.items():
            if k not in ("gpu__time_duration.sum",):
                e[k] = v
        res["kernels"][key] = e
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
