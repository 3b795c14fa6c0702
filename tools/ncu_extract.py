"""Extract the roofline evidence of one captured kernel from an ncu report
(ncu --set full ... -o rep) into JSON: duration, DRAM bytes, tensor-pipe and
issue activity, registers, grid / cluster shape.

  ncu -i rep.ncu-rep --page raw --csv > raw.csv
  python tools/ncu_extract.py raw.csv "<shape>" "<source command>" > out.json"""
import csv
import json
import sys

WANT = {
    "gpu__time_duration.sum": "gpu_time_us",
    "dram__bytes_read.sum": "dram_bytes_read",
    "dram__bytes_write.sum": "dram_bytes_write",
    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_realtime_pct_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "launch__registers_per_thread": "registers_per_thread",
    "launch__grid_size": "grid",
    "launch__cluster_dim_x": "cluster_x",
    "lts__t_bytes.sum": "l2_bytes",
}
SCALE = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main(path, shape, source):
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr, units, vals = rows[hdr_i], rows[hdr_i + 1], rows[hdr_i + 2]
    out = {"kernel": vals[hdr.index("Kernel Name")], "shape": shape, "source": source}
    for metric, key in WANT.items():
        # raw-page headers may carry a section prefix ("TPC.TriageCompute.")
        js = [j for j, h in enumerate(hdr) if h == metric or h.endswith("." + metric)]
        if js:
            j = js[0]
            try:
                v = float(vals[j].replace(",", ""))
            except ValueError:
                continue
            out[key] = v * SCALE.get(units[j], 1.0)
    if "dram_bytes_read" in out and "dram_bytes_write" in out:
        out["dram_bytes_per_launch"] = out["dram_bytes_read"] + out["dram_bytes_write"]
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3])
