#!/usr/bin/env python3
"""Summarise an ncu --csv launch list (gpu__time_duration, dram bytes) per
kernel: median duration, DRAM read/write per launch, achieved DRAM GB/s."""
import csv
import json
import sys

TU = {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}
BU = {"byte": 1, "Kbyte": 1e3, "KB": 1e3, "Mbyte": 1e6, "MB": 1e6, "Gbyte": 1e9, "GB": 1e9}


def main(path):
    lines = open(path).read().split("\n")
    start = [j for j, l in enumerate(lines) if l.startswith('"ID"')][0]
    agg = {}
    for r in csv.DictReader(lines[start:]):
        name = r["Kernel Name"].split("(")[0].replace("void ", "").replace("qgk::", "")
        agg.setdefault((r["ID"], name), {})[r["Metric Name"]] = (float(r["Metric Value"].replace(",", "")), r["Metric Unit"])
    per = {}
    for (_, name), m in agg.items():
        t, rb, wb = m["gpu__time_duration.sum"], m["dram__bytes_read.sum"], m["dram__bytes_write.sum"]
        per.setdefault(name, []).append((t[0] * TU[t[1]], rb[0] * BU[rb[1]], wb[0] * BU[wb[1]]))
    out = {}
    for name, v in per.items():
        v.sort()
        t, rb, wb = v[len(v) // 2]
        out[name] = {"launches": len(v), "median_ms": round(t * 1e3, 4), "dram_read_bytes": int(rb),
                     "dram_write_bytes": int(wb), "dram_gbs": round((rb + wb) / t / 1e9, 1)}
        print(f"{name:42s} n={len(v):3d} t={t * 1e3:.4f} ms  r={rb / 1e6:8.1f} MB  w={wb / 1e6:8.1f} MB  "
              f"{(rb + wb) / t / 1e9:7.0f} GB/s", file=sys.stderr)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1])
