#!/usr/bin/env python
"""Per-kernel time share + DRAM bytes from an ncu launch list that includes dram__bytes_{read,write}.sum
(bench.py's timed region selected with --nvtx --nvtx-include "bench_timed/").  Writes markdown to stdout
and, with --json PATH, the totals used for bench.py's roofline "traffic" field."""
import csv
import json
import re
import sys
from collections import defaultdict

UNIT_T = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
UNIT_B = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main():
    path = sys.argv[1]
    lines = [l for l in open(path) if l.startswith('"')]
    launch = defaultdict(dict)
    for r in csv.DictReader(lines):
        d = launch[int(r["ID"])]
        d["name"] = r["Kernel Name"]
        v = float(r["Metric Value"].replace(",", ""))
        if r["Metric Name"] == "gpu__time_duration.sum":
            d["us"] = v * UNIT_T[r["Metric Unit"]]
        else:
            d[r["Metric Name"]] = v * UNIT_B[r["Metric Unit"]]
    agg = defaultdict(lambda: [0, 0.0, 0.0])
    for d in launch.values():
        n = re.sub(r"\(.*", "", d["name"]).replace("conv2d::<unnamed>::", "").replace("void ", "")
        a = agg[n]
        a[0] += 1
        a[1] += d.get("us", 0.0)
        a[2] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    tot = sum(v[1] for v in agg.values())
    print(f"# ncu launch list: `{path}`\n\n{len(launch)} launches, {tot:.1f} us serialised (cold-cache, one "
          f"launch at a time: compare shares with bench.py's live CUDA-event times, not absolutes)\n")
    print("| share | total us | launches | DRAM MB (r+w) | kernel |\n|---:|---:|---:|---:|---|")
    for n, (c, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| {100 * t / tot:5.1f}% | {t:9.1f} | {c:4d} | {b / 1e6:9.1f} | `{n}` |")
    if "--json" in sys.argv:
        g = [(k, v) for k, v in agg.items() if k.startswith("gemm2sm_kernel")]
        out = {"source": path, "gemm_launches": sum(v[0] for _, v in g), "gemm_us": sum(v[1] for _, v in g),
               "gemm_dram_bytes": sum(v[2] for _, v in g), "total_us": tot}
        json.dump(out, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)


if __name__ == "__main__":
    main()
