#!/usr/bin/env python
"""Per-launch DRAM traffic of the GEMM kernels in one timed bench.py step, from an ncu launch list
taken with --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum over the
NVTX range "bench_timed" (one step).  Writes the JSON bench.py's roofline.traffic reads.

    python tools/step_traffic.py gpurun_out/launches.csv [global_batch=256] > profiles/round1_step_traffic.json

(bench.py uses the file only for the workload it was captured on: b256 -> round1_step_traffic.json,
any other batch B -> round1_step_traffic_b{B}.json.)
"""
import csv
import json
import re
import sys
from collections import defaultdict

GEMM = re.compile(r"gemm2sm_kernel|halo_kernel")


def main():
    path = sys.argv[1]
    batch = int(sys.argv[2]) if len(sys.argv) > 2 else 256
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    per = defaultdict(dict)
    names = {}
    for r in csv.DictReader(lines):
        per[r["ID"]][r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
        names[r["ID"]] = r["Kernel Name"]
    n = 0
    us = total = byts = 0.0
    for i, m in per.items():
        t = m.get("gpu__time_duration.sum", 0.0) / 1e3  # ns -> us
        total += t
        if GEMM.search(names[i]):
            n += 1
            us += t
            byts += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    step_bytes = sum(m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0) for m in per.values())
    json.dump({"source": path, "global_batch": batch, "gemm_launches": n, "gemm_us": us, "gemm_dram_bytes": byts,
               "total_us": total, "gemm_time_share": us / total if total else None, "step_launches": len(per),
               "step_dram_bytes": step_bytes}, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main()
