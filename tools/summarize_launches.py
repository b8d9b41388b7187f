#!/usr/bin/env python
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into per-kernel shares.

    python tools/summarize_launches.py gpurun_out/launches.csv [--skip-regex synth|vectorized] > profiles/x.md

ncu's per-launch times are cold-cache and serialised: compare SHARES with bench.py's live
CUDA-event numbers, not absolute times (B200_PROFILING.md).
"""
import csv
import re
import sys
from collections import defaultdict


def main():
    path = sys.argv[1]
    skip = None
    if "--skip-regex" in sys.argv:
        skip = re.compile(sys.argv[sys.argv.index("--skip-regex") + 1])
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    rd = csv.DictReader(lines)
    for r in rd:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"]
        if skip and skip.search(name):
            continue
        unit = r.get("Metric Unit", "")
        v = float(r["Metric Value"].replace(",", ""))
        scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(unit, 1.0)
        rows.append((name, v * scale))
    agg = defaultdict(lambda: [0, 0.0])
    for n, t in rows:
        short = re.sub(r"\(.*", "", n)
        short = re.sub(r"conv2d::<unnamed>::|conv2d::\(anonymous namespace\)::", "", short)
        m = re.search(r"<(.*)>", n)
        key = short if not m else short  # template args kept in the name column
        agg[n][0] += 1
        agg[n][1] += t
    total = sum(v[1] for v in agg.values())
    print(f"# ncu launch list summary: {path}\n")
    print(f"{len(rows)} launches, {total:.1f} us total (serialised, cold-cache)\n")
    print("| share | total us | launches | kernel |")
    print("|---:|---:|---:|---|")
    for n, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| {100 * t / total:5.1f}% | {t:9.1f} | {c:4d} | `{n[:150]}` |")


if __name__ == "__main__":
    main()
