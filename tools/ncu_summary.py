#!/usr/bin/env python
"""Key metrics of an ncu --set full capture (.ncu-rep) as markdown: duration, DRAM bytes,
tensor-pipe / smem-pipe utilisation, L2 hit rate, stall top-list (source page).

    python tools/ncu_summary.py gpurun_out/full_R17.ncu-rep "R17 b256 3xTF32" [algorithmic_bytes]
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe active % (elapsed)"),
    ("l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem tensor-core read pipe %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem LSU pipe %"),
    ("dram__bytes_read.sum.pct_of_peak_sustained_elapsed", "DRAM read % of peak"),
    ("dram__bytes_write.sum.pct_of_peak_sustained_elapsed", "DRAM write % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__cluster_dim_x", "cluster x"),
]


def main():
    rep, title = sys.argv[1], sys.argv[2]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    print(f"## {title}\n\n`{rep}`\n")
    for v in rows[2:]:  # one table per captured kernel
        name = v[h.index("Kernel Name")] if "Kernel Name" in h else "?"
        print(f"kernel `{name[:160]}`\n\n| metric | value |\n|---|---:|")
        for k, label in KEYS:
            if k in h:
                i = h.index(k)
                print(f"| {label} (`{k}`) | {v[i]} {units[i]} |")
        print()
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    srows = list(csv.reader(io.StringIO(src)))
    if len(srows) > 2:
        hh = srows[1]
        data = srows[2:]
        i_s, i_src = hh.index("Warp Stall Sampling (All Samples)"), hh.index("Source")
        tot = sum(float(r[i_s] or 0) for r in data) or 1.0
        print("\nTop stall sites (share of all warp samples; SASS):\n")
        for r in sorted(data, key=lambda r: -float(r[i_s] or 0))[:8]:
            print(f"- {100 * float(r[i_s]) / tot:5.1f}%  `{r[i_src].strip()[:80]}`")
    print()


if __name__ == "__main__":
    main()
