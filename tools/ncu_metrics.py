#!/usr/bin/env python
"""Print the key utilisation metrics and the top stall-sampled SASS lines of every kernel in an
ncu --set full report.   python tools/ncu_metrics.py report.ncu-rep [kernel-regex] [top]"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_requests.sum", "lts__t_sector_hit_rate.pct",
        "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum",
        "l1tex__m_l1tex2xbar_write_bytes_mem_global_op_tma_st.sum"]


def ncu(rep, *a):
    return subprocess.run(["ncu", "-i", rep, *a], capture_output=True, text=True).stdout


def main():
    rep = sys.argv[1]
    kre = sys.argv[2] if len(sys.argv) > 2 else "."
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 12
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    h, units = rows[0], rows[1]
    for r in rows[2:]:
        print("==", r[h.index("Kernel Name")][:100])
        for k in KEYS:
            if k in h:
                print(f"   {k}: {r[h.index(k)]} {units[h.index(k)]}")
    src = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source=sass", "-k", "regex:" + kre))))
    hdr = next(i for i, r in enumerate(src) if "Source" in r and "Address" in r)
    h = src[hdr]
    data = src[hdr + 1:]
    i_s, i_src = h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
    tot = sum(int(r[i_s]) for r in data if len(r) > i_s and r[i_s].isdigit())
    print(f"== top stall lines ({tot} samples)")
    order = sorted(range(len(data)), key=lambda i: -int(data[i][i_s]) if len(data[i]) > i_s and data[i][i_s].isdigit() else 0)
    for i in order[:top]:
        r = data[i]
        print(f"   {int(r[i_s]):7d} {100 * int(r[i_s]) / max(tot, 1):5.1f}%  [{i:5d}] {r[i_src].strip()[:90]}")


if __name__ == "__main__":
    main()
