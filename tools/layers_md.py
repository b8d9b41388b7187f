#!/usr/bin/env python
"""Render bench_layers.py JSON tables as markdown (the paper's Fig. 1 methodology: GFLOP/s per layer and
algorithm, plus the fraction of each layer's own roofline).

    python tools/layers_md.py [--oracle oracle_layers.json] gpurun_out/tab_resnet50_b32_fp32.json ... > profiles/round2_layers.md

direct / tiled cells show their fraction of the CUDA-core ceiling (FFMA 74.4 TF/s or HBM, whichever bounds the
layer) in square brackets after the tensor-roofline fraction.  --oracle adds the host oracle's GFLOP/s per layer
(bench.py --oracle-layers: one image, all host cores; the batch does not change a per-image rate).
"""
import json
import sys

ALGOS = ["direct", "tiled", "implicit_gemm", "winograd_f2x2_3x3", "winograd_f4x4_3x3", "matmul_1x1", "auto"]


def main():
    argv = sys.argv[1:]
    orc = None
    if argv and argv[0] == "--oracle":
        orc = json.load(open(argv[1]))
        argv = argv[2:]
        orc_layers = orc["oracle_layers"]
    for path in argv:
        d = json.load(open(path))
        peak = d["peak_useful_tflops"]
        print(f"### {d['set']} batch {d['batch']}, math {d['math']} "
              f"(useful peak {peak:.1f} TF/s, HBM {d['hbm_gbs']:.0f} GB/s; `{path.split('/')[-1]}`)\n")
        extra = f" | oracle ({orc['cores']} cores)" if orc else ""
        print("| layer | K,S,H,W,C,F | GFLOP | roofline us | " + " | ".join(a for a in ALGOS) + " | auto chose" + extra
              + " |")
        print("|---|---|---:|---:|" + "---:|" * len(ALGOS) + "---|" + ("---:|" if orc else ""))
        for r in d["layers"]:
            cells = []
            for a in ALGOS:
                e = r["algos"].get(a)
                if e is None:
                    cells.append("—")
                    continue
                ff = f" [{e['ffma_frac']:.2f}]" if "ffma_frac" in e else ""
                cells.append(f"{e['gflops']/1e3:.1f} TF ({e['roofline_frac']:.2f}){ff}")
            chose = r["algos"].get("auto", {}).get("chose", "")
            oc = ""
            if orc:
                o = orc_layers.get(r["layer"])
                oc = f" | {o['gflops']:.1f} GF" if o else " | —"
            print(f"| {r['layer']} | {','.join(map(str, r['tuple']))} | {r['gflop']:.2f} | {r['roofline_us']:.1f} | "
                  + " | ".join(cells) + f" | {chose}{oc} |")
        # which algorithm wins how often (the paper's "no single algorithm always performing best")
        wins = {}
        for r in d["layers"]:
            cand = [a for a in r["algos"] if a != "auto"] or list(r["algos"])
            best = min(cand, key=lambda a: r["algos"][a]["best_us"])
            wins[best] = wins.get(best, 0) + 1
        print("\nFastest algorithm per layer: " + ", ".join(f"{k} x{v}" for k, v in sorted(wins.items())) + "\n")


if __name__ == "__main__":
    main()
