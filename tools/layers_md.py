#!/usr/bin/env python
"""Render bench_layers.py JSON tables as markdown (the paper's Fig. 1 methodology: GFLOP/s per layer and
algorithm, plus the fraction of each layer's own roofline).

    python tools/layers_md.py gpurun_out/tab_resnet50_b32_fp32.json ... > profiles/round1_layers.md
"""
import json
import sys

ALGOS = ["direct", "tiled", "implicit_gemm", "winograd_f2x2_3x3", "winograd_f4x4_3x3", "matmul_1x1", "auto"]


def main():
    for path in sys.argv[1:]:
        d = json.load(open(path))
        peak = d["peak_useful_tflops"]
        print(f"### {d['set']} batch {d['batch']}, math {d['math']} "
              f"(useful peak {peak:.1f} TF/s, HBM {d['hbm_gbs']:.0f} GB/s; `{path.split('/')[-1]}`)\n")
        print("| layer | K,S,H,W,C,F | GFLOP | roofline us | " + " | ".join(a for a in ALGOS) + " | auto chose |")
        print("|---|---|---:|---:|" + "---:|" * len(ALGOS) + "---|")
        for r in d["layers"]:
            cells = []
            for a in ALGOS:
                e = r["algos"].get(a)
                cells.append("—" if e is None else f"{e['gflops']/1e3:.1f} TF ({e['roofline_frac']:.2f})")
            chose = r["algos"].get("auto", {}).get("chose", "")
            print(f"| {r['layer']} | {','.join(map(str, r['tuple']))} | {r['gflop']:.2f} | {r['roofline_us']:.1f} | "
                  + " | ".join(cells) + f" | {chose} |")
        # which algorithm wins how often (the paper's "no single algorithm always performing best")
        wins = {}
        for r in d["layers"]:
            cand = [a for a in r["algos"] if a != "auto"] or list(r["algos"])
            best = min(cand, key=lambda a: r["algos"][a]["best_us"])
            wins[best] = wins.get(best, 0) + 1
        print("\nFastest algorithm per layer: " + ", ".join(f"{k} x{v}" for k, v in sorted(wins.items())) + "\n")


if __name__ == "__main__":
    main()
