#!/usr/bin/env python
"""Per-layer conv2d forward GFLOP/s on B200 -- the paper's Fig. 1 methodology:
every algorithm x every layer of a set, plus the auto-selector's pick.

    python bench_layers.py --set resnet50|vgg16|stack|R4,R17 --batch 32 [--algos all|auto|direct,...]
                           [--math fp32|tf32] [--iters 10] [--warmup 3] [--out table.json]

Each (layer, algo) is timed with CUDA events over --iters launches after --warmup, with a
256 MiB L2 flush before every timed launch (outside the events); the best and median are
reported with GFLOP/s (direct-normalised flops, reading R8), GB/s (algorithmic bytes) and
the fraction of the layer's own roofline max(flops/peak, bytes/HBM).  Inputs are seeded
synthetic tensors generated on the device (synth.py twin).  Also used as the ncu target:
--layers R4 --algos implicit_gemm --iters 2.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1904_04174_b200 import layers as L  # noqa: E402
from paper_1904_04174_b200 import synth  # noqa: E402
from bench import layer_bytes, load_peaks  # noqa: E402

FFMA_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12  # 74.4 TF/s: the CUDA-core fp32 FMA ceiling at max SM clock


def layer_set(name):
    if name == "resnet50":
        return list(L.RESNET50_SETS)
    if name == "vgg16":
        return [l for l, _ in L.VGG16_LAYERS]
    if name == "stack":
        seen, out = set(), []
        for _, l in L.resnet50_v15_stack():
            if l.name not in seen:
                seen.add(l.name)
                out.append(l)
        return out
    return [L.by_name(n) for n in name.split(",")]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--set", default="resnet50")
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--algos", default="all")
    ap.add_argument("--math", choices=["fp32", "tf32"], default="fp32")
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--eager", action="store_true", help="time eager calls instead of CUDA-graph replays")
    ap.add_argument("--out", default="")
    args = ap.parse_args()

    import torch
    from paper_1904_04174_b200 import conv2d as C

    torch.cuda.set_device(0)
    math = C.MATH_FP32 if args.math == "fp32" else C.MATH_TF32
    peaks, src = load_peaks()
    tf32 = peaks["bf16_tflops"] / 2
    useful = tf32 / 3 if math == C.MATH_FP32 else tf32
    hbm = peaks["hbm_gbs"]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()
    C.conv2d_set_autotune_flush(flush)  # 'auto' tunes with cache-cold repetitions, as timed below
    if args.algos == "all":
        algos = list(range(1, C.NUM_ALGOS)) + [C.ALGO_AUTO]
    else:
        algos = [C.ALGO_BY_NAME[a] for a in args.algos.split(",")]
    rows = []
    for li, l in enumerate(layer_set(args.set)):
        p = C.Params(**l.params(args.batch), math=math)
        (n, ho, wo, f), _ = C.conv2d_output_shape(p)
        x = torch.empty(args.batch * l.rows * l.cols * l.channels, device="cuda")
        C.conv2d_synth_fill(x, x.numel(), synth.stream_key(synth.SEED, 900 + li, 0), 0, 0)
        w = torch.empty(l.window * l.window * l.channels * l.features, device="cuda")
        C.conv2d_synth_fill(w, w.numel(), synth.stream_key(synth.SEED, 900 + li, 1), 0, 0)
        y = torch.empty(n * ho * wo * f, device="cuda")
        need = C.conv2d_query_workspace(p, C.ALGO_AUTO)
        ws = torch.empty(max(need, 16), dtype=torch.uint8, device="cuda")
        flops = C.conv2d_flop_count(p)
        nbytes = layer_bytes(l, args.batch)
        roof_ms = max(flops / (useful * 1e12), nbytes / (hbm * 1e9)) * 1e3
        row = {"layer": l.name, "tuple": [l.window, l.stride, l.rows, l.cols, l.channels, l.features],
               "batch": args.batch, "gflop": round(flops / 1e9, 4), "mb": round(nbytes / 1e6, 2),
               "roofline_us": round(roof_ms * 1e3, 2), "algos": {}}
        for a in algos:
            if not C.conv2d_supports(p, a):
                continue
            name = C.ALGO_NAMES[a]
            if a == C.ALGO_AUTO:
                C.conv2d_clear_selection_cache()
            for _ in range(args.warmup):
                C.conv2d_forward(p, a, x, w, y, ws, ws.numel(), stream)
            torch.cuda.synchronize()
            # replay a captured CUDA graph of the call (as bench.py does) so host-side work -- tensor-map
            # encoding, launch calls -- is not inside the device-timed interval
            graph = None
            if not args.eager:
                try:
                    graph = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(graph, capture_error_mode="thread_local"):
                        C.conv2d_forward(p, a, x, w, y, ws, ws.numel(), torch.cuda.current_stream())
                    graph.replay()
                    torch.cuda.synchronize()
                except Exception:
                    graph = None
            times = []
            for _ in range(args.iters):
                if not args.no_flush:
                    flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                if graph is not None:
                    graph.replay()
                else:
                    C.conv2d_forward(p, a, x, w, y, ws, ws.numel(), stream)
                e1.record(stream)
                e1.synchronize()
                times.append(e0.elapsed_time(e1))
            best, med = min(times), statistics.median(times)
            ent = {"best_us": round(best * 1e3, 2), "median_us": round(med * 1e3, 2),
                   "gflops": round(flops / (best / 1e3) / 1e9, 1), "gbs": round(nbytes / (best / 1e3) / 1e9, 1),
                   "roofline_frac": round(roof_ms / best, 3)}
            if a in (C.ALGO_DIRECT, C.ALGO_TILED):
                # CUDA-core kernels graded against their own ceiling: the FFMA pipe (148 SMs x 128 FMA/clk x
                # 2 flop x 1.965 GHz = 74.4 TF/s) or HBM, whichever bounds the layer
                ffma_ms = max(flops / (FFMA_TFLOPS * 1e12), nbytes / (hbm * 1e9)) * 1e3
                ent["ffma_frac"] = round(ffma_ms / best, 3)
            if a == C.ALGO_AUTO:
                ent["chose"] = C.ALGO_NAMES[C.conv2d_selected(p)]
            row["algos"][name] = ent
        rows.append(row)
        if not row["algos"]:
            continue
        cand = [k for k in row["algos"] if k != "auto"] or list(row["algos"])
        best_algo = min(cand, key=lambda k: row["algos"][k]["best_us"])
        print(f"{l.name:4s} {str(row['tuple']):26s} roof {row['roofline_us']:9.1f}us  " +
              "  ".join(f"{k[:6]}:{v['gflops']/1e3:6.1f}TF({v['roofline_frac']:.2f})" for k, v in row["algos"].items())
              + f"  best={best_algo}", flush=True)
    out = {"set": args.set, "batch": args.batch, "math": args.math, "peak_useful_tflops": useful,
           "hbm_gbs": hbm, "peak_source": src, "layers": rows}
    if args.out:
        with open(args.out, "w") as fh:
            json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
