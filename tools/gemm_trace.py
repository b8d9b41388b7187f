#!/usr/bin/env python
"""Per-CTA timeline of the GEMM core for a few layers (include/conv2d_debug.h).

    python tools/gemm_trace.py --layers R3,R12,R26 --batch 32 [--math fp32|tf32]

For each layer: one warm call, L2 flush, then one traced call (eager) bracketed by CUDA events.
Prints, relative to the earliest CTA entry (us): spread of CTA entries, setup done, first TMA issue,
first MMA stage, first accumulator, last store issued, stores drained, exit -- as median / max over
CTAs -- next to the event-timed duration of the whole conv2d_forward call.
"""
from __future__ import annotations

import argparse
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1904_04174_b200 import layers as L  # noqa: E402
from paper_1904_04174_b200 import synth  # noqa: E402

NAMES = ["entry", "setup", "tma0", "mma0", "acc0", "st_last", "drain", "exit"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", default="R3,R12,R26")
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--math", choices=["fp32", "tf32"], default="fp32")
    ap.add_argument("--flush", choices=["dirty", "clean", "none"], default="dirty",
                    help="before the traced call: write 256 MiB (L2 full of dirty lines, as after a previous "
                         "conv's output), read 256 MiB (clean lines), or nothing (inputs hot in L2)")
    args = ap.parse_args()

    import torch
    from paper_1904_04174_b200 import conv2d as C

    torch.cuda.set_device(0)
    math = C.MATH_FP32 if args.math == "fp32" else C.MATH_TF32
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()
    for li, name in enumerate(args.layers.split(",")):
        l = L.by_name(name)
        p = C.Params(**l.params(args.batch), math=math)
        (n, ho, wo, f), _ = C.conv2d_output_shape(p)
        x = torch.empty(args.batch * l.rows * l.cols * l.channels, device="cuda")
        C.conv2d_synth_fill(x, x.numel(), synth.stream_key(synth.SEED, 900 + li, 0), 0, 0)
        w = torch.empty(l.window * l.window * l.channels * l.features, device="cuda")
        C.conv2d_synth_fill(w, w.numel(), synth.stream_key(synth.SEED, 900 + li, 1), 0, 0)
        y = torch.empty(n * ho * wo * f, device="cuda")
        ws = torch.empty(max(C.conv2d_query_workspace(p, C.ALGO_AUTO), 16), dtype=torch.uint8, device="cuda")
        for _ in range(3):
            C.conv2d_forward(p, C.ALGO_AUTO, x, w, y, ws, ws.numel(), stream)
        algo = C.ALGO_NAMES[C.conv2d_selected(p)]
        torch.cuda.synchronize()
        C.conv2d_debug_trace(1)
        if args.flush == "dirty":
            flush.zero_()
        elif args.flush == "clean":
            flush.max()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        C.conv2d_forward(p, C.ALGO_AUTO, x, w, y, ws, ws.numel(), stream)
        e1.record(stream)
        torch.cuda.synchronize()
        t = C.conv2d_debug_trace(0, read=True)
        ctas = [t[i * 8:(i + 1) * 8] for i in range(148) if t[i * 8] != 0]
        if not ctas:
            print(f"{name}: {algo} -- no GEMM-core launch traced (halo/direct/tiled path)")
            continue
        base = min(c[0] for c in ctas)
        cols = []
        for k in range(8):
            v = [(c[k] - base) / 1e3 for c in ctas if c[k] != 0]
            cols.append((statistics.median(v), max(v)) if v else (float("nan"), float("nan")))
        print(f"{name:4s} {algo:14s} ctas={len(ctas):3d} call={e0.elapsed_time(e1) * 1e3:7.1f}us  " +
              " ".join(f"{NAMES[k]}={cols[k][0]:.1f}/{cols[k][1]:.1f}" for k in range(8)), flush=True)


if __name__ == "__main__":
    main()
