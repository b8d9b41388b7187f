#!/usr/bin/env python
"""Timing data for the learned algorithm selector ("these tuning
decisions involve many parameters and a large number of features ... a good candidate for a learned
solution rather than a hand tuned one").

    python tools/selector_data.py --shapes 400 --seed 3 --out gpurun_out/selector_data.json
    python tools/selector_data.py --replay profiles/data/selector_data_r1*.json --only c4 --out ...

(--replay re-times the shapes of earlier data files -- filtered by --only -- with the current library: a
round-2 path change, e.g. the 4-channel halo of 3x3/s1 C <= 4 layers, changes what a candidate means there, and
tools/train_selector.py lets the later file's rows replace the earlier ones.)

For every conv shape -- the paper's 35 layer tuples at batch 1 / 32 / 256 in both math modes, then random
CNN-like shapes (window 1/3/5/7, stride 1/2, 7..224 pixels, 3..2048 channels, batch 1..256, bounded work) --
times every candidate the auto-selector would consider -- each supported algorithm, and for
implicit_gemm / matmul_1x1 each enumerated parameter variant (conv2d_set_variant) -- as the best of 3
cache-cold conv2d_forward calls (256 MiB L2 flush before each, CUDA events), microseconds.  Inputs are seeded synthetic tensors generated on the device.
tools/train_selector.py turns the JSON into the decision tree compiled into libconv2d.so.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1904_04174_b200 import layers as L  # noqa: E402
from paper_1904_04174_b200 import synth  # noqa: E402


def paper_shapes():
    out = []
    for l in L.RESNET50_SETS + [v for v, _ in L.VGG16_LAYERS]:
        for b in (1, 32, 256):
            for math in (0, 1):
                out.append(dict(l.params(b), math=math))
    return out


def random_shapes(n, rng):
    out = []
    while len(out) < n:
        k = int(rng.choice([1, 1, 1, 3, 3, 3, 3, 5, 7]))
        s = int(rng.choice([1, 1, 1, 2])) if k != 7 else 2
        h = int(rng.choice([7, 13, 14, 27, 28, 55, 56, 112, 224]))
        c = int(rng.choice([3, 16, 32, 48, 64, 96, 128, 256, 384, 512, 1024, 2048]))
        f = int(rng.choice([16, 32, 64, 96, 128, 192, 256, 512, 1024, 2048]))
        b = int(rng.choice([1, 2, 8, 16, 32, 64, 128, 256]))
        pad = int(rng.random() < 0.15)  # 1 = VALID
        math = int(rng.random() < 0.35)
        if pad == 1 and k > h:
            continue
        ho = (h - k) // s + 1 if pad else -(-h // s)
        flops = 2 * b * ho * ho * k * k * c * f
        elems = b * h * h * c + b * ho * ho * f
        if flops > 60e9 or elems * 4 > 3e9 or flops < 1e6:
            continue
        out.append(dict(batch=b, in_rows=h, in_cols=h, channels=c, features=f, window_rows=k, window_cols=k,
                        stride_rows=s, stride_cols=s, padding=pad, math=math))
    return out


def time_us(p, a, x, w, y, ws, need, reps=3):
    """Best of `reps` cache-cold conv2d_forward calls (256 MiB L2 flush before each, outside the events)."""
    import torch
    from paper_1904_04174_b200 import conv2d as C
    s = torch.cuda.current_stream()
    C.conv2d_forward(p, a, x, w, y, ws, need, s)  # warm-up (first-call setup)
    best = float("inf")
    for _ in range(reps):
        FLUSH[0].zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        C.conv2d_forward(p, a, x, w, y, ws, need, s)
        e1.record(s)
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3)
    return round(best, 2)


FLUSH = [None]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", type=int, default=400)
    ap.add_argument("--seed", type=int, default=3)
    ap.add_argument("--out", default="gpurun_out/selector_data.json")
    ap.add_argument("--replay", nargs="*", default=[], help="re-time the shapes of these data files instead")
    ap.add_argument("--only", choices=["all", "c4"], default="all",
                    help="c4: only 3x3 / stride 1 shapes with C <= 4, W*C % 4 == 0, F <= 128 (A_C4-eligible)")
    args = ap.parse_args()

    import torch
    from paper_1904_04174_b200 import conv2d as C

    torch.cuda.set_device(0)
    FLUSH[0] = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    rng = np.random.default_rng(args.seed)
    if args.replay:
        import gzip
        shapes = []
        for path in args.replay:
            fh = gzip.open(path, "rt") if path.endswith(".gz") else open(path)
            shapes += [r["params"] for r in json.load(fh)["rows"]]
    else:
        shapes = paper_shapes() + random_shapes(args.shapes, rng)
    if args.only == "c4":
        shapes = [sp for sp in shapes if sp["window_rows"] == 3 and sp["window_cols"] == 3 and sp["stride_rows"] == 1
                  and sp["stride_cols"] == 1 and sp["channels"] <= 4 and (sp["in_cols"] * sp["channels"]) % 4 == 0
                  and sp["features"] <= 128]
    rows = []
    for i, sp in enumerate(shapes):
        p = C.Params(**sp)
        (n, ho, wo, f), _ = C.conv2d_output_shape(p)
        x = torch.empty(sp["batch"] * sp["in_rows"] * sp["in_cols"] * sp["channels"], device="cuda")
        w = torch.empty(sp["window_rows"] * sp["window_cols"] * sp["channels"] * sp["features"], device="cuda")
        C.conv2d_synth_fill(x, x.numel(), synth.stream_key(synth.SEED, 3000 + i, synth.ROLE_INPUT), 0, 0)
        C.conv2d_synth_fill(w, w.numel(), synth.stream_key(synth.SEED, 3000 + i, synth.ROLE_FILTER), 0, 0)
        y = torch.empty(n * ho * wo * f, device="cuda")
        need = C.conv2d_query_workspace(p, C.ALGO_AUTO)
        ws = torch.empty(max(need, 16), dtype=torch.uint8, device="cuda")
        times = {}
        for a in range(1, C.NUM_ALGOS):
            if not C.conv2d_supports(p, a):
                continue
            variants = [None]
            if a in (C.ALGO_IMPLICIT_GEMM, C.ALGO_MATMUL_1X1):
                variants = []
                for v in range(64):  # the enumerated variants are exactly those set_variant accepts
                    try:
                        C.conv2d_set_variant(p, a, v)
                        variants.append(v)
                    except C.Conv2dError:
                        pass
            for v in variants:
                if v is not None:
                    C.conv2d_set_variant(p, a, v)
                times[C.ALGO_NAMES[a] + ("" if v is None else f"/{v}")] = time_us(p, a, x, w, y, ws, need)
        best = min(times, key=times.get)
        rows.append({"params": sp, "best": best, "times_us": times, "gflop": C.conv2d_flop_count(p) / 1e9})
        print(f"{i:4d} {sp} -> {best}  {times[best]:.1f} us ({len(times)} candidates)", flush=True)
        del x, w, y, ws
    with open(args.out, "w") as fh:
        out = {"device": torch.cuda.get_device_name(0), "rows": rows}
        if args.replay and args.only != "all":
            out["supersedes"] = args.only  # tools/train_selector.py drops the earlier rows of this class
        json.dump(out, fh)


if __name__ == "__main__":
    main()
