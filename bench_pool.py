#!/usr/bin/env python
"""NHWC pooling throughput on B200 against the HBM roofline (include/pool2d.h).

    python bench_pool.py [--iters 20] [--warmup 3] [--out profiles/data/pool_r1.json] [--no-cpu]

Workloads: the pooling layers of the paper's networks -- ResNet-50's stem max pool (3x3 / 2 SAME on
112x112x64) at b256 and b32, its global average pool (7x7 VALID on 7x7x2048), and VGG-16's five 2x2 / 2
max pools at b32.  Algorithmic bytes = 4 * (input + output) elements; each timed launch is a CUDA-graph
replay bracketed by CUDA events on the launching stream, with a 256 MiB L2 flush before it (outside
the events).  Inputs are seeded synthetic tensors generated on the device.  --cpu times the oracle
(oracle/pool.c) on one image of each workload on the host cores for reference.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1904_04174_b200 import synth  # noqa: E402
from bench import load_peaks  # noqa: E402

# name, batch, H, W, C, K, S, padding (0 SAME, 1 VALID), op (0 max, 1 avg)
WORKLOADS = [
    ("resnet50_stem_maxpool", 256, 112, 112, 64, 3, 2, 0, 0),
    ("resnet50_stem_maxpool", 32, 112, 112, 64, 3, 2, 0, 0),
    ("resnet50_global_avgpool", 256, 7, 7, 2048, 7, 1, 1, 1),
    ("vgg16_pool1", 32, 224, 224, 64, 2, 2, 1, 0),
    ("vgg16_pool2", 32, 112, 112, 128, 2, 2, 1, 0),
    ("vgg16_pool3", 32, 56, 56, 256, 2, 2, 1, 0),
    ("vgg16_pool4", 32, 28, 28, 512, 2, 2, 1, 0),
    ("vgg16_pool5", 32, 14, 14, 512, 2, 2, 1, 0),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--out", default="")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()

    import torch
    from paper_1904_04174_b200 import conv2d as C

    torch.cuda.set_device(0)
    peaks, src = load_peaks()
    hbm = peaks["hbm_gbs"]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()
    rows = []
    for i, (name, n, h, w, c, k, s, pad, op) in enumerate(WORKLOADS):
        p = C.PoolParams(n, h, w, c, k, k, s, s, pad, op)
        (_, ho, wo, _), _ = C.pool2d_output_shape(p)
        x = torch.empty(n * h * w * c, dtype=torch.float32, device="cuda")
        C.conv2d_synth_fill(x, x.numel(), synth.stream_key(synth.SEED, 1200 + i, synth.ROLE_INPUT), 0, 0)
        y = torch.empty(n * ho * wo * c, dtype=torch.float32, device="cuda")
        for _ in range(args.warmup):
            C.pool2d_forward(p, x, y, stream)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, capture_error_mode="thread_local"):
            C.pool2d_forward(p, x, y, torch.cuda.current_stream())
        g.replay()
        torch.cuda.synchronize()
        times = []
        for _ in range(args.iters):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            g.replay()
            e1.record(stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1) / 1e3)
        nbytes = 4 * (x.numel() + y.numel())
        best, med = min(times), statistics.median(times)
        row = {"workload": name, "batch": n, "in": [h, w, c], "window": k, "stride": s,
               "padding": "valid" if pad else "same", "op": "avg" if op else "max", "mb": round(nbytes / 1e6, 2),
               "best_us": round(best * 1e6, 2), "median_us": round(med * 1e6, 2),
               "gbs": round(nbytes / best / 1e9, 1), "roofline_frac": round(nbytes / best / 1e9 / hbm, 3)}
        if not args.no_cpu:
            import numpy as np
            import oracle as O
            xi = synth.input_nhwc(1, h, w, c, layer_id=1200 + i)
            op_ = O.PoolParams(1, h, w, c, k, k, s, s, pad, op)
            t0 = time.perf_counter()
            O.pool2d(op_, xi)
            dt = time.perf_counter() - t0
            row["cpu_oracle_gbs_1img"] = round(4 * (xi.size + np.prod(O.pool_output_shape(op_)[0])) / dt / 1e9, 2)
        rows.append(row)
        print(f"{name:24s} b{n:<3d} {row['op']} {k}x{k}/{s} {row['padding']:5s} {row['mb']:8.1f} MB "
              f"{row['best_us']:8.1f} us  {row['gbs']:7.1f} GB/s  {row['roofline_frac']:.2f} of HBM", flush=True)
    out = {"hbm_gbs": hbm, "peak_source": src, "workloads": rows,
           "timing": "CUDA-graph replay, CUDA events on the launching stream, 256 MiB L2 flush before each"}
    if args.out:
        with open(args.out, "w") as fh:
            json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
