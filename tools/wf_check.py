#!/usr/bin/env python
"""Fused Winograd F(2x2) bring-up check: CONV2D_ALGO_WINOGRAD_F2X2_3X3 on shapes that exercise the tile-block
geometries (whole images with NB > 1, ragged blocks, odd Ho/Wo, VALID, F % 32 != 0, C % 16 != 0), integer
(bit-exact) and uniform (normalised error) data, both math modes, against the oracle.
    python tools/wf_check.py [--quick]"""
import sys
import os
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1904_04174_b200 import conv2d as C  # noqa: E402
from paper_1904_04174_b200 import synth  # noqa: E402
import oracle as O  # noqa: E402

SHAPES = [  # N H W C F pad
    (1, 8, 8, 32, 32, 0),
    (1, 14, 14, 256, 256, 0),
    (2, 7, 7, 512, 512, 0),
    (1, 56, 56, 64, 64, 0),
    (3, 15, 9, 64, 68, 1),
    (1, 9, 7, 40, 36, 0),
    (5, 28, 28, 128, 128, 0),
    (9, 7, 7, 32, 96, 0),
    (1, 224, 224, 64, 64, 0),
]


def run(p, x, w):
    (n, ho, wo, f), _ = C.conv2d_output_shape(p)
    y = torch.full((n, ho, wo, f), float("nan"), device="cuda")
    need = C.conv2d_query_workspace(p, C.ALGO_WINOGRAD_F2X2_3X3)
    ws = torch.full((max(need, 16),), 0xFF, dtype=torch.uint8, device="cuda")
    xd, wd = torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda()
    C.conv2d_forward(p, C.ALGO_WINOGRAD_F2X2_3X3, xd, wd, y, ws, need)
    torch.cuda.synchronize()
    return y.cpu().numpy(), (xd, wd, y, ws, need)


def main():
    O.build()
    bad = 0
    for (n, h, w_, c, f, pad) in SHAPES:
        for math in (0, 1):
            p = C.Params(n, h, w_, c, f, 3, 3, 1, 1, pad, math=math)
            op = O.Params(n, h, w_, c, f, 3, 3, 1, 1, pad)
            for dist in (synth.DIST_INT5, synth.DIST_UNIFORM):
                x = synth.input_nhwc(n, h, w_, c, layer_id=7, dist=dist)
                wt = synth.filter_hwcf(3, 3, c, f, layer_id=7, dist=dist)
                ref, den = O.conv2d(op, x, wt, with_denom=True)
                y, bufs = run(p, x, wt)
                if dist == synth.DIST_INT5:
                    nbad = int(np.sum(y != ref))
                    ok = nbad == 0
                    msg = f"int bad={nbad}/{y.size}"
                    if not ok:
                        idx = np.argwhere(y != ref)[:5].tolist()
                        msg += f" first={idx} got={[float(y[tuple(i)]) for i in idx]} ref={[float(ref[tuple(i)]) for i in idx]}"
                else:
                    e = O.normalized_error(y, ref, den)
                    ok = np.all(np.isfinite(y)) and e <= (1e-5 if math == 0 else 2e-3)
                    msg = f"uniform err={e:.2e} finite={bool(np.all(np.isfinite(y)))}"
                bad += 0 if ok else 1
                print(f"{'ok ' if ok else 'BAD'} {(n, h, w_, c, f, pad)} math={math} {msg}", flush=True)
            # timing (device events), 10 reps
            xd, wd, yd, ws, need = bufs
            s = torch.cuda.current_stream()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            for _ in range(2):
                C.conv2d_forward(p, C.ALGO_WINOGRAD_F2X2_3X3, xd, wd, yd, ws, need)
            e0.record(s)
            for _ in range(10):
                C.conv2d_forward(p, C.ALGO_WINOGRAD_F2X2_3X3, xd, wd, yd, ws, need)
            e1.record(s)
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 100.0
            gf = 2.0 * n * (h if pad == 0 else h - 2) * (w_ if pad == 0 else w_ - 2) * 9 * c * f / us / 1e3
            print(f"    time {us:.1f} us  {gf:.1f} GFLOP/s (direct-normalised)", flush=True)
    print("FAILURES", bad)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
