#!/usr/bin/env python
"""Small-size driver for compute-sanitizer (VERDICT r1 "next" item 7): every kernel of
libconv2d.so -- every algorithm, every enumerated parameter variant of implicit_gemm / matmul_1x1 (each A path:
im2col, dense, gather, narrow, row-segment, stem, halo, space-to-depth; both B paths; K splits), both math
modes, plus pooling -- once on a small seeded input, checked for finiteness (parity is the test suite's job).

    compute-sanitizer --tool memcheck|racecheck|synccheck python tools/sanitize_driver.py [--quick]

Exit 0 when every call returned CONV2D_OK and every output is finite.  Prints one line per call.
"""
from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1904_04174_b200 import conv2d as C  # noqa: E402
from paper_1904_04174_b200 import synth  # noqa: E402

# (N, H, W, C, F, KH, KW, SH, SW, pad): each reaches a different A-operand path / kernel
SHAPES = [
    (1, 8, 8, 4, 8, 3, 3, 1, 1, 0),          # config 1: direct, tiled, A_C4 (row-segment alternative)
    (2, 20, 20, 64, 64, 3, 3, 1, 1, 0),      # halo (F <= 128), im2col alternative, Winograd F2/F4
    (1, 14, 14, 128, 256, 3, 3, 1, 1, 1),    # im2col BN=256 / 128, Winograd VALID
    (2, 12, 12, 64, 256, 1, 1, 1, 1, 0),     # dense 1x1 (matmul_1x1), direct-B and K-major B
    (1, 15, 13, 128, 160, 3, 3, 2, 2, 0),    # im2col stride 2, SAME corners, ragged N
    (2, 7, 7, 512, 512, 3, 3, 1, 1, 0),      # deep K: balanced split + reduce, Winograd split
    (2, 150, 128, 256, 64, 1, 1, 1, 1, 0),   # remainder split (rsplit_reduce)
    (1, 37, 29, 3, 64, 7, 7, 2, 2, 0),       # s2d stem (C = 3), row-segment / stem alternatives
    (2, 23, 19, 3, 64, 7, 7, 2, 2, 0),       # row-segment stem
    (1, 44, 43, 48, 100, 1, 1, 1, 1, 0),     # gather A path with 3xTF32 lo in TMEM
    (3, 11, 12, 8, 16, 4, 4, 2, 1, 0),       # narrow im2col boxes
    (1, 13, 11, 5, 130, 3, 3, 2, 1, 0),      # C % 4 != 0: channel padding + gather
    (2, 33, 68, 3, 64, 3, 3, 1, 1, 0),       # 4-channel halo (A_C4), row-segment alternative
    (3, 17, 12, 1, 17, 3, 3, 1, 1, 1),       # A_C4 with C = 1, VALID, F % 4 != 0
]
QUICK = SHAPES[:4]


def run(p, algo, x, w, variant=None):
    (n, ho, wo, f), _ = C.conv2d_output_shape(p)
    y = torch.full((n * ho * wo * f,), float("nan"), device="cuda")
    if variant is not None:
        C.conv2d_set_variant(p, algo, variant)
    need = C.conv2d_query_workspace(p, algo)
    ws = torch.empty(max(need, 16), dtype=torch.uint8, device="cuda")
    C.conv2d_forward(p, algo, x, w, y, ws, ws.numel())
    torch.cuda.synchronize()
    ok = bool(torch.isfinite(y).all())
    print(f"{'ok  ' if ok else 'FAIL'} {C.ALGO_NAMES[algo]:18s} v={variant} math={p.math} {tuple(p.c().__getattribute__(k) for k in ('batch', 'in_rows', 'in_cols', 'channels', 'features', 'window_rows', 'stride_rows'))}",
          flush=True)
    return ok


def main():
    quick = "--quick" in sys.argv
    torch.cuda.set_device(0)
    fails = 0
    for i, case in enumerate(QUICK if quick else SHAPES):
        p0 = C.Params(*case)
        xh = synth.input_nhwc(p0.batch, p0.in_rows, p0.in_cols, p0.channels, layer_id=3000 + i)
        wh = synth.filter_hwcf(p0.window_rows, p0.window_cols, p0.channels, p0.features, layer_id=3000 + i)
        x, w = torch.from_numpy(xh).cuda(), torch.from_numpy(wh).cuda()
        for math in (C.MATH_FP32, C.MATH_TF32):
            p = p0.replace(math=math)
            for a in range(1, C.NUM_ALGOS):
                if not C.conv2d_supports(p, a):
                    continue
                if a in (C.ALGO_IMPLICIT_GEMM, C.ALGO_MATMUL_1X1, C.ALGO_WINOGRAD_F2X2_3X3):
                    for v in C.conv2d_variants(p, a):
                        fails += not run(p, a, x, w, v)
                else:
                    fails += not run(p, a, x, w)
    for op in (C.POOL_MAX, C.POOL_AVG):
        pp = C.PoolParams(2, 19, 17, 64, 3, 3, 2, 2, C.PAD_SAME, op)
        x = torch.from_numpy(synth.input_nhwc(2, 19, 17, 64, layer_id=3100)).cuda()
        (n, ho, wo, c), _ = C.pool2d_output_shape(pp)
        y = torch.full((n, ho, wo, c), float("nan"), device="cuda")
        C.pool2d_forward(pp, x, y)
        torch.cuda.synchronize()
        ok = bool(torch.isfinite(y).all())
        fails += not ok
        print(f"{'ok  ' if ok else 'FAIL'} pool2d op={op}", flush=True)
    print(f"sanitize_driver: {fails} failures", flush=True)
    return 1 if fails else 0


if __name__ == "__main__":
    sys.exit(main())
