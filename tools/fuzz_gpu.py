#!/usr/bin/env python
"""Randomised GPU parity sweep (a robustness check beyond tests/; not part of the suite).

    python tools/fuzz_gpu.py [--cases 2000] [--seed 1]

Each case draws a random shape (batch, rows, cols, channels, features, window 1-8, stride 1-3, SAME /
VALID), a math mode and a forced tuned-parameter variant (CONV2D_FORCE_VARIANT is read once per process,
so the variant is cycled through by re-running with --variant), runs every supported algorithm through
the C-ABI and checks the north_star tolerance against the oracle (integer inputs: bit-exact, F(4x4):
tolerance).  Prints failures and a summary; exit code 1 on any failure.
"""
from __future__ import annotations

import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", type=int, default=2000)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--focus", choices=["all", "c4", "s2d"], default="all",
                    help="c4: only 3x3 / stride 1 with C <= 4 (implicit_gemm's A_C4 4-channel halo path); "
                         "s2d: only 7x7 / 8x8 stride-2 stems with C <= 4 (the space-to-depth halo paths)")
    args = ap.parse_args()

    import torch
    import oracle as O
    from paper_1904_04174_b200 import conv2d as C
    from paper_1904_04174_b200 import synth

    O.build()
    rng = np.random.default_rng(args.seed)
    fails, runs = 0, 0
    for case in range(args.cases):
        k = int(rng.choice([1, 1, 3, 3, 3, 5, 7, 8, 2, 4]))
        kw = k if rng.random() < 0.8 else int(rng.integers(1, 8))
        s = int(rng.choice([1, 1, 1, 2, 2, 3]))
        n = int(rng.choice([1, 2, 3, 5, 8, 16]))
        h = int(rng.integers(max(k, 1), 72))
        w = int(rng.integers(max(kw, 1), 72))
        c = int(rng.choice([1, 2, 3, 4, 5, 8, 16, 24, 32, 48, 64, 96, 128, 256]))
        f = int(rng.choice([1, 3, 8, 16, 32, 33, 64, 96, 100, 128, 160, 256, 288, 512]))
        if args.focus == "c4":
            k = kw = 3
            s = 1
            c = int(rng.choice([1, 2, 3, 4]))
            w = int(rng.integers(1, 40)) * (4 // np.gcd(c, 4))  # W*C % 4 == 0 (raw 16-byte rows)
            h = int(rng.integers(1, 72))
            f = int(rng.choice([1, 3, 8, 17, 32, 36, 64, 96, 100, 128]))
        if args.focus == "s2d":
            k = int(rng.choice([7, 8]))
            kw = int(rng.choice([7, 8]))
            s = 2
            c = int(rng.choice([1, 2, 3, 3, 4]))
            w = int(rng.integers(kw, 90))
            h = int(rng.integers(k, 90))
            f = int(rng.choice([1, 3, 8, 17, 32, 36, 64, 96, 100, 128]))
        pad = int(rng.integers(0, 2))
        math = int(rng.integers(0, 2))
        integer = rng.random() < 0.3
        p = C.Params(n, h, w, c, f, k, kw, s, s, pad, math=math)
        try:
            (N, ho, wo, F), _ = C.conv2d_output_shape(p)
        except Exception:
            continue
        dist = synth.DIST_INT5 if integer else synth.DIST_UNIFORM
        x = synth.input_nhwc(n, h, w, c, layer_id=2000 + case, dist=dist)
        wt = synth.filter_hwcf(k, kw, c, f, layer_id=2000 + case, dist=dist)
        ref, den = O.conv2d(O.Params(n, h, w, c, f, k, kw, s, s, pad), x, wt, with_denom=True)
        xd, wd = torch.from_numpy(x).cuda(), torch.from_numpy(wt).cuda()
        for a in range(1, C.NUM_ALGOS):
            if not C.conv2d_supports(p, a):
                continue
            y = torch.full((N * ho * wo * F,), float("nan"), device="cuda")
            need = C.conv2d_query_workspace(p, a)
            ws = torch.full((max(need, 16),), 0xFF, dtype=torch.uint8, device="cuda")
            C.conv2d_forward(p, a, xd, wd, y, ws, need)
            torch.cuda.synchronize()
            got = y.cpu().numpy().reshape(ref.shape)
            runs += 1
            tensor = a in (C.ALGO_IMPLICIT_GEMM, C.ALGO_MATMUL_1X1, C.ALGO_WINOGRAD_F2X2_3X3, C.ALGO_WINOGRAD_F4X4_3X3)
            tol = 2e-3 if (math == C.MATH_TF32 and tensor) else 1e-5
            if integer and a != C.ALGO_WINOGRAD_F4X4_3X3:
                ok = np.array_equal(got, ref)
                err = float(np.nanmax(np.abs(got - ref))) if not ok else 0.0
            else:
                err = O.normalized_error(got, ref, den) if np.all(np.isfinite(got)) else float("inf")
                ok = err <= tol
            if not ok:
                fails += 1
                print(f"FAIL case {case}: {p} int={integer} algo={C.ALGO_NAMES[a]} err={err:.3e}", flush=True)
    print(f"fuzz: {runs} algorithm runs over {args.cases} cases, {fails} failures "
          f"(CONV2D_FORCE_VARIANT={os.environ.get('CONV2D_FORCE_VARIANT', 'unset')})", flush=True)
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()
