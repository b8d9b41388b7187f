#!/usr/bin/env python
"""Error model behind the P10 ceilings: a numpy emulation of what the kernels
compute, sampled outputs of the paper's layers on uniform [-1,1) data, max e = |y - y_exact| / sum|x||w|.

  gemm3x  : 3xTF32 implicit GEMM -- operands split hi = trunc_tf32(x), lo = x - hi (reading R16); per K=8
            MMA step the three products lo*hi, hi*lo, hi*hi (in this order) are summed
            exactly and added to an fp32 accumulator rounded either to nearest (RN) or toward zero (RZ)
  wino4   : Winograd F(4x4,3x3) in 3xTF32 -- the fp32 filter / input / output transforms of winograd.cu (same
            operation order) around an exactly-summed 3xTF32 contraction; isolates the transforms' rounding
  gemm1x  : plain TF32 (hi*hi only), RZ accumulation

Results are printed as a table; DESIGN.md quotes them next to the measured maxima of the GPU suite.

    python tools/error_model.py [--samples 300]
"""
from __future__ import annotations

import argparse
import sys
import os

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1904_04174_b200 import synth  # noqa: E402

f32 = np.float32


def trunc_tf32(x):
    return (np.asarray(x, f32).view(np.uint32) & np.uint32(0xFFFFE000)).view(f32)


def add_rz(acc, v):
    """fp32 acc + v rounded toward zero (exact sum in double, then truncate the binary64 -> binary32)."""
    s = acc.astype(np.float64) + v
    r = s.astype(f32)  # RN
    # move one ulp toward zero where RN rounded away from zero
    away = np.abs(r.astype(np.float64)) > np.abs(s)
    r[away] = np.nextafter(r[away], f32(0))
    return r


def gemm_emul(a, b, mode="3x", rounding="RZ"):
    """a: [P, K] fp32 rows, b: [K] fp32 column; per K=8 step accumulate in fp32."""
    ah, bh = trunc_tf32(a), trunc_tf32(b)
    al, bl = (a - ah).astype(f32), (b - bh).astype(f32)
    al, bl = trunc_tf32(al), trunc_tf32(bl)  # the MMA reads TF32 operands
    acc = np.zeros(a.shape[0], f32)
    add = add_rz if rounding == "RZ" else (lambda x, v: (x.astype(np.float64) + v).astype(f32))
    for k0 in range(0, a.shape[1], 8):
        sl = slice(k0, k0 + 8)
        terms = [(al, bh), (ah, bl), (ah, bh)] if mode == "3x" else [(ah, bh)]
        for p, q in terms:
            acc = add(acc, (p[:, sl].astype(np.float64) * q[sl].astype(np.float64)).sum(axis=1))
    return acc


def im2col_rows(x, kh, kw, pt, pl, pts):
    n, h, w, c = x.shape
    rows = []
    for (i, j) in pts:
        r = np.zeros((kh, kw, c), f32)
        for a in range(kh):
            for b in range(kw):
                ih, iw = i + a - pt, j + b - pl
                if 0 <= ih < h and 0 <= iw < w:
                    r[a, b] = x[0, ih, iw]
        rows.append(r.reshape(-1))
    return np.stack(rows)


# F(4x4,3x3) transforms in fp32, the operation order of csrc/winograd.cu (g4 / bt4 / at4)
def g4(g):
    return [f32(0.25) * g[0], -(g[0] + g[1] + g[2]) * f32(1 / 6), -(g[0] - g[1] + g[2]) * f32(1 / 6),
            g[0] * f32(1 / 24) + g[1] * f32(1 / 12) + g[2] * f32(1 / 6),
            g[0] * f32(1 / 24) - g[1] * f32(1 / 12) + g[2] * f32(1 / 6), g[2]]


def bt4(d):
    return [f32(4) * d[0] - f32(5) * d[2] + d[4], f32(-4) * d[1] - f32(4) * d[2] + d[3] + d[4],
            f32(4) * d[1] - f32(4) * d[2] - d[3] + d[4], f32(-2) * d[1] - d[2] + f32(2) * d[3] + d[4],
            f32(2) * d[1] - d[2] - f32(2) * d[3] + d[4], f32(4) * d[1] - f32(5) * d[3] + d[5]]


def at4(m):
    return [m[0] + m[1] + m[2] + m[3] + m[4], m[1] - m[2] + f32(2) * m[3] - f32(2) * m[4],
            m[1] + m[2] + f32(4) * m[3] + f32(4) * m[4], m[1] - m[2] + f32(8) * m[3] - f32(8) * m[4] + m[5]]


def two_d(fn, t, rows_in, cols_in):
    """apply a 1-D transform along axis 0 then axis 1 of t[rows_in][cols_in][...] (lists of arrays)."""
    cols = [fn([t[a][b] for a in range(rows_in)]) for b in range(cols_in)]  # column b -> list over out rows
    q = [[cols[b][a] for b in range(cols_in)] for a in range(len(cols[0]))]
    return [fn(q[a]) for a in range(len(q))]


def wino4_tile(x, w, th, tw, f):
    """4x4 outputs of feature f for the tile at (4th, 4tw) of image 0, SAME pad 1; x fp32 NHWC, w HWCF."""
    _, h, wd, c = x.shape
    d = [[np.zeros(c, f32) for _ in range(6)] for _ in range(6)]
    for a in range(6):
        for b in range(6):
            ih, iw = 4 * th + a - 1, 4 * tw + b - 1
            if 0 <= ih < h and 0 <= iw < wd:
                d[a][b] = x[0, ih, iw].astype(f32)
    V = two_d(bt4, d, 6, 6)                     # [6][6] arrays over c
    g = [[w[a, b, :, f].astype(f32) for b in range(3)] for a in range(3)]
    U = two_d(g4, g, 3, 3)
    M = [[f32(0)] * 6 for _ in range(6)]
    for a in range(6):
        for b in range(6):
            M[a][b] = gemm_emul(V[a][b][None, :], U[a][b], "3x", "RZ")[0]
    Y = two_d(at4, M, 6, 6)
    return np.array([[Y[i][j] for j in range(4)] for i in range(4)], np.float64)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--samples", type=int, default=300)
    a = ap.parse_args()
    rng = np.random.default_rng(0)
    print("| shape (H, C, F, 3x3 SAME) | model | max e | mean e |")
    print("|---|---|---:|---:|")
    for (h, c, fo) in [(28, 512, 512), (56, 256, 256), (56, 64, 64)]:
        x = synth.input_nhwc(1, h, h, c, layer_id=7000 + c)
        w = synth.filter_hwcf(3, 3, c, fo, layer_id=7000 + c)
        pts = [(int(rng.integers(0, h)), int(rng.integers(0, h))) for _ in range(a.samples)]
        fs = rng.integers(0, fo, a.samples)
        A = im2col_rows(x, 3, 3, 1, 1, pts)
        exact = np.array([A[i].astype(np.float64) @ w[:, :, :, fs[i]].reshape(-1).astype(np.float64)
                          for i in range(len(pts))])
        den = np.array([np.abs(A[i]).astype(np.float64) @ np.abs(w[:, :, :, fs[i]].reshape(-1)).astype(np.float64)
                        for i in range(len(pts))])
        for mode, rnd in (("3x", "RN"), ("3x", "RZ"), ("1x", "RZ")):
            got = np.array([gemm_emul(A[i:i + 1], w[:, :, :, fs[i]].reshape(-1), mode, rnd)[0] for i in range(len(pts))])
            e = np.abs(got - exact) / den
            print(f"| {h}, {c}, {fo} | gemm {mode}TF32 acc {rnd} | {e.max():.2e} | {e.mean():.2e} |")
        # Winograd F(4x4): compare whole tiles
        errs = []
        for i in range(max(8, a.samples // 16)):
            th, tw = int(rng.integers(0, h // 4)), int(rng.integers(0, h // 4))
            f = int(rng.integers(0, fo))
            y = wino4_tile(x, w, th, tw, f)
            for u in range(4):
                for v in range(4):
                    r = im2col_rows(x, 3, 3, 1, 1, [(4 * th + u, 4 * tw + v)])[0].astype(np.float64)
                    wf = w[:, :, :, f].reshape(-1).astype(np.float64)
                    errs.append(abs(y[u, v] - r @ wf) / (np.abs(r) @ np.abs(wf)))
        print(f"| {h}, {c}, {fo} | winograd F(4x4) fp32 transforms + 3xTF32 RZ | {max(errs):.2e} | {np.mean(errs):.2e} |")


if __name__ == "__main__":
    main()
