#!/usr/bin/env python
"""Run one conv2d_forward through the C-ABI and compare with the oracle (debug helper).
    python tools/probe_conv.py N H W C F KH KW SH SW PAD [math] [algo]"""
import os
import sys
import numpy as np
import torch
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_1904_04174_b200 import conv2d as C
import oracle as O

a = [int(v) for v in sys.argv[1:11]]
math = int(sys.argv[11]) if len(sys.argv) > 11 else 0
algo = C.ALGO_BY_NAME[sys.argv[12]] if len(sys.argv) > 12 else C.ALGO_IMPLICIT_GEMM
n, h, w, c, f, kh, kw, sh, sw, pad = a
rng = np.random.default_rng(1)
uniform = os.environ.get("PROBE_UNIFORM") is not None
if uniform:
    x = rng.uniform(-1, 1, size=(n, h, w, c)).astype(np.float32)
    wt = rng.uniform(-1, 1, size=(kh, kw, c, f)).astype(np.float32)
else:
    x = rng.integers(-2, 3, size=(n, h, w, c)).astype(np.float32)
    wt = rng.integers(-2, 3, size=(kh, kw, c, f)).astype(np.float32)
p = C.Params(n, h, w, c, f, kh, kw, sh, sw, pad, math=math)
(N, ho, wo, F), _ = C.conv2d_output_shape(p)
y = torch.full((N * ho * wo * F,), float("nan"), device="cuda")
ws = torch.empty(max(C.conv2d_query_workspace(p, algo), 16), dtype=torch.uint8, device="cuda")
C.conv2d_forward(p, algo, torch.from_numpy(x).cuda(), torch.from_numpy(wt).cuda(), y, ws, ws.numel())
torch.cuda.synchronize()
O.build()
ref, den = O.conv2d(O.Params(n, h, w, c, f, kh, kw, sh, sw, pad), x, wt, with_denom=True)
got = y.cpu().numpy().reshape(ref.shape)
if uniform:
    e = np.abs(got.astype(np.float64) - ref) / den
    bad = np.argwhere(e > 1e-5)
    print(a, "norm err %.3e" % e.max(), "bad", len(bad), bad[:6].tolist())
else:
    bad = np.argwhere(got != ref)
    print(a, "bad", len(bad), "of", got.size, bad[:4].tolist())
