#!/usr/bin/env python
"""Time one conv2d_forward configuration through the C-ABI (A/B helper for kernel work).
    python tools/time_layer.py N H W C F KH KW SH SW PAD [math] [algo] [iters]
Env knobs (CONV2D_FORCE_VARIANT, CONV2D_NO_C4, ...) select the path under test.  Prints the median
event-timed ms per call (L2 flushed between calls), direct-normalised TFLOP/s and output GB/s."""
import os
import sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1904_04174_b200 import conv2d as C

a = [int(v) for v in sys.argv[1:11]]
math = int(sys.argv[11]) if len(sys.argv) > 11 else 0
algo = C.ALGO_BY_NAME[sys.argv[12]] if len(sys.argv) > 12 else C.ALGO_IMPLICIT_GEMM
iters = int(sys.argv[13]) if len(sys.argv) > 13 else 20
n, h, w, c, f, kh, kw, sh, sw, pad = a
p = C.Params(n, h, w, c, f, kh, kw, sh, sw, pad, math=math)
(N, ho, wo, F), _ = C.conv2d_output_shape(p)
x = torch.rand(n, h, w, c, device="cuda") - 0.5
wt = torch.rand(kh, kw, c, f, device="cuda") - 0.5
y = torch.empty(N * ho * wo * F, device="cuda")
ws = torch.empty(max(C.conv2d_query_workspace(p, algo), 16), dtype=torch.uint8, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    C.conv2d_forward(p, algo, x, wt, y, ws, ws.numel())
torch.cuda.synchronize()
ts = []
for _ in range(iters):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    C.conv2d_forward(p, algo, x, wt, y, ws, ws.numel())
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ts.sort()
ms = ts[len(ts) // 2]
flops = 2.0 * N * ho * wo * F * kh * kw * c
byts = 4.0 * (n * h * w * c + N * ho * wo * F)
print(f"{a} math={math} algo={algo} launches={C.conv2d_launch_count(p, algo)} ms={ms:.4f} "
      f"TF/s={flops / ms / 1e9:.1f} GB/s={byts / ms / 1e6:.0f} min_ms={ts[0]:.4f}")
