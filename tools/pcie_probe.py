#!/usr/bin/env python
"""Pinned-host <-> device copy bandwidth, each direction alone and both at once (e2e design check)."""
import torch, time
n = 1 << 28  # 1 GiB of fp32
h_in = torch.empty(n, dtype=torch.float32, pin_memory=True); h_in.fill_(1.0)
h_out = torch.empty(n, dtype=torch.float32, pin_memory=True)
d_a = torch.empty(n, device="cuda"); d_b = torch.ones(n, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def timed(fn, reps=3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / reps
def h2d():
    with torch.cuda.stream(s1): d_a.copy_(h_in, non_blocking=True)
def d2h():
    with torch.cuda.stream(s2): h_out.copy_(d_b, non_blocking=True)
def both():
    h2d(); d2h()
for name, fn in (("h2d", h2d), ("d2h", d2h), ("both", both)):
    fn(); t = timed(fn)
    gb = 4 * n / 1e9 * (2 if name == "both" else 1)
    print(f"{name}: {t*1e3:.1f} ms  {gb/t:.1f} GB/s total")
