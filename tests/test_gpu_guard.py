"""Memory-safety and race checks of every kernel without compute-sanitizer (closed on this pool: runs under it
left GPUs needing a reset).  SURVEY.md §5 asks for memcheck / racecheck evidence on the warp-specialised
mbarrier / TMEM pipelines; this is the substitute, on the shapes of tools/sanitize_driver.py (one per A path,
B path, split mode and CUDA-core kernel), every algorithm x every enumerated parameter variant x math mode:

  * out-of-bounds writes: the output and the workspace sit between 64 KiB guard bands filled with a canary bit
    pattern; every band must be intact afterwards (a stray store past either end of the output, the
    workspace tail or the split-K planes shows up here), and the inputs must be bit-unchanged;
  * unwritten outputs: the output is poisoned with NaN first (every element must be written);
  * races: three further launches into differently-poisoned outputs must reproduce the first bit for bit
    (a missing barrier in a producer/consumer ring shows up as run-to-run differences, as the gather race
    fixed in round 1 did), and the result is checked against the oracle within the P10 ceiling.
"""
import numpy as np
import pytest

import oracle as O
from paper_1904_04174_b200 import synth

from .parity import C, check_close, oparams

pytestmark = pytest.mark.gpu

GUARD = 64 * 1024  # bytes per guard band
CANARY = 0x7FBADBAD  # a NaN bit pattern no kernel produces from finite inputs

SHAPES = [
    (1, 8, 8, 4, 8, 3, 3, 1, 1, 0),
    (2, 20, 20, 64, 64, 3, 3, 1, 1, 0),
    (1, 14, 14, 128, 256, 3, 3, 1, 1, 1),
    (2, 12, 12, 64, 256, 1, 1, 1, 1, 0),
    (1, 15, 13, 128, 160, 3, 3, 2, 2, 0),
    (2, 7, 7, 512, 512, 3, 3, 1, 1, 0),
    (2, 150, 128, 256, 64, 1, 1, 1, 1, 0),
    (1, 37, 29, 3, 64, 7, 7, 2, 2, 0),
    (2, 23, 19, 3, 64, 7, 7, 2, 2, 0),
    (1, 44, 43, 48, 100, 1, 1, 1, 1, 0),
    (3, 11, 12, 8, 16, 4, 4, 2, 1, 0),
    (1, 13, 11, 5, 130, 3, 3, 2, 1, 0),
    (2, 33, 70, 3, 64, 3, 3, 1, 1, 0),       # V1-like small C for the tiled kernel's vector paths
    (2, 33, 68, 3, 64, 3, 3, 1, 1, 0),       # implicit_gemm A_C4 (4-channel halo; W*C % 4 == 0), ragged tiles
    (3, 17, 12, 1, 17, 3, 3, 1, 1, 1),       # A_C4, C = 1, VALID, F % 4 != 0 (LSU epilogue)
    (1, 9, 9, 20, 24, 5, 5, 1, 1, 0),        # tiled generic (runtime KW) path, F % 16 != 0
    # fused Winograd F(2x2) (winograd_f2x2_3x3 variant 1): ragged tile blocks / NB > 1 / odd Ho, F % 32 != 0
    (3, 15, 9, 64, 68, 3, 3, 1, 1, 1),
    (9, 7, 7, 32, 96, 3, 3, 1, 1, 0),
    (1, 9, 7, 40, 36, 3, 3, 1, 1, 0),
]


def _guarded(nbytes, dev="cuda"):
    """A uint8 buffer [guard | body (nbytes rounded to 16) | guard] with canaries in both guards."""
    import torch
    body = (max(nbytes, 16) + 15) // 16 * 16
    buf = torch.empty(GUARD + body + GUARD, dtype=torch.uint8, device=dev)
    buf.view(torch.int32).fill_(CANARY)
    return buf, body


def _guards_intact(buf, body):
    import torch
    w = buf.view(torch.int32)
    g = GUARD // 4
    return bool((w[:g] == CANARY).all()) and bool((w[g + body // 4:] == CANARY).all())


def _run(p, algo, x, w, variant, poison):
    import torch
    c = C()
    if variant is not None:
        c.conv2d_set_variant(p, algo, variant)
    (n, ho, wo, f), _ = c.conv2d_output_shape(p)
    nout = n * ho * wo * f
    yb, ybody = _guarded(nout * 4)
    y = yb[GUARD:GUARD + nout * 4].view(torch.float32)
    y.view(torch.int32).fill_(poison)
    need = c.conv2d_query_workspace(p, algo)
    wsb, wsbody = _guarded(need)
    ws = wsb[GUARD:GUARD + wsbody]
    ws.fill_(0xA5)
    c.conv2d_forward(p, algo, x, w, y, ws if need else None, need)
    torch.cuda.synchronize()
    assert _guards_intact(yb, ybody), f"{c.ALGO_NAMES[algo]} v={variant}: write outside the output"
    assert _guards_intact(wsb, wsbody), f"{c.ALGO_NAMES[algo]} v={variant}: write outside the workspace"
    return y.clone()


@pytest.mark.parametrize("case", SHAPES, ids=str)
def test_guard_bands_and_repeatability(cuda_ok, case):
    import torch
    c = C()
    p0 = c.Params(*case)
    xh, wh = (synth.input_nhwc(p0.batch, p0.in_rows, p0.in_cols, p0.channels, layer_id=3300),
              synth.filter_hwcf(p0.window_rows, p0.window_cols, p0.channels, p0.features, layer_id=3300))
    ref, den = O.conv2d(oparams(p0), xh, wh, with_denom=True)
    x, w = torch.from_numpy(xh).cuda(), torch.from_numpy(wh).cuda()
    x0, w0 = x.clone(), w.clone()
    for math in (c.MATH_FP32, c.MATH_TF32):
        p = p0.replace(math=math)
        for a in range(1, c.NUM_ALGOS):
            if not c.conv2d_supports(p, a):
                continue
            tuned = a in (c.ALGO_IMPLICIT_GEMM, c.ALGO_MATMUL_1X1, c.ALGO_WINOGRAD_F2X2_3X3)
            for v in (c.conv2d_variants(p, a) if tuned else [None]):
                y1 = _run(p, a, x, w, v, 0x7FC00000)  # quiet NaN
                assert bool(torch.isfinite(y1).all()), f"{case} {c.ALGO_NAMES[a]} v={v}: unwritten outputs"
                for poison in (0x7FC00001, 0x00000000, 0x7F800000):
                    y2 = _run(p, a, x, w, v, poison)
                    assert torch.equal(y1.view(torch.int32), y2.view(torch.int32)), \
                        f"{case} {c.ALGO_NAMES[a]} v={v} math={math}: run-to-run difference (race?)"
                assert torch.equal(x, x0) and torch.equal(w, w0), f"{c.ALGO_NAMES[a]} v={v}: input modified"
                check_close(p, y1.view(ref.shape).cpu().numpy(), ref, den, a, f"guard {case} {a} v={v} m={math}")
            if tuned:
                c.conv2d_set_variant(p, a, 0)
