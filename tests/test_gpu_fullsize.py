"""Full-size parity in the launch configuration bench.py times: every distinct conv of the
ResNet-50 v1.5 stack at batch 256 (BASELINE config 5, per-GPU batch at N=1), through
conv2d_forward(AUTO) after the same measured auto-selection, FP32 (3xTF32) mode; plus the
per-GPU batch of the 8-GPU run (32) for the small-M split-K configurations.

The oracle cannot run 2 TFLOP in seconds, so outputs are SAMPLED: all F features of the first
and last output pixel of the batch and ~1500 random (n, ho, wo, f), each evaluated by the
oracle's brute-force dot product in double (oracle_conv2d_points) on the same seeded inputs.
The tolerance is the north_star bound (reading R7).
"""
import numpy as np
import pytest

import oracle as O
from paper_1904_04174_b200 import layers as L
from paper_1904_04174_b200 import synth

from .parity import C, TOL_FP32, TOL_TF32, ceiling_for

pytestmark = pytest.mark.gpu


def _distinct_stack():
    seen, out = set(), []
    for conv_id, l in L.resnet50_v15_stack():
        if l.name not in seen:
            seen.add(l.name)
            out.append((conv_id, l))
    return out


def _sample_idx(rng, n, ho, wo, f, count):
    idx = np.stack([rng.integers(0, n, count), rng.integers(0, ho, count), rng.integers(0, wo, count),
                    rng.integers(0, f, count)], axis=1)
    edge = [[0, 0, 0, k] for k in range(f)] + [[n - 1, ho - 1, wo - 1, k] for k in range(f)]
    return np.concatenate([idx, np.array(edge)], axis=0).astype(np.int64)


def _run(conv_id, l, batch, math, samples=1500):
    import torch
    c = C()
    p = c.Params(**l.params(batch), math=math)
    (n, ho, wo, f), _ = c.conv2d_output_shape(p)
    x = torch.empty(batch * l.rows * l.cols * l.channels, device="cuda")
    c.conv2d_synth_fill(x, x.numel(), synth.stream_key(synth.SEED, conv_id, synth.ROLE_INPUT), 0, 0)
    w = torch.empty(l.window * l.window * l.channels * l.features, device="cuda")
    c.conv2d_synth_fill(w, w.numel(), synth.stream_key(synth.SEED, conv_id, synth.ROLE_FILTER), 0, 0)
    y = torch.full((n * ho * wo * f,), float("nan"), device="cuda")
    need = c.conv2d_query_workspace(p, c.ALGO_AUTO)
    ws = torch.empty(max(need, 16), dtype=torch.uint8, device="cuda")
    algo = c.conv2d_autotune(p, x, w, y, ws, ws.numel())
    y.fill_(float("nan"))
    c.conv2d_forward(p, c.ALGO_AUTO, x, w, y, ws, ws.numel())
    torch.cuda.synchronize()
    yh = y.view(n, ho, wo, f).cpu().numpy()
    assert np.isfinite(yh).all(), f"{l.name}: unwritten/non-finite outputs"
    # host copies of the SAME device-generated inputs (generator equality is its own test)
    xh = x.view(batch, l.rows, l.cols, l.channels).cpu().numpy()
    wh = w.view(l.window, l.window, l.channels, l.features).cpu().numpy()
    rng = np.random.default_rng(conv_id)
    idx = _sample_idx(rng, n, ho, wo, f, samples)
    op = O.Params(batch, l.rows, l.cols, l.channels, l.features, l.window, l.window, l.stride, l.stride, O.SAME)
    ref, den = O.conv2d_points(op, xh, wh, idx)
    got = yh[idx[:, 0], idx[:, 1], idx[:, 2], idx[:, 3]].astype(np.float64)
    e = float(np.max(np.abs(got - ref) / den))
    tol = min(TOL_FP32 if math == c.MATH_FP32 else TOL_TF32, ceiling_for(algo, math))
    assert e <= tol, f"{l.name} b{batch} math={math} algo={c.ALGO_NAMES[algo]}: err {e:.3e} > {tol}"
    return e, c.ALGO_NAMES[algo]


@pytest.mark.parametrize("conv_id,layer", _distinct_stack(), ids=lambda v: v.name if hasattr(v, "name") else str(v))
def test_stack_layer_b256_sampled(cuda_ok, conv_id, layer):
    _run(conv_id, layer, 256, 0)


@pytest.mark.parametrize("name", ["R1", "R4", "R17", "R20", "R24", "R26"])
def test_stack_layer_b32_sampled_both_modes(cuda_ok, name):
    conv_id, l = next((i, l) for i, l in _distinct_stack() if l.name == name)
    _run(conv_id, l, 32, 0)
    _run(conv_id, l, 32, 1)


def test_synth_input_equals_host_generator_at_size(cuda_ok):
    """The device-generated bench inputs are the host generator's values (first/last 10^5 of R1 b256)."""
    import torch
    c = C()
    l = L.by_name("R1")
    count = 256 * l.rows * l.cols * l.channels
    key = synth.stream_key(synth.SEED, 0, synth.ROLE_INPUT)
    x = torch.empty(count, device="cuda")
    c.conv2d_synth_fill(x, count, key, 0, 0)
    torch.cuda.synchronize()
    xh = x.cpu().numpy()
    assert np.array_equal(xh[:100000], synth.draw(100000, key, 0))
    assert np.array_equal(xh[-100000:], synth.draw(100000, key, count - 100000))


@pytest.mark.parametrize("k,f", [(1, 32), (3, 32)], ids=["1x1", "3x3"])
def test_input_beyond_2e31_elements(cuda_ok, k, f):
    """Maximum sizes (reading R20): an input of 65 x 512 x 512 x 128 = 2.18e9 elements (8.7 GB, > 2^31)
    through every supported algorithm (FP32 math), sampled against the oracle's point evaluation.
    Exercises the 64-bit offsets of every kernel and the TMA maps' 32-bit per-dimension coordinates."""
    import torch
    c = C()
    n, h, wd, ch = 65, 512, 512, 128
    p = c.Params(n, h, wd, ch, f, k, k, 1, 1, c.PAD_SAME)
    assert n * h * wd * ch > 2 ** 31
    (_, ho, wo, _), _ = c.conv2d_output_shape(p)
    x = torch.empty(n * h * wd * ch, device="cuda")
    c.conv2d_synth_fill(x, x.numel(), synth.stream_key(synth.SEED, 1300 + k, synth.ROLE_INPUT), 0, 0)
    w = torch.empty(k * k * ch * f, device="cuda")
    c.conv2d_synth_fill(w, w.numel(), synth.stream_key(synth.SEED, 1300 + k, synth.ROLE_FILTER), 0, 0)
    y = torch.empty(n * ho * wo * f, device="cuda")
    xh = x.view(n, h, wd, ch).cpu().numpy()
    wh = w.view(k, k, ch, f).cpu().numpy()
    rng = np.random.default_rng(k)
    idx = _sample_idx(rng, n, ho, wo, f, 400)
    ref, den = O.conv2d_points(O.Params(n, h, wd, ch, f, k, k, 1, 1, O.SAME), xh, wh, idx)
    for a in range(1, c.NUM_ALGOS):
        if not c.conv2d_supports(p, a):
            continue
        need = c.conv2d_query_workspace(p, a)
        ws = torch.empty(max(need, 16), dtype=torch.uint8, device="cuda")
        y.fill_(float("nan"))
        c.conv2d_forward(p, a, x, w, y, ws, ws.numel())
        torch.cuda.synchronize()
        del ws
        got = y.view(n, ho, wo, f)[idx[:, 0], idx[:, 1], idx[:, 2], idx[:, 3]].cpu().numpy().astype(np.float64)
        e = float(np.max(np.abs(got - ref) / den))
        assert e <= TOL_FP32, f"{c.ALGO_NAMES[a]} {k}x{k}: err {e:.3e}"
        torch.cuda.empty_cache()
