"""Parity at the paper's full batch sizes, per algorithm (VERDICT r1 "next" item 1):

  * every VGG-16 layer (V1-V9, BASELINE configs[1]) at batch 32, every supported algorithm, both math modes;
  * every distinct conv of the ResNet-50 v1.5 stack (BASELINE configs[2]/[4]) at batch 32, every supported
    algorithm, both math modes;
  * the stack at batch 256 in TF32 mode through conv2d_forward(AUTO) after the measured selection
    (the 3xTF32 run is tests/test_gpu_fullsize.py);
  * P11 at size: the 8 batch-32 shards of the batch-256 inputs, run with the algorithm (and tuned variant)
    AUTO chose for batch 256, equal the batch-256 output -- bitwise when both launch plans accumulate every
    output without a K split (conv2d_debug_splits == 1 for both), else within the tolerance (a split count
    follows the tile count and so the batch: include/conv2d_debug.h).

The oracle cannot run these sizes in full, so outputs are SAMPLED on the device: all F features of the first
and last output pixel plus ~1000 random (n, ho, wo, f), each evaluated by the oracle's brute-force dot product
in double (oracle.conv2d_points) on the same seeded inputs.  Tolerance: north_star (reading R7).
"""
import numpy as np
import pytest

import oracle as O
from paper_1904_04174_b200 import layers as L
from paper_1904_04174_b200 import synth

from .parity import C, TOL_FP32, TOL_TF32, ceiling_for, record_err, tol_for

pytestmark = pytest.mark.gpu
MATHS = (0, 1)


def _distinct_stack():
    seen, out = set(), []
    for conv_id, l in L.resnet50_v15_stack():
        if l.name not in seen:
            seen.add(l.name)
            out.append((conv_id, l))
    return out


STACK = _distinct_stack()
VGG = [(2000 + i, l) for i, (l, _) in enumerate(L.VGG16_LAYERS)]


class Case:
    """Device inputs of one layer at one batch (device twin of synth.py, global image indices)."""

    def __init__(self, layer_id, l, batch):
        import torch
        c = C()
        self.l, self.batch, self.layer_id = l, batch, layer_id
        self.x = torch.empty(batch * l.rows * l.cols * l.channels, device="cuda")
        c.conv2d_synth_fill(self.x, self.x.numel(), synth.stream_key(synth.SEED, layer_id, synth.ROLE_INPUT), 0, 0)
        self.w = torch.empty(l.window * l.window * l.channels * l.features, device="cuda")
        c.conv2d_synth_fill(self.w, self.w.numel(), synth.stream_key(synth.SEED, layer_id, synth.ROLE_FILTER), 0, 0)
        self._xh = None

    def params(self, math, batch=None):
        return C().Params(**self.l.params(batch or self.batch), math=math)

    def host_inputs(self):
        if self._xh is None:
            l = self.l
            self._xh = (self.x.view(self.batch, l.rows, l.cols, l.channels).cpu().numpy(),
                        self.w.view(l.window, l.window, l.channels, l.features).cpu().numpy())
        return self._xh


def _sample_idx(seed, n, ho, wo, f, count=1000):
    rng = np.random.default_rng(seed)
    idx = np.stack([rng.integers(0, n, count), rng.integers(0, ho, count), rng.integers(0, wo, count),
                    rng.integers(0, f, count)], axis=1)
    edge = [[0, 0, 0, k] for k in range(f)] + [[n - 1, ho - 1, wo - 1, k] for k in range(f)]
    return np.concatenate([idx, np.array(edge)], axis=0).astype(np.int64)


def _oracle_points(case, p, idx):
    xh, wh = case.host_inputs()
    l = case.l
    op = O.Params(p.batch, l.rows, l.cols, l.channels, l.features, l.window, l.window, l.stride, l.stride, O.SAME)
    return O.conv2d_points(op, xh, wh, idx)


def _gather(y, shape, idx):
    import torch
    n, ho, wo, f = shape
    flat = ((idx[:, 0] * ho + idx[:, 1]) * wo + idx[:, 2]) * f + idx[:, 3]
    return y[torch.from_numpy(flat).cuda()].cpu().numpy().astype(np.float64)


def _forward(p, algo, x, w, y):
    import torch
    c = C()
    need = c.conv2d_query_workspace(p, algo)
    ws = torch.empty(max(need, 16), dtype=torch.uint8, device="cuda")
    y.fill_(float("nan"))
    c.conv2d_forward(p, algo, x, w, y, ws, ws.numel())
    torch.cuda.synchronize()


def _check_every_algo(case, what):
    import torch
    c = C()
    errs = {}
    for math in MATHS:
        p = case.params(math)
        shape, _ = c.conv2d_output_shape(p)
        y = torch.empty(int(np.prod(shape)), device="cuda")
        idx = _sample_idx(case.layer_id, *shape)
        ref, den = _oracle_points(case, p, idx)
        for a in range(1, c.NUM_ALGOS):
            if not c.conv2d_supports(p, a):
                continue
            _forward(p, a, case.x, case.w, y)
            assert bool(torch.isfinite(y).all()), f"{what} {c.ALGO_NAMES[a]} math={math}: unwritten/non-finite"
            e = float(np.max(np.abs(_gather(y, shape, idx) - ref) / den))
            record_err(f"{what} math={math}", a, math, e, len(idx))
            tol = min(tol_for(a, math), ceiling_for(a, math))
            assert e <= tol, f"{what} {c.ALGO_NAMES[a]} math={math}: err {e:.3e} > {tol}"
            errs[(c.ALGO_NAMES[a], math)] = e
    return errs


@pytest.mark.parametrize("layer_id,layer", VGG, ids=[l.name for _, l in VGG])
def test_vgg16_b32_every_algorithm_both_modes(cuda_ok, layer_id, layer):
    _check_every_algo(Case(layer_id, layer, 32), f"{layer.name} b32")


@pytest.mark.parametrize("layer_id,layer", STACK, ids=[l.name for _, l in STACK])
def test_stack_b32_every_algorithm_both_modes(cuda_ok, layer_id, layer):
    _check_every_algo(Case(layer_id, layer, 32), f"{layer.name} b32")


@pytest.mark.parametrize("layer_id,layer", STACK, ids=[l.name for _, l in STACK])
def test_stack_b256_tf32_auto(cuda_ok, layer_id, layer):
    import torch
    c = C()
    case = Case(layer_id, layer, 256)
    p = case.params(1)
    shape, _ = c.conv2d_output_shape(p)
    y = torch.empty(int(np.prod(shape)), device="cuda")
    need = c.conv2d_query_workspace(p, c.ALGO_AUTO)
    ws = torch.empty(max(need, 16), dtype=torch.uint8, device="cuda")
    algo = c.conv2d_autotune(p, case.x, case.w, y, ws, ws.numel())
    _forward(p, c.ALGO_AUTO, case.x, case.w, y)
    idx = _sample_idx(layer_id + 1, *shape)
    ref, den = _oracle_points(case, p, idx)
    e = float(np.max(np.abs(_gather(y, shape, idx) - ref) / den))
    record_err(f"{layer.name} b256 auto", algo, 1, e, len(idx))
    assert e <= min(TOL_TF32, ceiling_for(algo, 1)), f"{layer.name} b256 tf32 auto={c.ALGO_NAMES[algo]}: err {e:.3e}"


@pytest.mark.parametrize("layer_id,layer", STACK, ids=[l.name for _, l in STACK])
def test_stack_b32_shards_of_b256(cuda_ok, layer_id, layer):
    """P11 at size, in the configuration the 8-GPU bench runs (batch-32 shards of the global batch 256)."""
    import torch
    c = C()
    case = Case(layer_id, layer, 256)
    p = case.params(0)
    shape, _ = c.conv2d_output_shape(p)
    y = torch.empty(int(np.prod(shape)), device="cuda")
    need = c.conv2d_query_workspace(p, c.ALGO_AUTO)
    ws = torch.empty(max(need, 16), dtype=torch.uint8, device="cuda")
    algo = c.conv2d_autotune(p, case.x, case.w, y, ws, ws.numel())
    _forward(p, algo, case.x, case.w, y)
    gemm_like = algo in (c.ALGO_IMPLICIT_GEMM, c.ALGO_MATMUL_1X1)
    ps = case.params(0, batch=32)
    if gemm_like:  # pin the b256 variant where the b32 plan enumerates it (else the default)
        try:
            c.conv2d_set_variant(ps, algo, c.conv2d_get_variant(p, algo))
        except c.Conv2dError:
            c.conv2d_set_variant(ps, algo, 0)
    s_full, s_shard = c.conv2d_debug_splits(p, algo), c.conv2d_debug_splits(ps, algo)
    (n, ho, wo, f) = shape
    per_in, per_out = layer.rows * layer.cols * layer.channels, ho * wo * f
    ys = torch.empty(32 * per_out, device="cuda")
    for r in range(8):
        _forward(ps, algo, case.x[r * 32 * per_in:(r + 1) * 32 * per_in], case.w, ys)
        full = y[r * 32 * per_out:(r + 1) * 32 * per_out]
        if s_full == 1 and s_shard == 1:
            assert torch.equal(ys, full), f"{layer.name} shard {r} ({c.ALGO_NAMES[algo]}): not bitwise equal"
        else:
            d = (ys.double() - full.double()).abs()
            # both sides are tolerance-equal to the oracle; their difference is bounded by twice that
            idx = _sample_idx(layer_id + 10 + r, 32, ho, wo, f, 300)
            idx_g = idx.copy()
            idx_g[:, 0] += 32 * r
            ref, den = _oracle_points(case, p, idx_g)
            e = float(np.max(np.abs(_gather(ys, (32, ho, wo, f), idx) - ref) / den))
            assert e <= TOL_FP32, f"{layer.name} shard {r} splits {s_full}/{s_shard}: err {e:.3e}"
            assert bool(torch.isfinite(d).all())
