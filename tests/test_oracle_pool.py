"""Pins of the pooling oracle (oracle/pool.c) against things other than itself:
SPEC.md's worked examples, the identity / constant invariants, the in-window membership of every
max, and torch's float64 library pooling after an explicit asymmetric pad (a different computation:
-inf padding for max; window sums and in-bounds counts as two avg_pool2d passes for the average)."""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

import oracle as O

MAX, AVG = O.POOL_MAX, O.POOL_AVG


def P(n, h, w, c, kh, kw, sh, sw, pad, op):
    return O.PoolParams(n, h, w, c, kh, kw, sh, sw, pad, op)


def test_spec_examples():
    # SPEC.md:374 / 383: [[1,2],[3,4]], window 2, stride 2, VALID -> max [[4]], avg [[2.5]]
    x = np.array([1, 2, 3, 4], np.float32).reshape(1, 2, 2, 1)
    assert O.pool2d(P(1, 2, 2, 1, 2, 2, 2, 2, O.VALID, MAX), x).ravel().tolist() == [4.0]
    assert O.pool2d(P(1, 2, 2, 1, 2, 2, 2, 2, O.VALID, AVG), x).ravel().tolist() == [2.5]


@pytest.mark.parametrize("op", [MAX, AVG])
@pytest.mark.parametrize("pad", [O.SAME, O.VALID])
def test_window1_is_identity(op, pad):
    x = np.random.default_rng(0).standard_normal((2, 5, 7, 3)).astype(np.float32)
    assert np.array_equal(O.pool2d(P(2, 5, 7, 3, 1, 1, 1, 1, pad, op), x), x)


@pytest.mark.parametrize("op", [MAX, AVG])
@pytest.mark.parametrize("shape", [(1, 7, 7, 2, 3, 3, 2, 2, O.SAME), (2, 6, 9, 3, 5, 4, 1, 3, O.SAME),
                                   (1, 8, 8, 1, 2, 2, 2, 2, O.VALID), (1, 5, 5, 4, 5, 5, 1, 1, O.SAME)])
def test_constant_input_gives_constant(op, shape):
    # SPEC.md:386 "Same-padded corner of a constant input -> that constant (in-bounds divisor)"
    n, h, w, c, kh, kw, sh, sw, pad = shape
    x = np.full((n, h, w, c), 0.7, np.float32)
    y = O.pool2d(P(n, h, w, c, kh, kw, sh, sw, pad, op), x)
    assert np.all(y == np.float32(0.7))


def _torch_ref(x, p):
    """float64 torch pooling with the SAME pads applied explicitly (SPEC.md:48-56 split)."""
    (_, ho, wo, _), (pt, pb, pl, pr) = O.pool_output_shape(p)
    t = torch.from_numpy(x.astype(np.float64)).permute(0, 3, 1, 2)
    k, s = (p.window_rows, p.window_cols), (p.stride_rows, p.stride_cols)
    if p.op == MAX:
        tp = F.pad(t, (pl, pr, pt, pb), value=float("-inf"))
        y = F.max_pool2d(tp, k, s)
    else:
        ones = torch.ones_like(t)
        tp = F.pad(t, (pl, pr, pt, pb), value=0.0)
        op_ = F.pad(ones, (pl, pr, pt, pb), value=0.0)
        y = F.avg_pool2d(tp, k, s) / F.avg_pool2d(op_, k, s)  # sum / in-bounds count
    y = y[:, :, :ho, :wo].permute(0, 2, 3, 1).numpy()
    return y


CASES = [(2, 13, 11, 5, 3, 3, 2, 2, O.SAME), (1, 112, 112, 8, 3, 3, 2, 2, O.SAME),  # ResNet stem pool
         (3, 14, 14, 4, 2, 2, 2, 2, O.VALID), (1, 9, 10, 3, 4, 2, 3, 1, O.SAME),
         (2, 7, 7, 16, 7, 7, 1, 1, O.VALID), (1, 17, 5, 2, 5, 3, 2, 2, O.SAME), (1, 6, 6, 1, 1, 1, 2, 2, O.SAME)]


@pytest.mark.parametrize("case", CASES, ids=str)
@pytest.mark.parametrize("op", [MAX, AVG])
def test_matches_torch_float64(case, op):
    n, h, w, c, kh, kw, sh, sw, pad = case
    p = P(n, h, w, c, kh, kw, sh, sw, pad, op)
    x = np.random.default_rng(hash(case) % 2**32).uniform(-1, 1, (n, h, w, c)).astype(np.float32)
    y = O.pool2d(p, x)
    ref = _torch_ref(x, p)
    assert y.shape == ref.shape
    if op == MAX:
        assert np.array_equal(y, ref.astype(np.float32))
    else:
        # the oracle's average is the correctly rounded fp32 of the exact mean: within half an fp32 ulp
        # of the float64 library value (whose own error is ~1e-16 relative)
        half_ulp = 0.5 * np.spacing(np.abs(y).astype(np.float32)).astype(np.float64)
        assert np.all(np.abs(y.astype(np.float64) - ref) <= half_ulp + 1e-15 * np.abs(ref)), np.abs(y - ref).max()


@pytest.mark.parametrize("case", CASES[:4], ids=str)
def test_max_is_a_window_element(case):
    n, h, w, c, kh, kw, sh, sw, pad = case
    p = P(n, h, w, c, kh, kw, sh, sw, pad, MAX)
    x = np.random.default_rng(3).uniform(-1, 1, (n, h, w, c)).astype(np.float32)
    y = O.pool2d(p, x)
    _, (pt, _, pl, _) = O.pool_output_shape(p)
    for (b, i, j, ch) in [(0, 0, 0, 0), (n - 1, y.shape[1] - 1, y.shape[2] - 1, c - 1), (0, y.shape[1] // 2, 1, c // 2)]:
        win = [x[b, i * sh + a - pt, j * sw + e - pl, ch] for a in range(kh) for e in range(kw)
               if 0 <= i * sh + a - pt < h and 0 <= j * sw + e - pl < w]
        assert y[b, i, j, ch] in win and y[b, i, j, ch] == max(win)


def test_shapes_follow_the_conv_algebra_and_reject_valid_overflow():
    for case in CASES:
        n, h, w, c, kh, kw, sh, sw, pad = case
        (pn, ph, pw, pc), pads = O.pool_output_shape(P(n, h, w, c, kh, kw, sh, sw, pad, MAX))
        (cn, ch, cw, cf), cpads = O.output_shape(O.Params(n, h, w, c, c, kh, kw, sh, sw, pad))
        assert (pn, ph, pw, pc, pads) == (cn, ch, cw, cf, cpads)
    with pytest.raises(ValueError):
        O.pool_output_shape(P(1, 4, 4, 1, 5, 5, 1, 1, O.VALID, MAX))
    with pytest.raises(ValueError):
        O.pool_output_shape(P(1, 4, 4, 1, 2, 2, 1, 1, O.SAME, 7))
