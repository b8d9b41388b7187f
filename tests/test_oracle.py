"""Pins for the CPU oracle (oracle/) against things other than itself.

Every test here runs without a GPU.  Each pin cites where its expected value
comes from (tests/golden/*.json hold the fixtures with citations):

* closed-form shapes / flops        -- SPEC.md:48-65, SURVEY.md Appendix A
* hand cases                        -- SPEC.md:123-125, 255, 265
* config-1 closed forms             -- SURVEY.md §8(c) P4 (tap counting)
* SAME-split discriminator          -- SURVEY.md §8(c) P5 (reading R3)
* golden integer fixture            -- SURVEY.md §8(c) P6
* library routine                   -- torch float64 conv2d after explicit F.pad (P8)
* 1x1 s1 = matrix product           -- numpy float64 matmul (P8)
* brute force                       -- pure-Python loops over the definition, tiny inputs
* invariants                        -- linearity, batch independence, translation

A plausible bug in the oracle -- swapped pad split, transposed filter index,
flipped kernel, wrong stride, dropped tap, single-precision accumulation --
fails at least one of these (see the per-test notes).
"""
import json
import os

import numpy as np
import pytest

import oracle as O
from paper_1904_04174_b200 import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def _pad(s):
    return O.SAME if s == "SAME" else O.VALID


# ---------------------------------------------------------------- shapes / flops
def test_spec_output_shape_examples():
    g = _gold("spec_examples.json")
    for e in g["output_shape"]:
        n, h, w, c = e["in"]
        p = O.Params(n, h, w, c, e["F"], e["K"], e["K"], e["S"], e["S"], _pad(e["padding"]))
        assert list(O.output_shape(p)[0]) == e["out"], e["cite"]


def test_spec_flop_examples_and_linearity_in_batch():
    g = _gold("spec_examples.json")
    for e in g["flop_count"]:
        n, h, w, c = e["in"]
        p = O.Params(n, h, w, c, e["F"], e["K"], e["K"], e["S"], e["S"], _pad(e["padding"]))
        assert O.flop_count(p) == e["flops"], e["cite"]
        p32 = O.Params(32, h, w, c, e["F"], e["K"], e["K"], e["S"], e["S"], _pad(e["padding"]))
        assert O.flop_count(p32) == 32 * e["flops"]  # SPEC.md:88 linear in batch


def test_paper_shapes_appendix_a():
    g = _gold("paper_shapes.json")
    assert len(g["layers"]) == 35
    for e in g["layers"]:
        p = O.Params(1, e["H"], e["W"], e["C"], e["F"], e["K"], e["K"], e["S"], e["S"], O.SAME)
        shp, pads = O.output_shape(p)
        assert shp == (1, e["out"], e["out"], e["F"]), e["name"]
        assert list(pads) == e["pads_tblr"], e["name"]
        assert round(O.flop_count(p) / 1e9, 3) == pytest.approx(e["gflop_b1"], abs=1.5e-3), e["name"]


def test_invalid_params_rejected():
    with pytest.raises(ValueError):
        O.output_shape(O.Params(1, 2, 2, 1, 1, 3, 3, 1, 1, O.VALID))  # VALID with K > H
    for bad in [O.Params(0, 4, 4, 1, 1, 1, 1), O.Params(1, 4, 4, 0, 1, 1, 1), O.Params(1, 4, 4, 1, 0, 1, 1),
                O.Params(1, 4, 4, 1, 1, 1, 1, 0, 1), O.Params(1, 4, 4, 1, 1, 1, 1, 1, 1, 7)]:
        with pytest.raises(ValueError):
            O.output_shape(bad)


def test_valid_shape_closed_form_bruteforce():
    # VALID: number of window placements counted one by one (floor((H-K)/S)+1)
    for h in range(1, 12):
        for k in range(1, h + 1):
            for s in range(1, 4):
                cnt = sum(1 for start in range(0, h) if start % s == 0 and start + k <= h)
                p = O.Params(1, h, h, 1, 1, k, k, s, s, O.VALID)
                assert O.output_shape(p)[0][1] == cnt


def test_same_shape_closed_form_bruteforce():
    # SAME: Ho = number of stride steps covering the input = ceil(H/S); total pad makes the
    # last window end exactly at (Ho-1)*S+K, split floor/ceil (reading R3)
    for h in range(1, 12):
        for k in (1, 2, 3, 5, 7):
            for s in (1, 2, 3):
                p = O.Params(1, h, h, 1, 1, k, k, s, s, O.SAME)
                (n, ho, wo, f), (pt, pb, pl, pr) = O.output_shape(p)
                assert ho == len(range(0, h, s))
                assert pt + h + pb >= (ho - 1) * s + k
                assert pt + pb == max((ho - 1) * s + k - h, 0) and pt == (pt + pb) // 2


# ---------------------------------------------------------------- hand cases
def test_hand_cases_spec():
    g = _gold("spec_examples.json")
    # all-ones 2x2 Valid -> 4
    p = O.Params(1, 2, 2, 1, 1, 2, 2, 1, 1, O.VALID)
    y = O.conv2d(p, np.ones((1, 2, 2, 1), np.float32), np.ones((2, 2, 1, 1), np.float32))
    assert y.shape == (1, 1, 1, 1) and y[0, 0, 0, 0] == g["all_ones_valid_2x2"]["value"]
    # zero filter -> 0
    x = synth.input_nhwc(2, 7, 5, 3, layer_id=11)
    p = O.Params(2, 7, 5, 3, 4, 3, 3, 1, 1, O.SAME)
    assert np.all(O.conv2d(p, x, np.zeros((3, 3, 3, 4), np.float32)) == 0)
    # centre-tap delta -> identity, per channel
    w = np.zeros((3, 3, 3, 3), np.float32)
    for c in range(3):
        w[1, 1, c, c] = 1
    p = O.Params(2, 7, 5, 3, 3, 3, 3, 1, 1, O.SAME)
    assert np.array_equal(O.conv2d(p, x, w), x)
    # identity 1x1 filter -> identity
    p = O.Params(2, 7, 5, 3, 3, 1, 1, 1, 1, O.SAME)
    assert np.array_equal(O.conv2d(p, x, np.eye(3, dtype=np.float32).reshape(1, 1, 3, 3)), x)


def test_off_centre_delta_is_a_shift():
    # a delta at tap (kh,kw) must read x[h+kh-pt, w+kw-pl] -- catches a flipped kernel (convolution
    # instead of correlation, reading R2) and swapped kh/kw filter indexing
    x = synth.input_nhwc(1, 6, 7, 1, layer_id=12)
    p = O.Params(1, 6, 7, 1, 1, 3, 3, 1, 1, O.SAME)
    for kh in range(3):
        for kw in range(3):
            w = np.zeros((3, 3, 1, 1), np.float32)
            w[kh, kw, 0, 0] = 1
            y = O.conv2d(p, x, w)[0, :, :, 0]
            for h in range(6):
                for ww in range(7):
                    ih, iw = h + kh - 1, ww + kw - 1
                    exp = x[0, ih, iw, 0] if 0 <= ih < 6 and 0 <= iw < 7 else 0
                    assert y[h, ww] == exp


def test_config1_closed_forms():
    g = _gold("config1_closed_forms.json")
    p = O.Params(1, 8, 8, 4, 8, 3, 3, 1, 1, O.SAME)
    y = O.conv2d(p, np.ones((1, 8, 8, 4), np.float32), np.ones((3, 3, 4, 8), np.float32))
    for f in range(8):
        assert y[0, 0, 0, f] == g["all_ones"]["corner"] and y[0, 7, 7, f] == g["all_ones"]["corner"]
        assert y[0, 0, 3, f] == g["all_ones"]["edge"] and y[0, 4, 7, f] == g["all_ones"]["edge"]
        assert y[0, 3, 3, f] == g["all_ones"]["interior"]
    ramp = np.broadcast_to(np.arange(8, dtype=np.float32).reshape(1, 8, 1, 1), (1, 8, 8, 4)).copy()
    y = O.conv2d(p, ramp, np.ones((3, 3, 4, 8), np.float32))
    assert list(y[0, :, 3, 0]) == g["ramp_h"]["col3"]
    assert list(y[0, :, 0, 0]) == g["ramp_h"]["col0"]


def test_same_pad_discriminator():
    g = _gold("same_pad_discriminator.json")
    for cs in g["cases"]:
        k, s, h, c = cs["K"], cs["S"], cs["H"], cs["C"]
        p = O.Params(1, h, h, c, 1, k, k, s, s, O.SAME)
        y = O.conv2d(p, np.ones((1, h, h, c), np.float32), np.ones((k, k, c, 1), np.float32))
        for (ho, wo, v) in cs["points"]:
            assert y[0, ho, wo, 0] == v


def test_golden_integer_config1():
    g = _gold("config1_integer.json")
    x = np.array([[[[((h * 8 + w) * 4 + c) % 7 - 3 for c in range(4)] for w in range(8)] for h in range(8)]],
                 dtype=np.float32)
    wt = np.array([[[[(((kh * 3 + kw) * 4 + c) * 8 + f) % 5 - 2 for f in range(8)] for c in range(4)]
                    for kw in range(3)] for kh in range(3)], dtype=np.float32)
    for key in ("same_s1", "valid_s1", "same_s2"):
        e = g[key]
        p = O.Params(1, 8, 8, 4, 8, 3, 3, e["stride"], e["stride"], _pad(e["padding"]))
        y = O.conv2d(p, x, wt)
        assert list(y.shape) == e["shape"]
        for (n, a, b, f, v) in e["points"]:
            assert y[n, a, b, f] == v
        assert y.sum() == e["sum"]
        if "abs_sum" in e:
            assert np.abs(y).sum() == e["abs_sum"]
        if "pads" in e:
            assert list(O.output_shape(p)[1]) == e["pads"]


# ---------------------------------------------------------------- library routines / brute force
def _torch_ref(p, x, w):
    """torch.nn.functional.conv2d in float64 after an explicit asymmetric F.pad (P8)."""
    import torch
    import torch.nn.functional as F
    xt = torch.from_numpy(x.astype(np.float64)).permute(0, 3, 1, 2)
    wt = torch.from_numpy(w.astype(np.float64)).permute(3, 2, 0, 1)
    if p.padding == O.SAME:
        # pad totals from first principles: the last window must end at (Ho-1)*S+K
        ho = -(-p.in_rows // p.stride_rows)
        wo = -(-p.in_cols // p.stride_cols)
        tr = max((ho - 1) * p.stride_rows + p.window_rows - p.in_rows, 0)
        tc = max((wo - 1) * p.stride_cols + p.window_cols - p.in_cols, 0)
        xt = F.pad(xt, (tc // 2, tc - tc // 2, tr // 2, tr - tr // 2))
    y = F.conv2d(xt, wt, stride=(p.stride_rows, p.stride_cols))
    return y.permute(0, 2, 3, 1).numpy()


@pytest.mark.parametrize("case", [
    (2, 9, 11, 5, 6, 3, 3, 1, 1, O.SAME), (1, 10, 10, 3, 4, 7, 7, 2, 2, O.SAME),
    (3, 8, 7, 2, 3, 5, 5, 2, 1, O.SAME), (1, 9, 9, 4, 5, 3, 3, 2, 2, O.VALID),
    (2, 6, 13, 3, 2, 1, 1, 2, 2, O.SAME), (1, 12, 12, 8, 8, 5, 3, 1, 2, O.VALID),
    (1, 5, 5, 1, 1, 7, 7, 1, 1, O.SAME), (2, 15, 9, 6, 7, 2, 4, 3, 2, O.SAME),
])
def test_matches_torch_float64(case):
    p = O.Params(*case)
    x = synth.input_nhwc(p.batch, p.in_rows, p.in_cols, p.channels, layer_id=21)
    w = synth.filter_hwcf(p.window_rows, p.window_cols, p.channels, p.features, layer_id=21)
    y, d = O.conv2d(p, x, w, with_denom=True)
    ref = _torch_ref(p, x, w)
    assert y.shape == ref.shape
    # oracle = double sum rounded once; torch float64 differs only in summation order (~1e-15 rel)
    assert np.all(np.abs(y.astype(np.float64) - ref) <= 0.5 * np.spacing(np.abs(ref).astype(np.float32)) + 1e-12 * d)


def test_1x1_equals_float64_matmul():
    p = O.Params(2, 6, 5, 16, 12, 1, 1, 1, 1, O.SAME)
    x = synth.input_nhwc(2, 6, 5, 16, layer_id=22)
    w = synth.filter_hwcf(1, 1, 16, 12, layer_id=22)
    y = O.conv2d(p, x, w)
    ref = (x.reshape(-1, 16).astype(np.float64) @ w.reshape(16, 12).astype(np.float64)).astype(np.float32)
    assert np.array_equal(y.reshape(-1, 12), ref)


def test_bruteforce_python_definition():
    p = O.Params(2, 5, 4, 3, 2, 3, 2, 2, 1, O.SAME)
    x = synth.input_nhwc(2, 5, 4, 3, layer_id=23)
    w = synth.filter_hwcf(3, 2, 3, 2, layer_id=23)
    y, d = O.conv2d(p, x, w, with_denom=True)
    (N, HO, WO, F), (pt, pb, pl, pr) = O.output_shape(p)
    for n in range(N):
        for ho in range(HO):
            for wo in range(WO):
                for f in range(F):
                    s = 0.0
                    a = 0.0
                    for kh in range(3):
                        for kw in range(2):
                            for c in range(3):
                                ih, iw = ho * 2 + kh - pt, wo * 1 + kw - pl
                                if 0 <= ih < 5 and 0 <= iw < 4:
                                    t = float(x[n, ih, iw, c]) * float(w[kh, kw, c, f])
                                    s += t
                                    a += abs(t)
                    assert abs(float(y[n, ho, wo, f]) - s) <= 1e-7 * a
                    assert d[n, ho, wo, f] == pytest.approx(a, rel=1e-14)


def test_points_match_full():
    p = O.Params(2, 9, 8, 5, 7, 3, 3, 2, 2, O.SAME)
    x = synth.input_nhwc(2, 9, 8, 5, layer_id=24)
    w = synth.filter_hwcf(3, 3, 5, 7, layer_id=24)
    y, d = O.conv2d(p, x, w, with_denom=True)
    idx = np.array([[n, a, b, f] for n in range(2) for a in range(5) for b in range(4) for f in range(7)])
    yp, dp = O.conv2d_points(p, x, w, idx)
    assert np.array_equal(yp.astype(np.float32), y.reshape(-1))
    assert np.allclose(dp, d.reshape(-1), rtol=1e-15, atol=0)
    with pytest.raises(ValueError):
        O.conv2d_points(p, x, w, np.array([[0, 5, 0, 0]]))


# ---------------------------------------------------------------- invariants
def test_double_accumulation_is_exact_on_cancellation():
    # sum of 1 + 2^-30 ... - 1 : float32 accumulation would lose the small term; double keeps it
    c = 3
    x = np.array([1.0, 2.0 ** -30, -1.0], np.float32).reshape(1, 1, 1, c)
    w = np.ones((1, 1, c, 1), np.float32)
    y = O.conv2d(O.Params(1, 1, 1, c, 1, 1, 1), x, w)
    assert y[0, 0, 0, 0] == np.float32(2.0 ** -30)


def test_linearity_batch_independence_translation():
    p = O.Params(3, 10, 9, 4, 5, 3, 3, 1, 1, O.VALID)
    x = synth.input_nhwc(3, 10, 9, 4, layer_id=25, dist=synth.DIST_INT5)
    w = synth.filter_hwcf(3, 3, 4, 5, layer_id=25, dist=synth.DIST_INT5)
    y = O.conv2d(p, x, w)
    # linearity (integer data: exact): conv(2x) = 2 conv(x); conv(x, w1+w2) = conv(x,w1)+conv(x,w2)
    assert np.array_equal(O.conv2d(p, 2 * x, w), 2 * y)
    w2 = synth.filter_hwcf(3, 3, 4, 5, layer_id=26, dist=synth.DIST_INT5)
    assert np.array_equal(O.conv2d(p, x, w + w2), y + O.conv2d(p, x, w2))
    # batch independence: each image alone gives its slice
    for n in range(3):
        pn = O.Params(1, 10, 9, 4, 5, 3, 3, 1, 1, O.VALID)
        assert np.array_equal(O.conv2d(pn, x[n:n + 1], w), y[n:n + 1])
    # translation on VALID: shifting the input by one row shifts the output
    pt = O.Params(3, 9, 9, 4, 5, 3, 3, 1, 1, O.VALID)
    assert np.array_equal(O.conv2d(pt, x[:, 1:], w), y[:, 1:])


def test_normalized_error_metric():
    y = np.array([1.0, 0.0, 2.0])
    assert O.normalized_error(y, y, np.array([1.0, 0.0, 1.0])) == 0.0
    assert O.normalized_error(y + np.array([1e-6, 0, 0]), y, np.array([10.0, 0.0, 1.0])) == pytest.approx(1e-7)
    assert O.normalized_error(np.array([0.0, 1e-30]), np.array([0.0, 0.0]), np.array([1.0, 0.0])) == float("inf")


def test_golden_config1_regenerates_from_its_generator():
    """The committed P6 fixture is what tools/gen_golden_config1.py derives (torch float64 + pure-Python brute
    force, neither touching oracle/ nor the CUDA path)."""
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "gen_golden_config1", os.path.join(os.path.dirname(GOLD), "..", "tools", "gen_golden_config1.py"))
    gen = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(gen)
    fresh = gen.generate()
    committed = _gold("config1_integer.json")
    for key in ("same_s1", "valid_s1", "same_s2"):
        assert fresh[key] == committed[key], key
