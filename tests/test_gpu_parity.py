"""GPU parity: every algorithm x math mode of libconv2d.so (called through the C-ABI)
against the CPU oracle on the same seeded inputs (north_star tolerance:
max|err| / sum|x||w| <= 1e-5 for fp32 and 3xTF32, <= 2e-3 for TF32; shapes bit-exact).
"""
import json
import os

import numpy as np
import pytest

import oracle as O
from paper_1904_04174_b200 import layers as L
from paper_1904_04174_b200 import synth

from .parity import C, assert_int_exact, check_close, gpu_conv, make_inputs, oparams, supported_algos

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")
MATHS = (0, 1)  # FP32 (3xTF32 on tensor paths), TF32


def P(batch, h, w, c, f, kh, kw, sh=1, sw=1, pad=0, math=0):
    return C().Params(batch, h, w, c, f, kh, kw, sh, sw, pad, math)


def test_config1_golden_integer_all_algos(cuda_ok):
    g = json.load(open(os.path.join(GOLD, "config1_integer.json")))
    x = np.array([[[[((h * 8 + w) * 4 + c) % 7 - 3 for c in range(4)] for w in range(8)] for h in range(8)]],
                 dtype=np.float32)
    wt = np.array([[[[(((kh * 3 + kw) * 4 + c) * 8 + f) % 5 - 2 for f in range(8)] for c in range(4)]
                    for kw in range(3)] for kh in range(3)], dtype=np.float32)
    for key in ("same_s1", "valid_s1", "same_s2"):
        e = g[key]
        for math in MATHS:
            p = P(1, 8, 8, 4, 8, 3, 3, e["stride"], e["stride"], 0 if e["padding"] == "SAME" else 1, math)
            ref = O.conv2d(oparams(p), x, wt)
            for a in supported_algos(p):
                y = gpu_conv(p, x, wt, a)
                assert list(y.shape) == e["shape"]
                assert np.array_equal(y, ref), (key, math, C().conv2d_algo_name(a))
                for (n, i, j, f, v) in e["points"]:
                    assert y[n, i, j, f] == v
                assert y.sum() == e["sum"]


ALL_SHAPES = [l for l in L.RESNET50_SETS] + [l for l, _ in L.VGG16_LAYERS]


@pytest.mark.parametrize("layer", ALL_SHAPES, ids=lambda l: l.name)
def test_exact_integer_regime_b1(cuda_ok, layer):
    """P7: integer data in [-2,2] makes every partial sum exact -> every algorithm bit-exact (F(4x4):
    tolerance, reading R21)."""
    p0 = C().Params(**layer.params(1))
    x, w = make_inputs(p0, layer_id=100, dist=synth.DIST_INT5)
    ref, den = O.conv2d(oparams(p0), x, w, with_denom=True)
    for math in MATHS:
        p = p0.replace(math=math)
        for a in supported_algos(p):
            y = gpu_conv(p, x, w, a)
            assert_int_exact(p, y, ref, den, a, f"{layer.name} math={math} {C().conv2d_algo_name(a)}")


@pytest.mark.parametrize("layer", ALL_SHAPES, ids=lambda l: l.name)
def test_uniform_paper_shapes_b1(cuda_ok, layer):
    p0 = C().Params(**layer.params(1))
    x, w = make_inputs(p0, layer_id=200)
    ref, den = O.conv2d(oparams(p0), x, w, with_denom=True)
    for math in MATHS:
        p = p0.replace(math=math)
        for a in supported_algos(p):
            check_close(p, gpu_conv(p, x, w, a), ref, den, a, f"{layer.name} math={math} {C().conv2d_algo_name(a)}")


def _fuzz_cases(n=200, seed=1234):
    # SPEC.md:278 / 534: spatial 1..20, C,F 1..32, K in {1,3,5,7}, S in {1,2}, both paddings, batch 1..3
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < n:
        k = int(rng.choice([1, 3, 5, 7]))
        h, w = int(rng.integers(1, 21)), int(rng.integers(1, 21))
        pad = int(rng.integers(0, 2))
        if pad == 1 and (k > h or k > w):
            continue
        out.append((int(rng.integers(1, 4)), h, w, int(rng.integers(1, 33)), int(rng.integers(1, 33)), k, k,
                    int(rng.integers(1, 3)), int(rng.integers(1, 3)), pad))
    return out


def test_spec_fuzz_200(cuda_ok):
    for i, case in enumerate(_fuzz_cases()):
        p0 = P(*case)
        x, w = make_inputs(p0, layer_id=300 + i)
        ref, den = O.conv2d(oparams(p0), x, w, with_denom=True)
        for math in MATHS:
            p = p0.replace(math=math)
            for a in supported_algos(p):
                check_close(p, gpu_conv(p, x, w, a), ref, den, a, f"fuzz {case} math={math} {C().conv2d_algo_name(a)}")


EDGE = [
    (1, 1, 1, 1, 1, 1, 1, 1, 1, 0),          # single element
    (1, 1, 1, 7, 5, 3, 3, 1, 1, 0),          # window larger than image, SAME
    (2, 3, 2, 3, 9, 7, 7, 2, 2, 0),          # 7x7 s2 on tiny input
    (1, 9, 7, 40, 33, 3, 3, 1, 1, 0),        # odd Ho/Wo Winograd tiles, F%4 != 0
    (3, 15, 9, 64, 70, 3, 3, 1, 1, 1),       # VALID Winograd, ragged N
    (1, 33, 35, 1, 1, 5, 5, 1, 1, 0),        # C=1, F=1
    (1, 13, 11, 5, 130, 3, 3, 2, 1, 0),      # C%4 != 0 scalar gather, ragged N tile
    (2, 7, 7, 2048, 64, 1, 1, 1, 1, 0),      # deep K, split-K
    (1, 7, 7, 512, 512, 3, 3, 1, 1, 0),      # R24 b1: split-K winograd + igemm
    (64, 2, 2, 32, 16, 1, 1, 1, 1, 0),       # many images, tiny spatial
    (1, 20, 20, 96, 257, 1, 1, 1, 1, 0),     # F = 257 (one past a tile)
    (2, 17, 19, 36, 24, 2, 4, 3, 2, 0),      # non-square window / stride
    (1, 130, 3, 8, 8, 3, 3, 1, 1, 0),        # M just over one 128-row tile per image row sweep
    # halo-tile path (3x3 s1, C % 32 == 0, F <= 128): odd CTA-tile count, ragged spatial tiles
    (1, 9, 13, 64, 40, 3, 3, 1, 1, 0),       # 2x2 CTA tiles -> 2 pairs, F%4==0 but < BN
    (3, 17, 7, 96, 128, 3, 3, 1, 1, 1),      # VALID, 3 channel blocks, 15x5 output
    (1, 16, 8, 32, 64, 3, 3, 1, 1, 0),       # exactly one CTA tile -> one real + one dummy tile
    (2, 30, 31, 32, 66, 3, 3, 1, 1, 0),      # F=66 (F%4 != 0): direct-store epilogue
    # row-segment stem path (C < 32, KW*C4 <= 32): C=3/5/8, strides, VALID
    (2, 23, 19, 3, 64, 7, 7, 2, 2, 0),
    (1, 20, 21, 5, 24, 3, 3, 1, 2, 1),
    (3, 11, 12, 8, 16, 4, 4, 2, 1, 0),
    # direct-B path (B read from the HWCF filter as an MN-major operand, F % 32 == 0): a single 32-wide
    # n chunk (the pair's second half out of range), a ragged last chunk pair, a K tail in the dense
    # 1x1 path (C = 48), BN = 256 with a partial N tile, im2col with stride 2 and SAME corners
    (2, 9, 11, 64, 32, 1, 1, 1, 1, 0),
    (1, 12, 10, 64, 96, 3, 3, 2, 2, 0),
    (2, 10, 10, 48, 64, 1, 1, 1, 1, 0),
    (1, 6, 40, 64, 288, 1, 1, 1, 1, 0),
    (1, 15, 13, 128, 160, 3, 3, 2, 2, 0),
    # gather A path (C % 32 != 0) + 3xTF32 lo halves in TMEM (BN <= 128): each thread's lo row is gathered by
    # other threads' cp.asyncs (regression: tools/fuzz_gpu.py found the missing barrier)
    (1, 44, 43, 48, 100, 1, 1, 1, 1, 0),
    (3, 21, 26, 40, 64, 3, 3, 2, 2, 1),
    # space-to-depth stem path (K in {7, 8}, stride 2, C <= 4, F <= 128): ragged 8x16 output tiles,
    # odd image sizes, SAME corners, VALID, C = 1 / 2 / 4, K = 8, F not a multiple of 32
    (1, 37, 29, 3, 64, 7, 7, 2, 2, 0),
    (2, 40, 36, 1, 32, 7, 7, 2, 2, 1),
    (1, 33, 47, 2, 100, 8, 8, 2, 2, 0),
    (3, 20, 18, 4, 128, 7, 7, 2, 2, 0),
    (1, 64, 64, 3, 64, 8, 7, 2, 2, 1),
]


@pytest.mark.parametrize("case", EDGE, ids=str)
def test_edge_cases(cuda_ok, case):
    p0 = P(*case)
    x, w = make_inputs(p0, layer_id=400)
    ref, den = O.conv2d(oparams(p0), x, w, with_denom=True)
    xi, wi = make_inputs(p0, layer_id=401, dist=synth.DIST_INT5)
    refi, deni = O.conv2d(oparams(p0), xi, wi, with_denom=True)
    for math in MATHS:
        p = p0.replace(math=math)
        for a in supported_algos(p):
            check_close(p, gpu_conv(p, x, w, a), ref, den, a, f"edge {case} math={math} {C().conv2d_algo_name(a)}")
            assert_int_exact(p, gpu_conv(p, xi, wi, a), refi, deni, a, f"edge int {case} {math} {a}")


def test_determinism_and_shard_bitwise(cuda_ok):
    """P11: fixed (params, algo) -> bitwise identical reruns; batch slices run separately give
    the same bits as the full batch when neither launch plan splits K (conv2d_debug_splits == 1), for
    every algorithm; with a K split on either side (the split count follows the batch's tile count)
    the slices are held to the tolerance instead."""
    c = C()
    p = P(4, 28, 28, 64, 64, 3, 3)
    x, w = make_inputs(p, layer_id=500)
    for a in supported_algos(p):
        y1 = gpu_conv(p, x, w, a)
        y2 = gpu_conv(p, x, w, a)
        assert np.array_equal(y1, y2), c.conv2d_algo_name(a)
    bitwise = set()
    for case in [(8, 80, 80, 64, 64, 3, 3), (8, 80, 80, 64, 128, 1, 1), (8, 120, 120, 32, 128, 3, 3, 2, 2),
                 (8, 40, 40, 128, 128, 3, 3), (8, 7, 7, 512, 512, 3, 3), (8, 61, 57, 3, 64, 7, 7, 2, 2)]:
        for math in MATHS:
            p = P(*case, math=math)
            x, w = make_inputs(p, layer_id=501)
            ref, den = O.conv2d(oparams(p), x, w, with_denom=True)
            ph = p.replace(batch=4)
            for a in supported_algos(p):
                full = gpu_conv(p, x, w, a)
                same_plan = c.conv2d_debug_splits(p, a) == 1 and c.conv2d_debug_splits(ph, a) == 1
                for r in range(2):
                    part = gpu_conv(ph, x[4 * r:4 * r + 4], w, a)
                    if same_plan:
                        assert np.array_equal(part, full[4 * r:4 * r + 4]), (case, math, c.conv2d_algo_name(a), r)
                        bitwise.add(c.conv2d_algo_name(a))
                    else:
                        check_close(ph, part, ref[4 * r:4 * r + 4], den[4 * r:4 * r + 4], a, f"shard {case} {a}")
    # every algorithm is covered by at least one bitwise shard comparison
    assert bitwise >= {c.ALGO_NAMES[i] for i in range(1, c.NUM_ALGOS)}, bitwise


def test_autotune_and_auto_forward(cuda_ok):
    import torch
    c = C()
    c.conv2d_clear_selection_cache()
    p = P(2, 28, 28, 128, 128, 3, 3)
    x, w = make_inputs(p, layer_id=600)
    ref, den = O.conv2d(oparams(p), x, w, with_denom=True)
    xd, wd = torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda()
    y = torch.empty((2, 28, 28, 128), device="cuda")
    need = c.conv2d_query_workspace(p, c.ALGO_AUTO)
    ws = torch.empty(need, dtype=torch.uint8, device="cuda")
    a = c.conv2d_autotune(p, xd, wd, y, ws, need)
    assert a != c.ALGO_AUTO and c.conv2d_supports(p, a)
    times = c.conv2d_last_tune_times()
    assert set(times) == {c.ALGO_NAMES[i] for i in supported_algos(p)}
    assert min(times, key=lambda k: (times[k], c.ALGO_BY_NAME[k])) == c.ALGO_NAMES[a]  # argmin, ties by enum
    assert c.conv2d_selected(p) == a
    y.fill_(float("nan"))
    c.conv2d_forward(p, c.ALGO_AUTO, xd, wd, y, ws, need)
    torch.cuda.synchronize()
    check_close(p, y.cpu().numpy(), ref, den, c.ALGO_AUTO, "auto")
    # AUTO on a cache miss tunes implicitly
    p2 = p.replace(math=1)
    assert c.conv2d_selected(p2) is None
    out = c.forward(xd, wd, algo=c.ALGO_AUTO, math=1)
    check_close(p2, out.cpu().numpy(), ref, den, c.ALGO_AUTO, "auto tf32")
    assert c.conv2d_selected(p2) is not None


@pytest.mark.filterwarnings("ignore:The CUDA Graph is empty")
def test_auto_under_stream_capture(cuda_ok):
    """An AUTO cache miss inside a CUDA-graph capture is refused (tuning synchronises the stream) without
    breaking the capture; once tuned, AUTO captures and replays to the oracle's result."""
    import torch
    c = C()
    c.conv2d_clear_selection_cache()
    p = P(2, 20, 20, 64, 96, 3, 3)
    x, w = make_inputs(p, layer_id=610)
    ref, den = O.conv2d(oparams(p), x, w, with_denom=True)
    xd, wd = torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda()
    y = torch.full((2, 20, 20, 96), float("nan"), device="cuda")
    need = c.conv2d_query_workspace(p, c.ALGO_AUTO)
    ws = torch.empty(need, dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s, capture_error_mode="thread_local"):
        with pytest.raises(c.Conv2dError) as e:
            c.conv2d_forward(p, c.ALGO_AUTO, xd, wd, y, ws, need, s)
        assert e.value.status == c.ERR_UNSUPPORTED
        with pytest.raises(c.Conv2dError):
            c.conv2d_autotune(p, xd, wd, y, ws, need, s)
    assert c.conv2d_selected(p) is None
    c.conv2d_autotune(p, xd, wd, y, ws, need)  # outside the capture
    g2 = torch.cuda.CUDAGraph()
    y.fill_(float("nan"))
    torch.cuda.synchronize()
    with torch.cuda.graph(g2, stream=s, capture_error_mode="thread_local"):
        c.conv2d_forward(p, c.ALGO_AUTO, xd, wd, y, ws, need, s)
    g2.replay()
    torch.cuda.synchronize()
    check_close(p, y.cpu().numpy(), ref, den, c.ALGO_AUTO, "auto captured")


def test_auto_predict_policy_captures(cuda_ok):
    """CONV2D_AUTO_PREDICT: an AUTO cache miss takes the learned selector's choice (no timing, no sync), so
    it captures into a CUDA graph; the replay matches the oracle and the cached choice is the prediction."""
    import torch
    c = C()
    c.conv2d_clear_selection_cache()
    p = P(3, 18, 22, 64, 128, 3, 3)
    x, w = make_inputs(p, layer_id=620)
    ref, den = O.conv2d(oparams(p), x, w, with_denom=True)
    xd, wd = torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda()
    (n, ho, wo, f), _ = c.conv2d_output_shape(p)
    y = torch.full((n, ho, wo, f), float("nan"), device="cuda")
    need = c.conv2d_query_workspace(p, c.ALGO_AUTO)
    ws = torch.empty(need, dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    c.conv2d_set_auto_policy(c.AUTO_PREDICT)
    try:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s, capture_error_mode="thread_local"):
            c.conv2d_forward(p, c.ALGO_AUTO, xd, wd, y, ws, need, s)
        g.replay()
        torch.cuda.synchronize()
    finally:
        c.conv2d_set_auto_policy(c.AUTO_MEASURE)
    a, v = c.conv2d_predict(p)
    assert c.conv2d_selected(p) == a
    if a in (c.ALGO_IMPLICIT_GEMM, c.ALGO_MATMUL_1X1):
        assert c.conv2d_get_variant(p, a) == v
    check_close(p, y.cpu().numpy(), ref, den, c.ALGO_AUTO, "auto predict captured")


def test_auto_hybrid_policy_times_top_candidates(cuda_ok):
    """CONV2D_AUTO_HYBRID: conv2d_autotune times only the learned selector's top 3 candidates -- at most three
    algorithms report times, the prediction among them -- and the chosen algorithm is correct."""
    import torch
    c = C()
    c.conv2d_clear_selection_cache()
    p = P(2, 24, 24, 64, 96, 3, 3)
    x, w = make_inputs(p, layer_id=630)
    ref, den = O.conv2d(oparams(p), x, w, with_denom=True)
    xd, wd = torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda()
    (n, ho, wo, f), _ = c.conv2d_output_shape(p)
    y = torch.empty((n, ho, wo, f), device="cuda")
    need = c.conv2d_query_workspace(p, c.ALGO_AUTO)
    ws = torch.empty(need, dtype=torch.uint8, device="cuda")
    c.conv2d_set_auto_policy(c.AUTO_HYBRID)
    try:
        a = c.conv2d_autotune(p, xd, wd, y, ws, need)
        times = c.conv2d_last_tune_times()
    finally:
        c.conv2d_set_auto_policy(c.AUTO_MEASURE)
    assert 1 <= len(times) <= 3
    assert c.ALGO_NAMES[c.conv2d_predict(p)[0]] in times
    assert c.ALGO_NAMES[a] in times
    y.fill_(float("nan"))
    c.conv2d_forward(p, c.ALGO_AUTO, xd, wd, y, ws, need)
    torch.cuda.synchronize()
    check_close(p, y.cpu().numpy(), ref, den, c.ALGO_AUTO, "auto hybrid")


def test_pdl_chain_bitwise(cuda_ok):
    """Programmatic dependent launch keeps stream order: a 9-conv chain (each conv reads the previous output;
    dense, im2col, Winograd F2/F4, direct, tiled, strided paths) captured in one CUDA graph gives bit-identical
    outputs with PDL on every launch (CONV2D_PDL=1) and on none (CONV2D_PDL=0).  A kernel that touched global
    memory before griddepcontrol.wait would read a stale or half-written input here."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = {}
    for mode in ("0", "1"):
        env = dict(os.environ, CONV2D_PDL=mode)
        r = subprocess.run([sys.executable, os.path.join(root, "tests", "pdl_chain.py"), root], env=env,
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-3000:]
        out[mode] = r.stdout.split()
    assert len(out["0"]) == 9 and out["0"] == out["1"]


def test_device_synth_matches_host_generator(cuda_ok):
    import torch
    c = C()
    for dist in (0, 1):
        key = synth.stream_key(synth.SEED, 7, 0)
        d = torch.empty(100003, device="cuda")
        c.conv2d_synth_fill(d, d.numel(), key, 12345, dist)
        torch.cuda.synchronize()
        assert np.array_equal(d.cpu().numpy(), synth.draw(100003, key, 12345, dist))


def test_fault_injection_is_detected(cuda_ok):
    """P12: a single output perturbed by 1e-2 must fail the parity check."""
    p = P(1, 14, 14, 32, 32, 3, 3)
    x, w = make_inputs(p, layer_id=700)
    ref, den = O.conv2d(oparams(p), x, w, with_denom=True)
    y = gpu_conv(p, x, w, C().ALGO_IMPLICIT_GEMM)
    y[0, 5, 5, 5] += 1e-2
    with pytest.raises(AssertionError):
        check_close(p, y, ref, den, C().ALGO_IMPLICIT_GEMM, "fault")


def test_tf32_mma_reads_truncated_operands(cuda_ok):
    """Hardware characterisation behind the 3xTF32 split: kind::tf32
    MMAs ignore the low 13 mantissa bits of fp32 operands, so feeding raw fp32 (TF32 mode) and
    pre-truncated fp32 must give bit-identical outputs."""
    p = P(2, 16, 16, 64, 64, 3, 3, math=1)
    x, w = make_inputs(p, layer_id=800)
    xt = (x.view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32)
    wt = (w.view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32)
    a = C().ALGO_IMPLICIT_GEMM
    assert np.array_equal(gpu_conv(p, x, w, a), gpu_conv(p, xt, wt, a))


@pytest.mark.parametrize("variant", [0, 1, 2, 3, 4, 7, 8, 11, 16, 17, 18, 24, 32, 34])
@pytest.mark.parametrize("case", [(2, 28, 28, 64, 64, 3, 3, 1, 1, 0), (1, 14, 15, 128, 128, 3, 3, 1, 1, 1),
                                  (2, 12, 12, 64, 256, 1, 1, 1, 1, 0), (1, 9, 9, 64, 320, 3, 3, 2, 2, 0),
                                  (2, 21, 19, 3, 36, 7, 7, 2, 2, 0),
                                  # 3x3 / C = 3 (V1-like): row-segment boxes and the A_STEM halo path (bit 0)
                                  (2, 20, 22, 3, 64, 3, 3, 1, 1, 0), (1, 17, 9, 2, 40, 3, 2, 1, 1, 1),
                                  # remainder split: 150 / 85 / 100 pair tiles (last wave 2 / 11 / 26 of 74)
                                  (2, 150, 128, 256, 64, 1, 1, 1, 1, 0), (5, 68, 64, 96, 128, 3, 3, 1, 1, 0),
                                  (8, 28, 28, 256, 1024, 1, 1, 1, 1, 0),
                                  # 3x3 halo, F = 96 (a partly out-of-range 32-column chunk of the direct-B boxes)
                                  (2, 12, 12, 32, 96, 3, 3, 1, 1, 0),
                                  # balanced K split: 40 pair tiles of 32 k-blocks (74 / 40 = 1 -> modelled best 3)
                                  (10, 32, 32, 1024, 64, 1, 1, 1, 1, 0)], ids=str)
def test_algorithm_parameter_variants(cuda_ok, monkeypatch, variant, case):
    """Both A-operand variants the auto-selector may pick per layer (implicit_gemm: halo <-> im2col,
    matmul_1x1: dense <-> im2col) give the same results (integer-exact and within tolerance)."""
    monkeypatch.setenv("CONV2D_FORCE_VARIANT", str(variant))
    p0 = P(*case)
    x, w = make_inputs(p0, layer_id=900)
    ref, den = O.conv2d(oparams(p0), x, w, with_denom=True)
    xi, wi = make_inputs(p0, layer_id=901, dist=synth.DIST_INT5)
    refi, deni = O.conv2d(oparams(p0), xi, wi, with_denom=True)
    for math in MATHS:
        p = p0.replace(math=math)
        for a in (C().ALGO_IMPLICIT_GEMM, C().ALGO_MATMUL_1X1):
            if not C().conv2d_supports(p, a):
                continue
            check_close(p, gpu_conv(p, x, w, a), ref, den, a, f"variant {variant} {case} {math} {a}")
            assert_int_exact(p, gpu_conv(p, xi, wi, a), refi, deni, a, f"variant int {case} {a}")


C4_CASES = [  # (N, H, W, C, F, KH, KW, SH, SW, pad): 3x3 / s1, C <= 4, W*C % 4 == 0 (raw 16-byte rows)
    (1, 224, 224, 3, 64, 3, 3, 1, 1, 0),   # VGG conv1_1 at batch 1 (the north_star small layer)
    (2, 20, 24, 3, 64, 3, 3, 1, 1, 0),     # ragged 16-row tiles, 3 column tiles
    (3, 17, 12, 1, 17, 3, 3, 1, 1, 1),     # VALID, C = 1, F % 4 != 0 (LSU epilogue), odd tile count
    (1, 9, 6, 2, 40, 3, 3, 1, 1, 0),       # C = 2, one tile
    (2, 33, 29, 4, 128, 3, 3, 1, 1, 0),    # C = 4 (no zero slots), BN = 128
    (1, 40, 36, 3, 200, 3, 3, 1, 1, 1),    # F > 128: two N tiles
    (1, 31, 40, 3, 96, 3, 3, 1, 1, 0),     # F = 96: BN = 128 with a zero column block
]


@pytest.mark.parametrize("case", C4_CASES, ids=str)
def test_igemm_c4_halo(cuda_ok, monkeypatch, case):
    """implicit_gemm's A_C4 path (gemm_halo.cu G3C4: 3x3 / s1 with C <= 4, two taps per K=8 MMA step
    through overlapping 16-byte-pixel views) against the oracle: integer-exact and within tolerance,
    both math modes; bit 0 (the row-segment path) agrees with it."""
    p0 = P(*case)
    x, w = make_inputs(p0, layer_id=960)
    ref, den = O.conv2d(oparams(p0), x, w, with_denom=True)
    xi, wi = make_inputs(p0, layer_id=961, dist=synth.DIST_INT5)
    refi, deni = O.conv2d(oparams(p0), xi, wi, with_denom=True)
    a = C().ALGO_IMPLICIT_GEMM
    for variant in (0, 1):
        monkeypatch.setenv("CONV2D_FORCE_VARIANT", str(variant))
        for math in MATHS:
            p = p0.replace(math=math)
            if variant == 0 and p0.features <= 128:
                assert C().conv2d_launch_count(p, a) == 1  # one launch: the halo GEMM builds B itself
            check_close(p, gpu_conv(p, x, w, a), ref, den, a, f"c4 v{variant} {case} math={math}")
            assert_int_exact(p, gpu_conv(p, xi, wi, a), refi, deni, a, f"c4 int v{variant} {case} math={math}")


S2D_CASES = [  # 7x7 / 8x8 stride-2 stems with C <= 3 and W*C % 4 == 0: raw-patch s2d halos
    (1, 37, 28, 3, 64, 7, 7, 2, 2, 0),     # ragged 8x16 tiles, SAME corners
    (2, 40, 36, 1, 32, 7, 7, 2, 2, 1),     # C = 1, VALID
    (1, 33, 48, 2, 100, 8, 8, 2, 2, 0),    # C = 2, K = 8, F not a multiple of 32 (BN = 128)
    (2, 24, 20, 3, 17, 7, 8, 2, 2, 0),     # non-square window, F % 4 != 0
]


@pytest.mark.parametrize("case", S2D_CASES, ids=str)
def test_s2d_stem_packed_and_sw64(cuda_ok, monkeypatch, case):
    """implicit_gemm's space-to-depth stem in both halo forms: the packed chunk-plane halo (GS2P, default:
    K=8 steps pair arbitrary real (tap, plane) chunks through the descriptor LBO) and the SWIZZLE_64B halo
    (GS2D, CONV2D_S2D_SW64): each against the oracle, integer-exact and within tolerance, both math modes."""
    p0 = P(*case)
    x, w = make_inputs(p0, layer_id=970)
    ref, den = O.conv2d(oparams(p0), x, w, with_denom=True)
    xi, wi = make_inputs(p0, layer_id=971, dist=synth.DIST_INT5)
    refi, deni = O.conv2d(oparams(p0), xi, wi, with_denom=True)
    a = C().ALGO_IMPLICIT_GEMM
    monkeypatch.setenv("CONV2D_FORCE_VARIANT", "0")
    for sw64 in (False, True):
        if sw64:
            monkeypatch.setenv("CONV2D_S2D_SW64", "1")
        else:
            monkeypatch.delenv("CONV2D_S2D_SW64", raising=False)
        for math in MATHS:
            p = p0.replace(math=math)
            check_close(p, gpu_conv(p, x, w, a), ref, den, a, f"s2d sw64={sw64} {case} math={math}")
            assert_int_exact(p, gpu_conv(p, xi, wi, a), refi, deni, a, f"s2d int sw64={sw64} {case} math={math}")


WINO_FUSED_CASES = [l.params(1) for l in ALL_SHAPES if l.window == 3 and l.stride == 1 and l.channels >= 32] + [
    dict(batch=3, in_rows=15, in_cols=9, channels=64, features=68, window_rows=3, window_cols=3, stride_rows=1,
         stride_cols=1, padding=1),    # VALID, ragged tile blocks, F % 32 != 0
    dict(batch=1, in_rows=9, in_cols=7, channels=40, features=36, window_rows=3, window_cols=3, stride_rows=1,
         stride_cols=1, padding=0),    # odd Ho / Wo, C % 16 != 0
    dict(batch=9, in_rows=7, in_cols=7, channels=32, features=96, window_rows=3, window_cols=3, stride_rows=1,
         stride_cols=1, padding=0),    # whole images per tile block (NB = 8) plus a ragged block
    dict(batch=5, in_rows=28, in_cols=28, channels=128, features=128, window_rows=3, window_cols=3,
         stride_rows=1, stride_cols=1, padding=0),  # several units per cluster
    dict(batch=2, in_rows=2, in_cols=30, channels=32, features=32, window_rows=3, window_cols=3, stride_rows=1,
         stride_cols=1, padding=0),    # a single tile row (Ho = 2)
]


@pytest.mark.parametrize("case", WINO_FUSED_CASES, ids=lambda d: "x".join(str(v) for v in d.values()))
def test_winograd_fused_variant(cuda_ok, monkeypatch, case):
    """winograd_f2x2_3x3 variant 1 (the fused kernel, wino_fused.cu) on every paper 3x3/s1 shape and the
    block-geometry edge cases: bit-exact in the integer regime (P7), within tolerance and under the P10
    ceiling on uniform data, both math modes; and bitwise equal to itself run again (determinism)."""
    monkeypatch.setenv("CONV2D_FORCE_WINO_VARIANT", "1")
    p0 = C().Params(**case)
    a = C().ALGO_WINOGRAD_F2X2_3X3
    assert 1 in C().conv2d_variants(p0, a)
    x, w = make_inputs(p0, layer_id=950)
    ref, den = O.conv2d(oparams(p0), x, w, with_denom=True)
    xi, wi = make_inputs(p0, layer_id=951, dist=synth.DIST_INT5)
    refi, deni = O.conv2d(oparams(p0), xi, wi, with_denom=True)
    for math in MATHS:
        p = p0.replace(math=math)
        y = gpu_conv(p, x, w, a)
        check_close(p, y, ref, den, a, f"fused {case} math={math}")
        assert np.array_equal(y, gpu_conv(p, x, w, a)), "fused winograd not deterministic"
        assert_int_exact(p, gpu_conv(p, xi, wi, a), refi, deni, a, f"fused int {case} math={math}")


def test_selection_table_gpu_round_trip(cuda_ok, tmp_path):
    """N4: the tuned choice (algorithm + its parameter variant) survives save -> clear -> load, and
    conv2d_forward(AUTO) then runs the loaded choice without tuning (same bits)."""
    c = C()
    p = P(8, 28, 28, 128, 512, 1, 1, 1, 1, 0)
    x, w = make_inputs(p, layer_id=1000)
    c.conv2d_clear_selection_cache()
    y0 = gpu_conv(p, x, w, c.ALGO_AUTO)
    a0 = c.conv2d_selected(p)
    f = tmp_path / "sel.txt"
    c.conv2d_save_selection(str(f))
    text = f.read_text()
    assert f": {c.conv2d_algo_name(a0)}" in text
    c.conv2d_clear_selection_cache()
    assert c.conv2d_selected(p) is None
    assert c.conv2d_load_selection(str(f)) >= 1
    assert c.conv2d_selected(p) == a0
    y1 = gpu_conv(p, x, w, c.ALGO_AUTO)
    assert np.array_equal(y0, y1)
