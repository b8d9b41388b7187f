"""libconv2d.so host side, no GPU needed: it loads, exports every symbol include/conv2d.h
declares, and its shape / flop / compatibility / validation logic is right.

Shapes are cross-checked against the oracle's independent shape code (the two share no
code) and against the SURVEY Appendix A golden table.
"""
import json
import os
import re

import pytest
from hypothesis import given, settings, strategies as st

import oracle as O
from paper_1904_04174_b200 import build as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def C():
    B.build()
    from paper_1904_04174_b200 import conv2d
    return conv2d


def test_exports_every_declared_symbol(C):
    inc = os.path.join(ROOT, "include")
    hdr = "".join(open(os.path.join(inc, f)).read() for f in sorted(os.listdir(inc)) if f.endswith(".h"))
    declared = set(re.findall(r"\b((?:conv2d|pool2d)_[a-z_]+)\s*\(", hdr))
    declared = {d for d in declared if not d.endswith("_t")}
    assert declared == set(C.EXPORTED), declared ^ set(C.EXPORTED)
    for name in declared:
        assert hasattr(C._lib, name)


def test_enum_values_match_header(C):
    hdr = open(os.path.join(ROOT, "include", "conv2d.h")).read()
    for name, val in [("CONV2D_ALGO_DIRECT", 1), ("CONV2D_ALGO_TILED", 2), ("CONV2D_ALGO_IMPLICIT_GEMM", 3),
                      ("CONV2D_ALGO_WINOGRAD_F2X2_3X3", 4), ("CONV2D_ALGO_MATMUL_1X1", 5),
                      ("CONV2D_ALGO_WINOGRAD_F4X4_3X3", 6)]:
        assert re.search(rf"{name}\s*=\s*{val}\b", hdr)
        assert getattr(C, name.replace("CONV2D_", "")) == val
    assert C.conv2d_algo_name(C.ALGO_WINOGRAD_F2X2_3X3) == "winograd_f2x2_3x3"
    assert C.conv2d_algo_name(C.ALGO_WINOGRAD_F4X4_3X3) == "winograd_f4x4_3x3"
    assert re.search(r"#define CONV2D_NUM_ALGOS 7\b", hdr) and C.NUM_ALGOS == 7
    assert C.conv2d_status_string(C.ERR_WORKSPACE) == "CONV2D_ERR_WORKSPACE"


def test_paper_shapes_golden(C):
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "paper_shapes.json")))
    for e in g["layers"]:
        p = C.Params(1, e["H"], e["W"], e["C"], e["F"], e["K"], e["K"], e["S"], e["S"], C.PAD_SAME)
        shp, pads = C.conv2d_output_shape(p)
        assert shp == (1, e["out"], e["out"], e["F"]) and list(pads) == e["pads_tblr"], e["name"]
        assert C.conv2d_flop_count(p) == O.flop_count(O.Params(1, e["H"], e["W"], e["C"], e["F"], e["K"], e["K"],
                                                                 e["S"], e["S"], O.SAME))


@settings(max_examples=300, deadline=None)
@given(n=st.integers(1, 4), h=st.integers(1, 40), w=st.integers(1, 40), c=st.integers(1, 64),
       f=st.integers(1, 64), kh=st.sampled_from([1, 2, 3, 5, 7]), kw=st.sampled_from([1, 2, 3, 5, 7]),
       sh=st.integers(1, 4), sw=st.integers(1, 4), pad=st.sampled_from([0, 1]))
def test_shapes_match_oracle(C, n, h, w, c, f, kh, kw, sh, sw, pad):
    p = C.Params(n, h, w, c, f, kh, kw, sh, sw, pad)
    q = O.Params(n, h, w, c, f, kh, kw, sh, sw, pad)
    try:
        ref = O.output_shape(q)
    except ValueError:
        with pytest.raises(C.Conv2dError) as ei:
            C.conv2d_output_shape(p)
        assert ei.value.status == C.ERR_INVALID_PARAMS
        return
    assert C.conv2d_output_shape(p) == ref
    assert C.conv2d_flop_count(p) == O.flop_count(q)


def test_supports_table(C):
    P = C.Params
    p3 = P(1, 56, 56, 64, 64, 3, 3, 1, 1)
    assert C.conv2d_supports(p3, C.ALGO_WINOGRAD_F2X2_3X3)
    assert not C.conv2d_supports(p3, C.ALGO_MATMUL_1X1)  # SPEC.md:257 K=3 -> incompatible
    assert not C.conv2d_supports(p3.replace(channels=3), C.ALGO_WINOGRAD_F2X2_3X3)  # reading R16: C >= 32
    assert not C.conv2d_supports(p3.replace(stride_rows=2, stride_cols=2), C.ALGO_WINOGRAD_F2X2_3X3)
    assert C.conv2d_supports(p3, C.ALGO_WINOGRAD_F4X4_3X3)                       # FP32 math
    assert not C.conv2d_supports(p3.replace(math=C.MATH_TF32), C.ALGO_WINOGRAD_F4X4_3X3)  # reading R21
    assert not C.conv2d_supports(p3.replace(channels=16), C.ALGO_WINOGRAD_F4X4_3X3)
    assert not C.conv2d_supports(p3.replace(window_rows=5, window_cols=5), C.ALGO_WINOGRAD_F4X4_3X3)
    p1 = P(1, 56, 56, 64, 256, 1, 1, 1, 1)
    assert C.conv2d_supports(p1, C.ALGO_MATMUL_1X1)
    assert not C.conv2d_supports(p1.replace(stride_rows=2, stride_cols=2), C.ALGO_MATMUL_1X1)
    for a in (C.ALGO_AUTO, C.ALGO_DIRECT, C.ALGO_TILED, C.ALGO_IMPLICIT_GEMM):
        assert C.conv2d_supports(p1, a) and C.conv2d_supports(P(1, 224, 224, 3, 64, 7, 7, 2, 2), a)


@settings(max_examples=500, deadline=None)
@given(n=st.integers(1, 64), h=st.integers(1, 230), c=st.integers(1, 2048), f=st.integers(1, 2048),
       k=st.sampled_from([1, 3, 5, 7]), s=st.integers(1, 2), pad=st.sampled_from([0, 1]),
       math=st.sampled_from([0, 1]))
def test_workspace_query_for_every_supported_algo(C, n, h, c, f, k, s, pad, math):
    # selector soundness: AUTO's workspace covers every supported algorithm
    p = C.Params(n, h, h, c, f, k, k, s, s, pad, math)
    try:
        C.conv2d_output_shape(p)
    except C.Conv2dError:
        return
    ws_auto = C.conv2d_query_workspace(p, C.ALGO_AUTO)
    for a in range(1, C.NUM_ALGOS):
        if C.conv2d_supports(p, a):
            assert 0 <= C.conv2d_query_workspace(p, a) <= ws_auto
            assert C.conv2d_launch_count(p, a) >= 1
        else:
            with pytest.raises(C.Conv2dError) as ei:
                C.conv2d_query_workspace(p, a)
            assert ei.value.status == C.ERR_UNSUPPORTED


def test_forward_validation_errors_before_any_launch(C):
    p = C.Params(1, 8, 8, 4, 8, 3, 3)
    ws = 1 << 20
    fake = 0x1000  # never dereferenced: every case below fails validation first
    with pytest.raises(C.Conv2dError) as e:
        C.conv2d_forward(p.replace(batch=0), C.ALGO_DIRECT, fake, fake, fake, stream=0)
    assert e.value.status == C.ERR_INVALID_PARAMS
    with pytest.raises(C.Conv2dError) as e:
        C.conv2d_forward(p.replace(padding=1, window_rows=9), C.ALGO_DIRECT, fake, fake, fake, stream=0)
    assert e.value.status == C.ERR_INVALID_PARAMS
    with pytest.raises(C.Conv2dError) as e:
        C.conv2d_forward(p, C.ALGO_MATMUL_1X1, fake, fake, fake, stream=0)
    assert e.value.status == C.ERR_UNSUPPORTED
    with pytest.raises(C.Conv2dError) as e:
        C.conv2d_forward(p, C.ALGO_DIRECT, fake, 0, fake, stream=0)
    assert e.value.status == C.ERR_NULL
    with pytest.raises(C.Conv2dError) as e:
        C.conv2d_forward(p, C.ALGO_DIRECT, fake + 4, fake, fake, stream=0)
    assert e.value.status == C.ERR_ALIGNMENT
    need = C.conv2d_query_workspace(p, C.ALGO_IMPLICIT_GEMM)
    assert need > 0
    with pytest.raises(C.Conv2dError) as e:
        C.conv2d_forward(p, C.ALGO_IMPLICIT_GEMM, fake, fake, fake, fake, need - 1, stream=0)
    assert e.value.status == C.ERR_WORKSPACE
    with pytest.raises(C.Conv2dError) as e:
        C.conv2d_forward(p, 17, fake, fake, fake, stream=0)
    assert e.value.status == C.ERR_INVALID_PARAMS
    assert "workspace" in C.conv2d_last_error() or C.conv2d_last_error() != ""


def test_selection_cache_host_side(C):
    p = C.Params(2, 16, 16, 32, 32, 3, 3)
    C.conv2d_clear_selection_cache()
    assert C.conv2d_selected(p) is None
    C.conv2d_set_selected(p, C.ALGO_TILED)
    assert C.conv2d_selected(p) == C.ALGO_TILED
    assert C.conv2d_launch_count(p, C.ALGO_AUTO) == 1
    assert C.conv2d_selected(p.replace(math=C.MATH_TF32)) is None  # math is part of the key
    with pytest.raises(C.Conv2dError):
        C.conv2d_set_selected(p, C.ALGO_MATMUL_1X1)
    C.conv2d_clear_selection_cache()
    assert C.conv2d_selected(p) is None


def test_variant_get_set_host_side(C):
    """conv2d_get_variant / conv2d_set_variant (bench.py replays rank 0's tuned variants on every rank)."""
    p = C.Params(3, 40, 40, 64, 64, 3, 3)  # 3x3/s1: halo and im2col A paths (bit 0) both enumerated
    C.conv2d_set_variant(p, C.ALGO_IMPLICIT_GEMM, 1)
    assert C.conv2d_get_variant(p, C.ALGO_IMPLICIT_GEMM) == 1
    C.conv2d_set_variant(p, C.ALGO_IMPLICIT_GEMM, 0)
    assert C.conv2d_get_variant(p, C.ALGO_IMPLICIT_GEMM) == 0
    # bit 5 (the halo path's direct B in 3xTF32) is enumerated here, with bit 0 clear only
    C.conv2d_set_variant(p, C.ALGO_IMPLICIT_GEMM, 32)
    assert C.conv2d_get_variant(p, C.ALGO_IMPLICIT_GEMM) == 32
    assert 32 in C.conv2d_variants(p, C.ALGO_IMPLICIT_GEMM) and 33 not in C.conv2d_variants(p, C.ALGO_IMPLICIT_GEMM)
    assert 32 not in C.conv2d_variants(p.replace(math=C.MATH_TF32), C.ALGO_IMPLICIT_GEMM)  # TF32: always direct
    # bit 2 (LSU epilogue) is never enumerated; bit 5 with bit 0 (im2col path); out of range
    for bad in (4, 33, 64, -1):
        with pytest.raises(C.Conv2dError) as e:
            C.conv2d_set_variant(p, C.ALGO_IMPLICIT_GEMM, bad)
        assert e.value.status == C.ERR_INVALID_PARAMS
    with pytest.raises(C.Conv2dError) as e:
        C.conv2d_get_variant(p, C.ALGO_TILED)
    assert e.value.status == C.ERR_INVALID_PARAMS
    with pytest.raises(C.Conv2dError) as e:  # a 3x3 window is not a 1x1 matmul
        C.conv2d_set_variant(p, C.ALGO_MATMUL_1X1, 0)
    assert e.value.status == C.ERR_UNSUPPORTED


def test_winograd_f2x2_variants_host_side(C):
    """winograd_f2x2_3x3 parameter variants: 0 = transforms + batched GEMM, 1 = the fused kernel
    (wino_fused.cu), enumerated only where its TMA plan applies (C % 4 == 0, F % 4 == 0, Ho >= 2)."""
    W = C.ALGO_WINOGRAD_F2X2_3X3
    for math in (C.MATH_FP32, C.MATH_TF32):
        p = C.Params(2, 14, 14, 256, 256, 3, 3, math=math)  # R17-like
        assert C.conv2d_variants(p, W) == [0, 1]
        C.conv2d_set_variant(p, W, 1)
        assert C.conv2d_get_variant(p, W) == 1
        C.conv2d_set_variant(p, W, 0)
        assert C.conv2d_get_variant(p, W) == 0
        with pytest.raises(C.Conv2dError) as e:
            C.conv2d_set_variant(p, W, 2)
        assert e.value.status == C.ERR_INVALID_PARAMS
    # C % 4 != 0 (the halo boxes need 16-byte pixel strides) and a 1-row output: only the unfused form
    assert C.conv2d_variants(C.Params(1, 9, 7, 34, 36, 3, 3), W) == [0]
    assert C.conv2d_variants(C.Params(1, 1, 9, 32, 32, 3, 3), W) == [0]
    # the fused form needs only the filter transform in the workspace (16 x Fpad x Cpad hi + lo)
    assert C.conv2d_query_workspace(C.Params(2, 14, 14, 256, 256, 3, 3), W) >= 2 * 16 * 256 * 256 * 4


@pytest.mark.parametrize("case", [(2, 13, 11, 5, 3, 3, 2, 2, 0), (256, 112, 112, 64, 3, 3, 2, 2, 0),
                                  (3, 14, 14, 4, 2, 2, 2, 2, 1), (1, 9, 10, 3, 4, 2, 3, 1, 0),
                                  (32, 7, 7, 2048, 7, 7, 1, 1, 1)], ids=str)
def test_pool_shapes_match_oracle(C, case):
    n, h, w, c, kh, kw, sh, sw, pad = case
    for op in (C.POOL_MAX, C.POOL_AVG):
        got = C.pool2d_output_shape(C.PoolParams(n, h, w, c, kh, kw, sh, sw, pad, op))
        assert got == O.pool_output_shape(O.PoolParams(n, h, w, c, kh, kw, sh, sw, pad, op))


def test_pool_validation_errors_before_any_launch(C):
    P = C.PoolParams
    for bad, code in [(P(0, 4, 4, 1, 2, 2), "INVALID_PARAMS"), (P(1, 4, 4, 1, 5, 5, 1, 1, C.PAD_VALID), "INVALID_PARAMS"),
                      (P(1, 4, 4, 1, 2, 2, 1, 1, C.PAD_SAME, 9), "INVALID_PARAMS"),
                      (P(1, 4, 4, 1, 2, 2, 0, 1), "INVALID_PARAMS")]:
        with pytest.raises(RuntimeError) as ei:
            C.pool2d_forward(bad, 16, 16, stream=0)
        assert code in str(ei.value)
    with pytest.raises(RuntimeError) as ei:
        C.pool2d_forward(P(1, 4, 4, 1, 2, 2), 0, 16, stream=0)
    assert "NULL" in str(ei.value)
    with pytest.raises(RuntimeError) as ei:
        C.pool2d_forward(P(1, 4, 4, 1, 2, 2), 18, 16, stream=0)
    assert "ALIGNMENT" in str(ei.value)


def test_autotune_flush_registration(C):
    with pytest.raises(RuntimeError) as ei:
        C.conv2d_set_autotune_flush(4096, 0)   # a buffer of 0 bytes
    assert "INVALID_PARAMS" in str(ei.value)
    C.conv2d_set_autotune_flush(4096, 1 << 20)  # registration only: never dereferenced on the host
    C.conv2d_set_autotune_flush(None)


def test_binding_fails_loudly_without_the_library(tmp_path):
    """No CPU or library fallback: with libconv2d.so absent, importing the binding raises."""
    import subprocess
    import sys
    code = "import paper_1904_04174_b200.conv2d"
    env = dict(os.environ, CONV2D_LIB=str(tmp_path / "absent" / "libconv2d.so"))
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True)
    assert r.returncode != 0
    assert "libconv2d.so not found" in r.stderr and "no fallback" in r.stderr
