"""Persisted selector table ("table serialization round-trips losslessly",
SPEC.md:354 line format).  Host-only: runs without a GPU."""
import os

import pytest

from paper_1904_04174_b200 import build as B


@pytest.fixture(scope="module")
def C():
    B.build()
    from paper_1904_04174_b200 import conv2d
    return conv2d


def _params(C):
    P = C.Params
    return [
        (P(32, 56, 56, 64, 256, 1, 1, 1, 1, C.PAD_SAME), C.ALGO_MATMUL_1X1),
        (P(32, 56, 56, 64, 64, 3, 3, 1, 1, C.PAD_SAME), C.ALGO_WINOGRAD_F2X2_3X3),
        (P(32, 224, 224, 3, 64, 7, 7, 2, 2, C.PAD_SAME), C.ALGO_IMPLICIT_GEMM),
        (P(1, 9, 7, 5, 3, 2, 4, 2, 1, C.PAD_VALID, math=C.MATH_TF32), C.ALGO_DIRECT),
        (P(2, 17, 19, 36, 24, 3, 3, 2, 2, C.PAD_SAME, math=C.MATH_TF32), C.ALGO_TILED),
    ]


def test_round_trip(C, tmp_path):
    C.conv2d_clear_selection_cache()
    entries = _params(C)
    for p, a in entries:
        C.conv2d_set_selected(p, a)
    f = tmp_path / "sel.txt"
    C.conv2d_save_selection(str(f))
    text = f.read_text()
    assert text.startswith("#")
    assert "default :" in text
    assert "32 224 224 3 64 7 7 2 2 same fp32 : implicit_gemm" in text
    assert "1 9 7 5 3 2 4 2 1 valid tf32 : direct" in text
    C.conv2d_clear_selection_cache()
    for p, _ in entries:
        assert C.conv2d_selected(p) is None
    assert C.conv2d_load_selection(str(f)) == len(entries)
    for p, a in entries:
        assert C.conv2d_selected(p) == a
    # saving again reproduces the file exactly (lossless)
    g = tmp_path / "sel2.txt"
    C.conv2d_save_selection(str(g))
    assert g.read_text() == text


def test_variants_comments_and_default_line(C, tmp_path):
    C.conv2d_clear_selection_cache()
    f = tmp_path / "v.txt"
    f.write_text("# tuned on a B200\n\n"
                 "256 56 56 64 256 1 1 1 1 same fp32 : matmul_1x1/10   # B path + N tile\n"
                 "256 14 14 256 256 3 3 1 1 same fp32 : implicit_gemm/10\n"
                 "default : implicit_gemm, matmul_1x1,winograd_f2x2_3x3,direct,tiled\n")
    assert C.conv2d_load_selection(str(f)) == 2
    P = C.Params
    assert C.conv2d_selected(P(256, 56, 56, 64, 256, 1, 1, 1, 1, C.PAD_SAME)) == C.ALGO_MATMUL_1X1
    g = tmp_path / "v2.txt"
    C.conv2d_save_selection(str(g))
    out = g.read_text()
    assert "256 56 56 64 256 1 1 1 1 same fp32 : matmul_1x1/10" in out
    assert "256 14 14 256 256 3 3 1 1 same fp32 : implicit_gemm/10" in out


@pytest.mark.parametrize("body,status", [
    ("1 8 8 4 8 3 3 1 1 same fp32 implicit_gemm\n", "CONV2D_ERR_INVALID_PARAMS"),        # no ':'
    ("1 8 8 4 8 3 3 1 same fp32 : direct\n", "CONV2D_ERR_INVALID_PARAMS"),                # 10 fields
    ("1 8 8 4 8 3 3 1 1 sane fp32 : direct\n", "CONV2D_ERR_INVALID_PARAMS"),              # padding
    ("1 8 8 4 8 3 3 1 1 same fp16 : direct\n", "CONV2D_ERR_INVALID_PARAMS"),              # math
    ("1 8 8 4 8 3 3 1 1 same fp32 : fft\n", "CONV2D_ERR_INVALID_PARAMS"),                 # algorithm
    ("1 8 8 4 8 3 3 1 1 same fp32 : auto\n", "CONV2D_ERR_INVALID_PARAMS"),                # not concrete
    ("1 8 8 4 8 9 9 1 1 valid fp32 : direct\n", "CONV2D_ERR_INVALID_PARAMS"),             # VALID, K > H
    ("1 8 8 4 8 7 7 2 2 same fp32 : winograd_f2x2_3x3\n", "CONV2D_ERR_UNSUPPORTED"),      # incompatible
    ("1 8 8 4 8 3 3 1 1 same fp32 : direct/2\n", "CONV2D_ERR_INVALID_PARAMS"),            # variant on direct
    ("1 8 8 4 8 3 3 1 1 same fp32 : implicit_gemm/99\n", "CONV2D_ERR_INVALID_PARAMS"),    # variant range
    ("256 56 56 64 256 1 1 1 1 same fp32 : matmul_1x1/4\n", "CONV2D_ERR_INVALID_PARAMS"),  # never enumerated
    ("default : direct,bogus\n", "CONV2D_ERR_INVALID_PARAMS"),
])
def test_invalid_files_leave_the_cache_untouched(C, tmp_path, body, status):
    C.conv2d_clear_selection_cache()
    P = C.Params
    keep = P(1, 8, 8, 4, 8, 1, 1, 1, 1, C.PAD_SAME)
    C.conv2d_set_selected(keep, C.ALGO_DIRECT)
    f = tmp_path / "bad.txt"
    f.write_text("1 8 8 4 8 1 1 1 1 same fp32 : matmul_1x1\n" + body)  # a valid first line
    with pytest.raises(RuntimeError) as ei:
        C.conv2d_load_selection(str(f))
    assert status in str(ei.value)
    assert "bad.txt:2" in C.conv2d_last_error()
    assert C.conv2d_selected(keep) == C.ALGO_DIRECT  # first line not applied either


def test_io_errors(C, tmp_path):
    with pytest.raises(RuntimeError) as ei:
        C.conv2d_load_selection(str(tmp_path / "missing.txt"))
    assert "CONV2D_ERR_IO" in str(ei.value)
    with pytest.raises(RuntimeError) as ei:
        C.conv2d_save_selection(str(tmp_path / "no_such_dir" / "x.txt"))
    assert "CONV2D_ERR_IO" in str(ei.value)
