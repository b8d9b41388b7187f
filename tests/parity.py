"""Shared parity helpers for the GPU tests (test infrastructure; imports the oracle).

CUDA side: paper_1904_04174_b200.conv2d (the C-ABI binding).  Oracle side: oracle/.
Inputs for both come from paper_1904_04174_b200.synth only.
"""
from __future__ import annotations

import json
import os

import numpy as np

import oracle as O
from paper_1904_04174_b200 import synth

TOL_FP32 = 1e-5   # north_star: fp32 and 3xTF32
TOL_TF32 = 2e-3   # north_star: plain TF32

_C = None


def C():
    global _C
    if _C is None:
        from paper_1904_04174_b200 import build
        build.build()
        from paper_1904_04174_b200 import conv2d
        _C = conv2d
    return _C


def tol_for(algo: int, math: int) -> float:
    c = C()
    if math == c.MATH_TF32 and algo in (c.ALGO_IMPLICIT_GEMM, c.ALGO_MATMUL_1X1, c.ALGO_WINOGRAD_F2X2_3X3,
                                        c.ALGO_AUTO):
        return TOL_TF32
    return TOL_FP32


# P10 error ceilings: the expected error of each algorithm's own
# arithmetic with margin -- an output inside the north_star tolerance but above its ceiling is a bug.  Sources:
# tools/error_model.py (numpy emulation: the tensor core's fp32 accumulation truncates, RZ -- 3xTF32 GEMM model
# 2.3e-6 on V8 vs 2.3e-6 measured) and the round-2 error census of the whole GPU suite (CONV2D_ERRLOG).
CEILING = {  # (algorithm name, math) -> max normalised error
    ("direct", 0): 1e-6, ("direct", 1): 1e-6, ("tiled", 0): 1e-6, ("tiled", 1): 1e-6,   # exact-fp32 FFMA: 3.3e-7
    ("implicit_gemm", 0): 4e-6, ("matmul_1x1", 0): 4e-6,          # 3xTF32, RZ accumulation over K <= 4608: 2.3e-6
    ("winograd_f2x2_3x3", 0): 2e-6,                                # K = C only: 3.9e-7
    ("winograd_f4x4_3x3", 0): 6e-6,                                # fp32 transforms x 3xTF32: 3.7e-6
    ("winograd_f2x2_3x3", 1): 1e-3,                                # TF32 (RNA-rounded U, V), C >= 32: 2.1e-4
    ("implicit_gemm", 1): TOL_TF32, ("matmul_1x1", 1): TOL_TF32,  # truncated TF32; tiny-K fuzz shapes 1.7e-3
}


def ceiling_for(algo: int, math: int) -> float:
    c = C()
    if algo == c.ALGO_AUTO:  # the largest ceiling among the candidates AUTO may pick
        return max(v for (a, m), v in CEILING.items() if m == math)
    return CEILING[(c.ALGO_NAMES[algo], int(math))]


def oparams(p) -> O.Params:
    return O.Params(p.batch, p.in_rows, p.in_cols, p.channels, p.features, p.window_rows, p.window_cols,
                    p.stride_rows, p.stride_cols, p.padding)


def make_inputs(p, layer_id: int = 0, dist: int = synth.DIST_UNIFORM):
    x = synth.input_nhwc(p.batch, p.in_rows, p.in_cols, p.channels, layer_id=layer_id, dist=dist)
    w = synth.filter_hwcf(p.window_rows, p.window_cols, p.channels, p.features, layer_id=layer_id, dist=dist)
    return x, w


def gpu_conv(p, x: np.ndarray, w: np.ndarray, algo: int) -> np.ndarray:
    import torch
    c = C()
    xd = torch.from_numpy(x).cuda()
    wd = torch.from_numpy(w).cuda()
    (n, ho, wo, f), _ = c.conv2d_output_shape(p)
    y = torch.full((n, ho, wo, f), float("nan"), dtype=torch.float32, device="cuda")  # poison: catches unwritten outputs
    need = c.conv2d_query_workspace(p, algo)
    ws = torch.full((max(need, 16),), 0xFF, dtype=torch.uint8, device="cuda") if need else None
    c.conv2d_forward(p, algo, xd, wd, y, ws, need)
    torch.cuda.synchronize()
    return y.cpu().numpy()


def supported_algos(p):
    c = C()
    return [a for a in range(1, c.NUM_ALGOS) if c.conv2d_supports(p, a)]


def record_err(what: str, algo: int, math: int, e: float, n: int = 0):
    """CONV2D_ERRLOG=path: append one JSON line per parity check (error census behind the P10 ceilings)."""
    path = os.environ.get("CONV2D_ERRLOG")
    if path:
        with open(path, "a") as fh:
            fh.write(json.dumps({"what": what, "algo": C().ALGO_NAMES[algo], "math": int(math), "err": float(e),
                                 "n": int(n)}) + "\n")


def check_close(p, y: np.ndarray, y_ref: np.ndarray, denom: np.ndarray, algo: int, what: str = ""):
    assert y.shape == y_ref.shape, (what, y.shape, y_ref.shape)
    assert np.all(np.isfinite(y)), f"{what}: non-finite output (unwritten or NaN)"
    e = O.normalized_error(y, y_ref, denom)
    record_err(what, algo, p.math, e, y.size)
    tol = tol_for(algo, p.math)
    assert e <= tol, f"{what}: normalized error {e:.3e} > {tol:.0e}"
    cap = ceiling_for(algo, p.math)
    assert e <= cap, f"{what}: normalized error {e:.3e} inside the tolerance but above the P10 ceiling {cap:.0e}"
    return e


def assert_int_exact(p, y: np.ndarray, y_ref: np.ndarray, denom: np.ndarray, algo: int, what: str = ""):
    """Integer regime (inputs in {-2..2}): every partial sum is exact, so every algorithm is bit-exact --
    except Winograd F(4x4,3x3), whose filter transform has non-dyadic constants (1/6, 1/12, 1/24) and is
    held to the fp32 tolerance instead (reading R21)."""
    if algo == C().ALGO_WINOGRAD_F4X4_3X3:
        check_close(p, y, y_ref, denom, algo, what)
    else:
        assert np.array_equal(y, y_ref), (what, int(np.sum(y != y_ref)))
