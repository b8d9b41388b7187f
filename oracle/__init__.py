"""CPU oracle for the fp32 NHWC conv2d forward pass -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product path (``paper_1904_04174_b200``) never imports it, and it never
imports the product path: the two share no code (the only shared module is
the seeded input generator ``paper_1904_04174_b200/synth.py``, which holds
none of the method's arithmetic and is not used here).

The arithmetic lives in ``oracle.c`` (a naive 7-loop, double accumulation,
one rounding to fp32 -- PAPER.md:206-210 "same numeric results", SPEC.md:117-125,
SURVEY.md §8(c)).  This module is argument marshalling plus the error metric
of BASELINE.json's north_star (max |err| / sum_taps |x||w|, R7).

Parity status: pinned (tests/test_oracle.py: closed forms, hand cases, golden
integer fixtures, torch float64 library conv, brute-force Python, invariants).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = [os.path.join(_HERE, "oracle.c"), os.path.join(_HERE, "pool.c")]

SAME, VALID = 0, 1


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (plain -O2, no fast-math: summation order is the source order)."""
    newest = max(os.path.getmtime(s) for s in _SRC + [os.path.join(_HERE, "oracle.h")])
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < newest:
        cmd = ["gcc", "-O2", "-std=c99", "-fPIC", "-shared", "-pthread", "-fno-fast-math",
               "-ffp-contract=off", "-o", _SO] + _SRC + ["-lm"]
        subprocess.check_call(cmd)
    return _SO


class _Params(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in (
        "batch", "in_rows", "in_cols", "channels", "features",
        "window_rows", "window_cols", "stride_rows", "stride_cols", "padding")]


@dataclass(frozen=True)
class Params:
    batch: int
    in_rows: int
    in_cols: int
    channels: int
    features: int
    window_rows: int
    window_cols: int
    stride_rows: int = 1
    stride_cols: int = 1
    padding: int = SAME  # SAME=0, VALID=1

    def c(self) -> _Params:
        return _Params(self.batch, self.in_rows, self.in_cols, self.channels, self.features,
                       self.window_rows, self.window_cols, self.stride_rows, self.stride_cols,
                       self.padding)


POOL_MAX, POOL_AVG = 0, 1


class _PoolParams(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in (
        "batch", "in_rows", "in_cols", "channels", "window_rows", "window_cols", "stride_rows",
        "stride_cols", "padding", "op")]


@dataclass(frozen=True)
class PoolParams:
    """NHWC pooling (pool.c): op POOL_MAX / POOL_AVG, padding SAME / VALID."""
    batch: int
    in_rows: int
    in_cols: int
    channels: int
    window_rows: int
    window_cols: int
    stride_rows: int = 1
    stride_cols: int = 1
    padding: int = SAME
    op: int = POOL_MAX

    def c(self) -> _PoolParams:
        return _PoolParams(self.batch, self.in_rows, self.in_cols, self.channels, self.window_rows,
                           self.window_cols, self.stride_rows, self.stride_cols, self.padding, self.op)


_lib = None


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        P = ctypes.POINTER(_Params)
        fp = ctypes.POINTER(ctypes.c_float)
        dp = ctypes.POINTER(ctypes.c_double)
        i32p = ctypes.POINTER(ctypes.c_int32)
        i64p = ctypes.POINTER(ctypes.c_int64)
        lib.oracle_output_shape.argtypes = [P, i32p, i32p]
        lib.oracle_output_shape.restype = ctypes.c_int
        lib.oracle_flop_count.argtypes = [P]
        lib.oracle_flop_count.restype = ctypes.c_uint64
        lib.oracle_conv2d.argtypes = [P, fp, fp, fp, dp, ctypes.c_int]
        lib.oracle_conv2d.restype = ctypes.c_int
        lib.oracle_conv2d_point.argtypes = [P, fp, fp, ctypes.c_int64, ctypes.c_int64,
                                            ctypes.c_int64, ctypes.c_int64, dp, dp]
        lib.oracle_conv2d_point.restype = ctypes.c_int
        lib.oracle_conv2d_points.argtypes = [P, fp, fp, i64p, ctypes.c_int64, dp, dp, ctypes.c_int]
        lib.oracle_conv2d_points.restype = ctypes.c_int
        PP = ctypes.POINTER(_PoolParams)
        lib.oracle_pool2d_shape.argtypes = [PP, i32p, i32p]
        lib.oracle_pool2d_shape.restype = ctypes.c_int
        lib.oracle_pool2d.argtypes = [PP, fp, fp, ctypes.c_int]
        lib.oracle_pool2d.restype = ctypes.c_int
        _lib = lib
    return _lib


def _fptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_float))


def _dptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def output_shape(p: Params):
    """((N, Ho, Wo, F), (pad_top, pad_bottom, pad_left, pad_right)); ValueError if invalid."""
    o = (ctypes.c_int32 * 4)()
    pd = (ctypes.c_int32 * 4)()
    if _load().oracle_output_shape(ctypes.byref(p.c()), o, pd):
        raise ValueError(f"invalid conv params {p}")
    return tuple(o), tuple(pd)


def flop_count(p: Params) -> int:
    v = _load().oracle_flop_count(ctypes.byref(p.c()))
    if v == 0:
        raise ValueError(f"invalid conv params {p}")
    return int(v)


def _check_operands(p: Params, x: np.ndarray, w: np.ndarray):
    x = np.ascontiguousarray(x, dtype=np.float32)
    w = np.ascontiguousarray(w, dtype=np.float32)
    if x.shape != (p.batch, p.in_rows, p.in_cols, p.channels):
        raise ValueError(f"input shape {x.shape} != NHWC {(p.batch, p.in_rows, p.in_cols, p.channels)}")
    if w.shape != (p.window_rows, p.window_cols, p.channels, p.features):
        raise ValueError(f"filter shape {w.shape} != HWCF")
    return x, w


def conv2d(p: Params, x: np.ndarray, w: np.ndarray, with_denom: bool = False, threads: int | None = None):
    """Full oracle convolution.  Returns y (fp32, N,Ho,Wo,F) [, denom (fp64 sum |x||w|)]."""
    x, w = _check_operands(p, x, w)
    shp, _ = output_shape(p)
    y = np.empty(shp, dtype=np.float32)
    d = np.empty(shp, dtype=np.float64) if with_denom else None
    if threads is None:
        threads = os.cpu_count() or 1
    if _load().oracle_conv2d(ctypes.byref(p.c()), _fptr(x), _fptr(w), _fptr(y), _dptr(d), threads):
        raise ValueError("oracle_conv2d failed")
    return (y, d) if with_denom else y


def conv2d_points(p: Params, x: np.ndarray, w: np.ndarray, idx: np.ndarray, threads: int | None = None):
    """Sampled outputs: idx (count,4) int64 of (n,ho,wo,f) -> (y fp64 unrounded, denom fp64)."""
    x, w = _check_operands(p, x, w)
    idx = np.ascontiguousarray(idx, dtype=np.int64).reshape(-1, 4)
    y = np.empty(idx.shape[0], dtype=np.float64)
    d = np.empty(idx.shape[0], dtype=np.float64)
    if threads is None:
        threads = os.cpu_count() or 1
    st = _load().oracle_conv2d_points(ctypes.byref(p.c()), _fptr(x), _fptr(w),
                                      idx.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                      idx.shape[0], _dptr(y), _dptr(d), threads)
    if st:
        raise ValueError("oracle_conv2d_points: invalid params or index")
    return y, d


def normalized_error(y: np.ndarray, y_ref: np.ndarray, denom: np.ndarray) -> float:
    """north_star metric: max_o |y_o - yref_o| / sum_taps |x||w| (R7).

    Where the denominator is 0 (every tap is a zero product) the output must be
    exactly 0; a nonzero value there returns +inf.
    """
    y = np.asarray(y, dtype=np.float64)
    y_ref = np.asarray(y_ref, dtype=np.float64)
    denom = np.asarray(denom, dtype=np.float64)
    err = np.abs(y - y_ref)
    zero = denom == 0
    if np.any(zero & (y != 0)):
        return float("inf")
    if y.size == 0:
        return 0.0
    ratio = np.where(zero, 0.0, err / np.where(zero, 1.0, denom))
    return float(ratio.max())


def pool_output_shape(p: PoolParams):
    """((N, Ho, Wo, C), (pad_top, pad_bottom, pad_left, pad_right)); ValueError if invalid."""
    o = (ctypes.c_int32 * 4)()
    pd = (ctypes.c_int32 * 4)()
    if _load().oracle_pool2d_shape(ctypes.byref(p.c()), o, pd):
        raise ValueError(f"invalid pool params {p}")
    return tuple(o), tuple(pd)


def pool2d(p: PoolParams, x: np.ndarray, threads: int | None = None) -> np.ndarray:
    """Oracle pooling of an NHWC fp32 tensor -> fp32 (N, Ho, Wo, C)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    if x.shape != (p.batch, p.in_rows, p.in_cols, p.channels):
        raise ValueError(f"input shape {x.shape} != NHWC {(p.batch, p.in_rows, p.in_cols, p.channels)}")
    shp, _ = pool_output_shape(p)
    y = np.empty(shp, dtype=np.float32)
    if threads is None:
        threads = os.cpu_count() or 1
    st = _load().oracle_pool2d(ctypes.byref(p.c()), _fptr(x), _fptr(y), threads)
    if st:
        raise ValueError(f"oracle_pool2d failed ({st})")
    return y
