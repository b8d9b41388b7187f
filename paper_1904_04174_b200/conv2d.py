"""Python binding of libconv2d.so (include/conv2d.h) -- argument marshalling only.

Every step of the convolution runs in the library's sm_100a kernels; this module
only converts torch tensors to device pointers, picks up the current CUDA stream
and raises on error codes.  There is no CPU or library fallback: if libconv2d.so
is missing or fails to load, importing this module raises.

Names mirror the C-ABI (conv2d_forward, conv2d_query_workspace, ...).  ``forward``
is the convenience call a user makes: it allocates the output and workspace with
torch and calls conv2d_forward on the current stream.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CONV2D_LIB", os.path.join(_HERE, "libconv2d.so"))

if not os.path.exists(LIB_PATH):
    raise ImportError(f"libconv2d.so not found at {LIB_PATH}: build it with "
                      f"`python -m paper_1904_04174_b200.build` (no fallback path exists)")
_lib = ctypes.CDLL(LIB_PATH)

PAD_SAME, PAD_VALID = 0, 1
MATH_FP32, MATH_TF32 = 0, 1
(ALGO_AUTO, ALGO_DIRECT, ALGO_TILED, ALGO_IMPLICIT_GEMM, ALGO_WINOGRAD_F2X2_3X3, ALGO_MATMUL_1X1,
 ALGO_WINOGRAD_F4X4_3X3) = range(7)
NUM_ALGOS = 7
ALGO_NAMES = ["auto", "direct", "tiled", "implicit_gemm", "winograd_f2x2_3x3", "matmul_1x1", "winograd_f4x4_3x3"]
ALGO_BY_NAME = {n: i for i, n in enumerate(ALGO_NAMES)}

STATUS = ["CONV2D_OK", "CONV2D_ERR_INVALID_PARAMS", "CONV2D_ERR_UNSUPPORTED", "CONV2D_ERR_WORKSPACE",
          "CONV2D_ERR_ALIGNMENT", "CONV2D_ERR_NULL", "CONV2D_ERR_CUDA", "CONV2D_ERR_NO_DEVICE",
                "CONV2D_ERR_IO"]
OK, ERR_INVALID_PARAMS, ERR_UNSUPPORTED, ERR_WORKSPACE, ERR_ALIGNMENT, ERR_NULL, ERR_CUDA, ERR_NO_DEVICE, ERR_IO = range(9)

EXPORTED = ["conv2d_output_shape", "conv2d_flop_count", "conv2d_supports", "conv2d_query_workspace",
            "conv2d_forward", "conv2d_autotune", "conv2d_selected", "conv2d_set_selected",
            "conv2d_clear_selection_cache", "conv2d_last_tune_times", "conv2d_launch_count",
            "conv2d_synth_fill", "conv2d_status_string", "conv2d_algo_name", "conv2d_last_error",
            "conv2d_debug_trace", "conv2d_debug_splits", "conv2d_save_selection", "conv2d_load_selection",
            "pool2d_output_shape", "pool2d_forward", "conv2d_set_autotune_flush", "conv2d_get_variant",
            "conv2d_set_variant", "conv2d_predict", "conv2d_set_auto_policy"]


class conv2d_params_t(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in (
        "batch", "in_rows", "in_cols", "channels", "features",
        "window_rows", "window_cols", "stride_rows", "stride_cols", "padding", "math")]


class Conv2dError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        detail = _lib.conv2d_last_error().decode()
        super().__init__(f"{where}: {STATUS[status] if 0 <= status < len(STATUS) else status}: {detail}")


_P = ctypes.POINTER(conv2d_params_t)
_vp = ctypes.c_void_p
_lib.conv2d_output_shape.argtypes = [_P, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32)]
_lib.conv2d_flop_count.argtypes = [_P, ctypes.POINTER(ctypes.c_uint64)]
_lib.conv2d_supports.argtypes = [_P, ctypes.c_int, ctypes.POINTER(ctypes.c_int)]
_lib.conv2d_query_workspace.argtypes = [_P, ctypes.c_int, ctypes.POINTER(ctypes.c_size_t)]
_lib.conv2d_forward.argtypes = [_P, ctypes.c_int, _vp, _vp, _vp, _vp, ctypes.c_size_t, _vp]
_lib.conv2d_autotune.argtypes = [_P, _vp, _vp, _vp, _vp, ctypes.c_size_t, _vp, ctypes.POINTER(ctypes.c_int)]
_lib.conv2d_selected.argtypes = [_P, ctypes.POINTER(ctypes.c_int)]
_lib.conv2d_set_selected.argtypes = [_P, ctypes.c_int]
_lib.conv2d_get_variant.argtypes = [_P, ctypes.c_int, ctypes.POINTER(ctypes.c_int)]
_lib.conv2d_set_variant.argtypes = [_P, ctypes.c_int, ctypes.c_int]
_lib.conv2d_predict.argtypes = [_P, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]
_lib.conv2d_set_auto_policy.argtypes = [ctypes.c_int]
_lib.conv2d_clear_selection_cache.argtypes = []
_lib.conv2d_clear_selection_cache.restype = None
_lib.conv2d_last_tune_times.argtypes = [ctypes.POINTER(ctypes.c_double)]
_lib.conv2d_last_tune_times.restype = None
_lib.conv2d_launch_count.argtypes = [_P, ctypes.c_int]
_lib.conv2d_synth_fill.argtypes = [_vp, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int, _vp]
_lib.conv2d_status_string.argtypes = [ctypes.c_int]
_lib.conv2d_status_string.restype = ctypes.c_char_p
_lib.conv2d_algo_name.argtypes = [ctypes.c_int]
_lib.conv2d_algo_name.restype = ctypes.c_char_p
_lib.conv2d_last_error.argtypes = []
_lib.conv2d_debug_trace.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
_lib.conv2d_debug_splits.argtypes = [_P, ctypes.c_int, ctypes.POINTER(ctypes.c_int)]
_lib.conv2d_save_selection.argtypes = [ctypes.c_char_p]
_lib.conv2d_set_autotune_flush.argtypes = [_vp, ctypes.c_size_t]
_lib.conv2d_load_selection.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_int)]
_lib.conv2d_debug_trace.restype = ctypes.c_int
_lib.conv2d_last_error.restype = ctypes.c_char_p
POOL_MAX, POOL_AVG = 0, 1


class pool2d_params_t(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in (
        "batch", "in_rows", "in_cols", "channels", "window_rows", "window_cols", "stride_rows", "stride_cols",
        "padding", "op")]


_PP = ctypes.POINTER(pool2d_params_t)
_lib.pool2d_output_shape.argtypes = [_PP, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32)]
_lib.pool2d_forward.argtypes = [_PP, _vp, _vp, _vp]
for _f in ("pool2d_output_shape", "pool2d_forward", "conv2d_output_shape", "conv2d_flop_count", "conv2d_supports", "conv2d_query_workspace",
           "conv2d_forward", "conv2d_autotune", "conv2d_selected", "conv2d_set_selected",
           "conv2d_launch_count", "conv2d_synth_fill"):
    getattr(_lib, _f).restype = ctypes.c_int


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
    padding: int = PAD_SAME
    math: int = MATH_FP32

    def c(self) -> conv2d_params_t:
        return conv2d_params_t(self.batch, self.in_rows, self.in_cols, self.channels, self.features,
                               self.window_rows, self.window_cols, self.stride_rows, self.stride_cols,
                               self.padding, self.math)

    def replace(self, **kw) -> "Params":
        d = self.__dict__.copy()
        d.update(kw)
        return Params(**d)


@dataclass(frozen=True)
class PoolParams:
    """include/pool2d.h pool2d_params_t: NHWC max (POOL_MAX) / average (POOL_AVG) pooling."""
    batch: int
    in_rows: int
    in_cols: int
    channels: int
    window_rows: int
    window_cols: int
    stride_rows: int = 1
    stride_cols: int = 1
    padding: int = PAD_SAME
    op: int = POOL_MAX

    def c(self) -> pool2d_params_t:
        return pool2d_params_t(self.batch, self.in_rows, self.in_cols, self.channels, self.window_rows,
                               self.window_cols, self.stride_rows, self.stride_cols, self.padding, self.op)


def pool2d_output_shape(p: PoolParams):
    o = (ctypes.c_int32 * 4)()
    pd = (ctypes.c_int32 * 4)()
    _check(_lib.pool2d_output_shape(ctypes.byref(p.c()), o, pd), "pool2d_output_shape")
    return tuple(o), tuple(pd)


def pool2d_forward(p: PoolParams, x, y, stream=None) -> None:
    """x, y: torch CUDA tensors (or raw device pointers as ints); one kernel launch."""
    _check(_lib.pool2d_forward(ctypes.byref(p.c()), _ptr(x), _ptr(y), _stream_ptr(stream)), "pool2d_forward")


def _check(st: int, where: str):
    if st != OK:
        raise Conv2dError(st, where)


def conv2d_output_shape(p: Params):
    o = (ctypes.c_int32 * 4)()
    pd = (ctypes.c_int32 * 4)()
    _check(_lib.conv2d_output_shape(ctypes.byref(p.c()), o, pd), "conv2d_output_shape")
    return tuple(o), tuple(pd)


def conv2d_flop_count(p: Params) -> int:
    v = ctypes.c_uint64()
    _check(_lib.conv2d_flop_count(ctypes.byref(p.c()), ctypes.byref(v)), "conv2d_flop_count")
    return int(v.value)


def conv2d_supports(p: Params, algo: int) -> bool:
    v = ctypes.c_int()
    _check(_lib.conv2d_supports(ctypes.byref(p.c()), int(algo), ctypes.byref(v)), "conv2d_supports")
    return bool(v.value)


def conv2d_query_workspace(p: Params, algo: int) -> int:
    v = ctypes.c_size_t()
    _check(_lib.conv2d_query_workspace(ctypes.byref(p.c()), int(algo), ctypes.byref(v)), "conv2d_query_workspace")
    return int(v.value)


def _stream_ptr(stream):
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return getattr(stream, "cuda_stream", stream)


def _ptr(t):
    if t is None:
        return None
    return t if isinstance(t, int) else t.data_ptr()


def conv2d_forward(p: Params, algo: int, x, w, y, ws=None, ws_bytes: int | None = None, stream=None) -> None:
    """x, w, y, ws: torch CUDA tensors (or raw device pointers as ints)."""
    if ws_bytes is None:
        ws_bytes = 0 if ws is None or isinstance(ws, int) else ws.numel() * ws.element_size()
    st = _lib.conv2d_forward(ctypes.byref(p.c()), int(algo), _ptr(x), _ptr(w), _ptr(y), _ptr(ws), ws_bytes,
                             _stream_ptr(stream))
    _check(st, f"conv2d_forward({conv2d_algo_name(algo)})")


def conv2d_autotune(p: Params, x, w, y, ws=None, ws_bytes: int | None = None, stream=None) -> int:
    if ws_bytes is None:
        ws_bytes = 0 if ws is None or isinstance(ws, int) else ws.numel() * ws.element_size()
    a = ctypes.c_int()
    _check(_lib.conv2d_autotune(ctypes.byref(p.c()), _ptr(x), _ptr(w), _ptr(y), _ptr(ws), ws_bytes,
                                _stream_ptr(stream), ctypes.byref(a)), "conv2d_autotune")
    return int(a.value)


def conv2d_selected(p: Params):
    a = ctypes.c_int()
    st = _lib.conv2d_selected(ctypes.byref(p.c()), ctypes.byref(a))
    return int(a.value) if st == OK else None


def conv2d_set_selected(p: Params, algo: int) -> None:
    _check(_lib.conv2d_set_selected(ctypes.byref(p.c()), int(algo)), "conv2d_set_selected")


def conv2d_get_variant(p: Params, algo: int) -> int:
    """Tuned parameter variant of implicit_gemm / matmul_1x1 / winograd_f2x2_3x3 for p (0 = defaults;
    include/conv2d.h)."""
    v = ctypes.c_int()
    _check(_lib.conv2d_get_variant(ctypes.byref(p.c()), int(algo), ctypes.byref(v)), "conv2d_get_variant")
    return int(v.value)


def conv2d_set_variant(p: Params, algo: int, variant: int) -> None:
    _check(_lib.conv2d_set_variant(ctypes.byref(p.c()), int(algo), int(variant)), "conv2d_set_variant")


def conv2d_variants(p: Params, algo: int) -> list:
    """The parameter variants the auto-selector enumerates for (p, algo): exactly those conv2d_set_variant
    accepts (probes 0..63, restores the recorded variant)."""
    if algo not in (ALGO_IMPLICIT_GEMM, ALGO_MATMUL_1X1, ALGO_WINOGRAD_F2X2_3X3):
        return [0]
    keep = conv2d_get_variant(p, algo)
    out = []
    for v in range(64):
        if _lib.conv2d_set_variant(ctypes.byref(p.c()), int(algo), v) == OK:
            out.append(v)
    conv2d_set_variant(p, algo, keep)
    return out


AUTO_MEASURE, AUTO_PREDICT, AUTO_HYBRID = 0, 1, 2


def conv2d_predict(p: Params) -> tuple[int, int]:
    """The learned selector's (algorithm, variant) for p (include/conv2d.h; runs nothing on the device)."""
    a, v = ctypes.c_int(), ctypes.c_int()
    _check(_lib.conv2d_predict(ctypes.byref(p.c()), ctypes.byref(a), ctypes.byref(v)), "conv2d_predict")
    return int(a.value), int(v.value)


def conv2d_set_auto_policy(policy: int) -> None:
    _check(_lib.conv2d_set_auto_policy(int(policy)), "conv2d_set_auto_policy")


def conv2d_clear_selection_cache() -> None:
    _lib.conv2d_clear_selection_cache()


def conv2d_last_tune_times():
    arr = (ctypes.c_double * NUM_ALGOS)()
    _lib.conv2d_last_tune_times(arr)
    return {ALGO_NAMES[i]: arr[i] for i in range(1, NUM_ALGOS) if arr[i] >= 0}


def conv2d_launch_count(p: Params, algo: int) -> int:
    return int(_lib.conv2d_launch_count(ctypes.byref(p.c()), int(algo)))


def conv2d_synth_fill(dst, count: int, key: int, offset: int = 0, dist: int = 0, stream=None) -> None:
    _check(_lib.conv2d_synth_fill(_ptr(dst), count, key, offset, dist, _stream_ptr(stream)), "conv2d_synth_fill")


def conv2d_algo_name(a: int) -> str:
    return _lib.conv2d_algo_name(int(a)).decode()


def conv2d_status_string(s: int) -> str:
    return _lib.conv2d_status_string(int(s)).decode()


def conv2d_last_error() -> str:
    return _lib.conv2d_last_error().decode()


def conv2d_set_autotune_flush(buf, nbytes: int | None = None) -> None:
    """Register (or with buf=None clear) a device scratch buffer the auto-selector overwrites before every
    timed repetition (cache-cold tuning).  buf: torch CUDA tensor or raw pointer."""
    if buf is None:
        _check(_lib.conv2d_set_autotune_flush(None, 0), "conv2d_set_autotune_flush")
        return
    if nbytes is None:
        nbytes = buf.numel() * buf.element_size()
    _check(_lib.conv2d_set_autotune_flush(_ptr(buf), int(nbytes)), "conv2d_set_autotune_flush")


def conv2d_save_selection(path: str) -> None:
    _check(_lib.conv2d_save_selection(str(path).encode()), "conv2d_save_selection")


def conv2d_load_selection(path: str) -> int:
    n = ctypes.c_int(0)
    _check(_lib.conv2d_load_selection(str(path).encode(), ctypes.byref(n)), "conv2d_load_selection")
    return n.value


def conv2d_debug_trace(enable: int, read: bool = False) -> list:
    """include/conv2d_debug.h: toggle the GEMM kernels' per-CTA globaltimer stamps; with read=True
    returns the 256 launch records x 148 CTAs x 8 stamps (ns) as a flat list."""
    n = 256 * 148 * 8
    buf = (ctypes.c_ulonglong * n)() if read else None
    got = _lib.conv2d_debug_trace(int(enable), buf, n if read else 0)
    if got < 0:
        raise RuntimeError("conv2d_debug_trace failed")
    return list(buf[:got]) if read else []


def conv2d_debug_splits(p: Params, algo: int) -> int:
    """include/conv2d_debug.h: K-split of the plan conv2d_forward(p, algo) would run now (1 = none)."""
    v = ctypes.c_int()
    _check(_lib.conv2d_debug_splits(ctypes.byref(p.c()), int(algo), ctypes.byref(v)), "conv2d_debug_splits")
    return int(v.value)


# ------------------------------------------------------------------ convenience (torch in, torch out)
def params_for(x, w, stride=(1, 1), padding: int = PAD_SAME, math: int = MATH_FP32) -> Params:
    n, h, wd, c = x.shape
    kh, kw, c2, f = w.shape
    if c != c2:
        raise ValueError(f"channel mismatch: input C={c}, filter C={c2}")
    return Params(n, h, wd, c, f, kh, kw, stride[0], stride[1], padding, math)


def forward(x, w, stride=(1, 1), padding: int = PAD_SAME, algo: int = ALGO_AUTO, math: int = MATH_FP32,
            out=None, workspace=None, stream=None):
    """y = conv2d(x NHWC fp32 CUDA, w HWCF fp32 CUDA) through conv2d_forward."""
    import torch
    p = params_for(x, w, stride, padding, math)
    (n, ho, wo, f), _ = conv2d_output_shape(p)
    if not (x.is_cuda and w.is_cuda and x.dtype == torch.float32 and w.dtype == torch.float32):
        raise ValueError("x and w must be float32 CUDA tensors")
    if w.device != x.device:
        raise ValueError(f"x is on {x.device} but w is on {w.device}")
    if out is not None:  # the kernels write n*ho*wo*f dense floats from out's base pointer
        if (tuple(out.shape) != (n, ho, wo, f) or out.dtype != torch.float32 or not out.is_contiguous()
                or out.device != x.device):
            raise ValueError(f"out must be a contiguous float32 tensor of shape {(n, ho, wo, f)} on {x.device}; "
                             f"got {tuple(out.shape)} {out.dtype} on {out.device} (contiguous={out.is_contiguous()})")
    if workspace is not None and workspace.device != x.device:
        raise ValueError(f"workspace is on {workspace.device}, not {x.device}")
    x = x.contiguous()
    w = w.contiguous()
    with torch.cuda.device(x.device):  # launch on x's GPU, on that device's current stream by default
        y = out if out is not None else torch.empty((n, ho, wo, f), dtype=torch.float32, device=x.device)
        need = conv2d_query_workspace(p, algo)
        if workspace is None or workspace.numel() * workspace.element_size() < need:
            workspace = torch.empty(max(need, 16), dtype=torch.uint8, device=x.device) if need else None
        conv2d_forward(p, algo, x, w, y, workspace, need if workspace is not None else 0,
                       stream if stream is not None else torch.cuda.current_stream(x.device))
    return y
