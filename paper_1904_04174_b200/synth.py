"""Seeded synthetic inputs shared by the tests, the bench and smoke().

This module holds NONE of the method's arithmetic: it only draws numbers.  It
is the single module both the oracle side and the CUDA side receive inputs
from (SURVEY.md §8(c) reading A15).

Generator (counter-based splitmix64, so any element -- or a shard of a batch --
can be produced independently of the others):

    sm64(z): z += 0x9E3779B97F4A7C15
             z  = (z ^ z>>30) * 0xBF58476D1CE4E5B9
             z  = (z ^ z>>27) * 0x94D049BB133111EB
             return z ^ z>>31
    key  S  = sm64(seed ^ (layer_id << 40) ^ (role << 32))   role 0 = input, 1 = filter
    elem i  : u = sm64(S + i) >> 40            (24 random bits; i = global linear index)
    uniform : x = u * 2^-23 - 1  in [-1, 1 - 2^-23], exact in fp32   (SPEC.md:66-74 range)
    integer : x = (u mod 5) - 2  in {-2..2}  (exact-arithmetic regime)

The same generator is implemented on the device by ``conv2d_synth_fill`` in
the product library (it is not part of the conv path; it only lets bench.py
fill multi-GB batches quickly).  tests/test_synth.py checks the two agree.
"""
from __future__ import annotations

import numpy as np

SEED = 1904_04174
ROLE_INPUT, ROLE_FILTER = 0, 1
DIST_UNIFORM, DIST_INT5 = 0, 1

_M = np.uint64(0xFFFFFFFFFFFFFFFF)
_G = np.uint64(0x9E3779B97F4A7C15)
_C1 = np.uint64(0xBF58476D1CE4E5B9)
_C2 = np.uint64(0x94D049BB133111EB)


def _sm64(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = z + _G
        z = (z ^ (z >> np.uint64(30))) * _C1
        z = (z ^ (z >> np.uint64(27))) * _C2
        return z ^ (z >> np.uint64(31))


def stream_key(seed: int, layer_id: int, role: int) -> int:
    z = np.array([(seed ^ (layer_id << 40) ^ (role << 32)) & 0xFFFFFFFFFFFFFFFF], dtype=np.uint64)
    return int(_sm64(z)[0])


def draw(count: int, key: int, offset: int = 0, dist: int = DIST_UNIFORM, chunk: int = 1 << 24) -> np.ndarray:
    """Elements [offset, offset+count) of stream ``key`` as float32."""
    out = np.empty(count, dtype=np.float32)
    k = np.uint64(key)
    for s in range(0, count, chunk):
        n = min(chunk, count - s)
        i = np.arange(offset + s, offset + s + n, dtype=np.uint64)
        with np.errstate(over="ignore"):
            u = _sm64(i + k) >> np.uint64(40)
        if dist == DIST_UNIFORM:
            out[s:s + n] = (u.astype(np.int64) - (1 << 23)).astype(np.float32) * np.float32(2.0 ** -23)
        else:
            out[s:s + n] = ((u % np.uint64(5)).astype(np.int64) - 2).astype(np.float32)
    return out


def input_nhwc(n: int, h: int, w: int, c: int, layer_id: int = 0, seed: int = SEED,
               dist: int = DIST_UNIFORM, batch_offset: int = 0) -> np.ndarray:
    """Images [batch_offset, batch_offset+n) of the global seeded NHWC input (shards are exact slices)."""
    per = h * w * c
    key = stream_key(seed, layer_id, ROLE_INPUT)
    return draw(n * per, key, batch_offset * per, dist).reshape(n, h, w, c)


def filter_hwcf(kh: int, kw: int, c: int, f: int, layer_id: int = 0, seed: int = SEED,
                dist: int = DIST_UNIFORM) -> np.ndarray:
    key = stream_key(seed, layer_id, ROLE_FILTER)
    return draw(kh * kw * c * f, key, 0, dist).reshape(kh, kw, c, f)
