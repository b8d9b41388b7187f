"""GPU parity of NHWC max / average pooling (include/pool2d.h) against the pooling
oracle (oracle/pool.c) through the C-ABI.  Both operations are bit-exact by construction (max is a
selection; the average sums in double in the oracle's order and rounds once), so every comparison
is array_equal, with outputs poisoned (NaN) before each call."""
import numpy as np
import pytest

import oracle as O
from paper_1904_04174_b200 import synth

from .parity import C

pytestmark = pytest.mark.gpu

CASES = [
    (256 // 64, 112, 112, 64, 3, 3, 2, 2, 0),   # ResNet-50 stem max pool (b4 slice)
    (2, 224, 224, 64, 2, 2, 2, 2, 1),           # VGG pool1
    (2, 28, 28, 512, 2, 2, 2, 2, 1),            # VGG pool4
    (4, 7, 7, 2048, 7, 7, 1, 1, 1),             # ResNet-50 global average pool (as a 7x7 VALID window)
    (3, 13, 11, 5, 3, 3, 2, 2, 0),              # C % 4 != 0: scalar path, SAME corners
    (1, 9, 10, 8, 4, 2, 3, 1, 0),               # non-square window / stride
    (2, 17, 5, 12, 5, 3, 2, 2, 0),
    (1, 1, 1, 4, 1, 1, 1, 1, 0),                # single element
    (1, 6, 6, 4, 1, 1, 2, 2, 0),                # stride > window
    (5, 3, 4, 3, 3, 4, 1, 1, 1),                # VALID window = whole image
]


def _gpu_pool(p, x, offset_floats=0):
    import torch
    c = C()
    (n, ho, wo, ch), _ = c.pool2d_output_shape(p)
    xd = torch.zeros(x.size + offset_floats, dtype=torch.float32, device="cuda")
    xd[offset_floats:] = torch.from_numpy(x.ravel()).cuda()
    y = torch.full((n * ho * wo * ch + offset_floats,), float("nan"), dtype=torch.float32, device="cuda")
    c.pool2d_forward(p, xd.data_ptr() + 4 * offset_floats, y.data_ptr() + 4 * offset_floats)
    torch.cuda.synchronize()
    return y[offset_floats:].cpu().numpy().reshape(n, ho, wo, ch)


@pytest.mark.parametrize("case", CASES, ids=str)
@pytest.mark.parametrize("op", [0, 1], ids=["max", "avg"])
def test_pool_bit_exact(cuda_ok, case, op):
    n, h, w, ch, kh, kw, sh, sw, pad = case
    c = C()
    p = c.PoolParams(n, h, w, ch, kh, kw, sh, sw, pad, op)
    x = synth.input_nhwc(n, h, w, ch, layer_id=1100 + op)
    ref = O.pool2d(O.PoolParams(n, h, w, ch, kh, kw, sh, sw, pad, op), x)
    got = _gpu_pool(p, x)
    assert np.array_equal(got, ref), (case, op, float(np.nanmax(np.abs(got - ref))))


@pytest.mark.parametrize("op", [0, 1], ids=["max", "avg"])
def test_pool_unaligned_pointers_take_the_scalar_path(cuda_ok, op):
    c = C()
    n, h, w, ch = 2, 15, 13, 16
    p = c.PoolParams(n, h, w, ch, 3, 3, 2, 2, 0, op)
    x = synth.input_nhwc(n, h, w, ch, layer_id=1110)
    ref = O.pool2d(O.PoolParams(n, h, w, ch, 3, 3, 2, 2, 0, op), x)
    assert np.array_equal(_gpu_pool(p, x, offset_floats=1), ref)


def test_pool_resnet_stem_b256_sampled_images(cuda_ok):
    """Full size (BASELINE config 5 batch): the stem max pool over 256 x 112 x 112 x 64 generated on the
    device; images 0, 1, 128, 255 recomputed by the oracle from the host twin of the generator."""
    import torch
    c = C()
    n, h, w, ch = 256, 112, 112, 64
    key = synth.stream_key(synth.SEED, 1120, synth.ROLE_INPUT)
    x = torch.empty(n * h * w * ch, dtype=torch.float32, device="cuda")
    c.conv2d_synth_fill(x, x.numel(), key, 0, 0)
    for op in (0, 1):
        p = c.PoolParams(n, h, w, ch, 3, 3, 2, 2, 0, op)
        (_, ho, wo, _), _ = c.pool2d_output_shape(p)
        y = torch.full((n * ho * wo * ch,), float("nan"), dtype=torch.float32, device="cuda")
        c.pool2d_forward(p, x, y)
        torch.cuda.synchronize()
        yh = y.view(n, ho, wo, ch)
        for img in (0, 1, 128, 255):
            xi = synth.input_nhwc(1, h, w, ch, layer_id=1120, batch_offset=img)
            ref = O.pool2d(O.PoolParams(1, h, w, ch, 3, 3, 2, 2, 0, op), xi)
            assert np.array_equal(yh[img:img + 1].cpu().numpy(), ref), (op, img)
