"""The seeded input generator (SPEC.md:66-74 determinism/range contract, reading A15)."""
import numpy as np

from paper_1904_04174_b200 import synth


def test_determinism_and_range():
    a = synth.input_nhwc(2, 5, 5, 3, layer_id=1)
    b = synth.input_nhwc(2, 5, 5, 3, layer_id=1)
    assert np.array_equal(a, b)
    c = synth.input_nhwc(2, 5, 5, 3, layer_id=2)
    assert not np.array_equal(a, c)
    f = synth.filter_hwcf(3, 3, 3, 4, layer_id=1)
    assert not np.array_equal(a.reshape(-1)[:36], f.reshape(-1)[:36])  # roles are distinct streams
    big = synth.draw(1 << 20, synth.stream_key(synth.SEED, 0, 0))
    assert big.min() >= -1.0 and big.max() <= 1.0 - 2.0 ** -23
    assert abs(float(big.mean())) < 5e-3 and big.dtype == np.float32
    # values are exact multiples of 2^-23
    assert np.all((big.astype(np.float64) * 2 ** 23) == np.round(big.astype(np.float64) * 2 ** 23))


def test_int_distribution():
    v = synth.draw(100000, synth.stream_key(synth.SEED, 3, 0), dist=synth.DIST_INT5)
    assert set(np.unique(v).tolist()) == {-2.0, -1.0, 0.0, 1.0, 2.0}


def test_shards_are_exact_slices():
    full = synth.input_nhwc(8, 4, 3, 5, layer_id=7)
    for g in (2, 4, 8):
        per = 8 // g
        for r in range(g):
            sl = synth.input_nhwc(per, 4, 3, 5, layer_id=7, batch_offset=r * per)
            assert np.array_equal(sl, full[r * per:(r + 1) * per])


def test_splitmix_reference_value():
    # splitmix64 first output for state 0 is 0xE220A8397B1DCDAF (Vigna's reference implementation)
    z = np.array([0], dtype=np.uint64)
    assert int(synth._sm64(z)[0]) == 0xE220A8397B1DCDAF
