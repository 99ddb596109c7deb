"""GPU codec parity: oocz_zfp_encode / oocz_zfp_decode (CUDA, sm_100a) vs the
bit-serial CPU oracle.  Bar: bit-exact streams and bit-exact fp32 output."""
import numpy as np
import pytest

import oracle
from paper_2109_05410_b200 import synth
from gpu_util import bits, gpu_decode, gpu_encode

pytestmark = pytest.mark.gpu


def _fields():
    rb = synth.random_blocks(5 * 3 * 7, seed=41)
    return {
        "c1_pulse": synth.pulse(64, 64, 64, sigma=4.0),          # C1 (BASELINE configs[0])
        "dense": synth.dense(48, 36, 20, seed=1),
        "layered": synth.layered(40, 24, 16),
        "adversarial": synth.blocks_to_field(rb, 5, 3, 7),       # ragged: 105 blocks < 128 per CTA
        "zeros": np.zeros((8, 8, 8), np.float32),
        "wide": synth.dense(1032, 8, 4, seed=2),                  # 258 blocks: 3 CTAs, ragged tail
        # white noise: every coefficient significant within the first planes, the
        # densest early planes -- the worst case of the encoder's overlapped
        # shared-memory row (planes and stream in one row, zfp.cu)
        "noise": np.random.default_rng(43).uniform(-1, 1, (16, 16, 32)).astype(np.float32),
        "noise_signs": (np.random.default_rng(44).integers(0, 2, (8, 8, 64)) * 2 - 1).astype(np.float32),
    }


@pytest.mark.parametrize("rate", [1, 4, 8, 12, 16, 24, 32, 40, 64])
def test_encode_bit_exact(rate):
    for name, f in _fields().items():
        want = oracle.zfp_encode(f, rate)
        got = gpu_encode(f, rate)
        assert got.shape == want.shape, name
        bad = np.nonzero(got != want)[0]
        assert bad.size == 0, (name, rate, bad[:5])


@pytest.mark.parametrize("rate", [1, 8, 12, 16, 24, 33, 64])
def test_decode_bit_exact(rate):
    for name, f in _fields().items():
        words = oracle.zfp_encode(f, rate)
        want = oracle.zfp_decode(words, f.shape, rate)
        got = gpu_decode(words, f.shape, rate)
        assert np.array_equal(bits(got), bits(want)), (name, rate)


@pytest.mark.parametrize("rate", [2, 7, 16, 31, 64])
def test_decode_arbitrary_streams_bit_exact(rate):
    rng = np.random.default_rng(rate)
    shape = (12, 16, 20)
    n = oracle.zfp_bytes(20, 16, 12, rate) // 8
    for trial in range(4):
        words = rng.integers(0, 1 << 63, n, dtype=np.uint64) * 2 + rng.integers(0, 2, n, dtype=np.uint64)
        if trial % 2:
            words &= rng.integers(0, 1 << 63, n, dtype=np.uint64)
            words |= np.uint64(1)
        want = oracle.zfp_decode(words, shape, rate)
        got = gpu_decode(words, shape, rate)
        assert np.array_equal(bits(got), bits(want)), (rate, trial)


def test_c2_full_size_stream_bit_exact():
    """BASELINE configs[1] size (512^3) at rate 16: the whole stream."""
    f = synth.dense(512, 512, 512, seed=1)
    want = oracle.zfp_encode(f, 16)
    got = gpu_encode(f, 16)
    assert got.nbytes == 256 << 20
    assert np.array_equal(got, want)
    back = gpu_decode(got, f.shape, 16)
    ref = oracle.zfp_decode(want, f.shape, 16)
    assert np.array_equal(bits(back), bits(ref))


def test_round_trip_error_small_at_rate_24():
    f = synth.dense(64, 64, 64, seed=3)
    g = gpu_decode(gpu_encode(f, 24), f.shape, 24)
    assert np.abs(g - f).max() <= 1e-5 * np.abs(f).max()


@pytest.mark.parametrize("seed", [21, 22])
def test_random_shapes_and_rates_bit_exact(seed):
    """Seeded random shapes (multiples of 4, ragged CTA counts) and rates 1..64:
    streams and decoded fields bit-exact against the oracle."""
    rng = np.random.default_rng(seed)
    for case in range(12):
        nx, ny, nz = (4 * int(rng.integers(1, 24)) for _ in range(3))
        rate = int(rng.integers(1, 65))
        f = synth.dense(nx, ny, nz, seed=300 + case) * np.float32(10.0 ** int(rng.integers(-30, 30)))
        f = f.astype(np.float32)
        want = oracle.zfp_encode(f, rate)
        got = gpu_encode(f, rate)
        assert np.array_equal(got, want), (nx, ny, nz, rate)
        back = gpu_decode(got, f.shape, rate)
        assert np.array_equal(bits(back), bits(oracle.zfp_decode(want, f.shape, rate))), (nx, ny, nz, rate)
