"""Randomized GPU codec parity beyond the test suite: seeded random shapes
(multiples of 4, up to a few CTAs with ragged tails), rates 1..64 and value
distributions (smooth, white noise, sparse, huge / tiny / denormal scales,
constants, mixed signs), fp32 and fp64; every stream and decoded field
bit-exact against the oracle.

  python tools/codec_random.py [cases] [seed]
"""
import os
import sys
import time

import numpy as np

R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(R, "tests"))
sys.path.insert(0, R)
import oracle  # noqa: E402  (test infrastructure)
from gpu_util import bits, gpu_decode, gpu_encode  # noqa: E402
from paper_2109_05410_b200 import synth  # noqa: E402


def field(rng, shape, kind):
    n = int(np.prod(shape))
    if kind == 0:
        return synth.dense(shape[2], shape[1], shape[0], seed=int(rng.integers(1, 1000)))
    if kind == 1:
        return rng.uniform(-1, 1, shape).astype(np.float32)
    if kind == 2:
        f = np.zeros(n, np.float32)
        idx = rng.integers(0, n, max(1, n // 50))
        f[idx] = rng.standard_normal(idx.size).astype(np.float32)
        return f.reshape(shape)
    if kind == 3:
        return (rng.standard_normal(shape) * 10.0 ** float(rng.integers(-44, 38))).astype(np.float32)
    if kind == 4:
        return np.full(shape, np.float32(rng.standard_normal()), np.float32)
    return (rng.integers(-3, 4, shape) * 2.0 ** float(rng.integers(-140, 100))).astype(np.float32)


def main():
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 300
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 7
    rng = np.random.default_rng(seed)
    t0 = time.time()
    for c in range(cases):
        shape = tuple(4 * int(rng.integers(1, 12)) for _ in range(3))
        rate = int(rng.integers(1, 65))
        f = field(rng, shape, c % 6)
        want = oracle.zfp_encode(f, rate)
        got = gpu_encode(f, rate)
        assert np.array_equal(got, want), ("encode", c, shape, rate, c % 6)
        back = gpu_decode(got, f.shape, rate)
        assert np.array_equal(bits(back), bits(oracle.zfp_decode(want, f.shape, rate))), ("decode", c, shape, rate)
        if c % 3 == 0:          # arbitrary streams: the budget ends anywhere
            words = rng.integers(0, 1 << 63, want.size, dtype=np.uint64) * 2 + rng.integers(0, 2, want.size, dtype=np.uint64)
            assert np.array_equal(bits(gpu_decode(words, f.shape, rate)),
                                  bits(oracle.zfp_decode(words, f.shape, rate))), ("arbitrary", c, shape, rate)
    print(f"codec random: {cases} cases (seed {seed}) bit-exact, {time.time() - t0:.1f} s", flush=True)


if __name__ == "__main__":
    main()
