"""CPU check of the CUDA path's word-parallel block coder (csrc/zfp_block.cuh,
compiled for the host by tests/native/zb_host.cpp) against the bit-serial
oracle.  The GPU kernels wrap exactly this per-block logic; the -m gpu tests
then check the kernels themselves bit for bit."""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

import oracle
from paper_2109_05410_b200 import synth

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "native", "zb_host.cpp")
LIB = os.path.join(HERE, "native", "libzb_host.so")


@pytest.fixture(scope="module")
def zb():
    hdr = os.path.join(HERE, "..", "paper_2109_05410_b200", "csrc", "zfp_block.cuh")
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(SRC), os.path.getmtime(hdr)):
        subprocess.run(["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-ffp-contract=off",
                        "-x", "c++", SRC, "-o", LIB], check=True)
    L = C.CDLL(LIB)
    f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
    u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
    L.zb_encode_block.argtypes = [f32p, C.c_int, u64p]
    L.zb_decode_block.argtypes = [u64p, C.c_int, f32p]
    return L


RATES = [1, 2, 3, 5, 8, 12, 16, 24, 32, 33, 34, 48, 64]


def test_encode_matches_oracle(zb):
    blocks = synth.random_blocks(1600, seed=31)
    for n, b in enumerate(blocks):
        for rate in RATES[n % 3::3]:
            want, _ = oracle.encode_block(b, rate)
            got = np.zeros(rate, np.uint64)
            zb.zb_encode_block(np.ascontiguousarray(b), rate, got)
            assert np.array_equal(got, want), (n, rate)


def test_decode_matches_oracle_on_valid_streams(zb):
    blocks = synth.random_blocks(800, seed=32)
    for n, b in enumerate(blocks):
        for rate in RATES[n % 4::4]:
            words, _ = oracle.encode_block(b, rate)
            want, _ = oracle.decode_block(words, rate)
            got = np.zeros(64, np.float32)
            zb.zb_decode_block(words, rate, got)
            assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), (n, rate)


def test_decode_matches_oracle_on_arbitrary_bits(zb):
    # any bit pattern is a decodable stream: exercises budget exhaustion
    # inside group tests, the implied bit at position 63 and wraparound
    rng = np.random.default_rng(33)
    for n in range(3000):
        rate = int(RATES[n % len(RATES)])
        words = rng.integers(0, 1 << 63, rate, dtype=np.uint64) * 2 + rng.integers(0, 2, rate, dtype=np.uint64)
        if n % 5 == 0:    # sparse streams: long zero runs
            words &= rng.integers(0, 1 << 63, rate, dtype=np.uint64) & rng.integers(0, 1 << 63, rate, dtype=np.uint64)
            words[0] |= 1
        want, _ = oracle.decode_block(words, rate)
        got = np.zeros(64, np.float32)
        zb.zb_decode_block(words, rate, got)
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), (n, rate)
