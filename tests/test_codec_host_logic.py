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
    f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
    L.zb_encode_block64.argtypes = [f64p, C.c_int, u64p]
    u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
    L.zb_encode_ints_rows.argtypes = [u32p, C.c_int, C.c_int, u64p]
    L.zb_encode_ints64_rows.argtypes = [u64p, C.c_int, C.c_int, u64p]
    L.zb_decode_block64.argtypes = [u64p, C.c_int, f64p]
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


def _blocks64(n, seed):
    """fp64 blocks: wide dynamic range, denormals, constants, fp32-promoted data."""
    rng = np.random.default_rng(seed)
    out = np.zeros((n, 64))
    f32 = synth.random_blocks(n, seed=seed + 1)
    for b in range(n):
        kind = b % 6
        if kind == 0:
            out[b] = rng.standard_normal(64) * 2.0 ** rng.integers(-900, 900)
        elif kind == 1:
            out[b] = rng.standard_normal(64) * 2.0 ** rng.integers(-1000, 1000, 64)
        elif kind == 2:
            out[b] = rng.integers(-(1 << 52), 1 << 52, 64).astype(np.float64) * 2.0 ** -1074
        elif kind == 3:
            out[b] = rng.standard_normal() * 2.0 ** rng.integers(-1074, 1000)
        elif kind == 4:
            out[b] = rng.standard_normal(64) * 2.0 ** rng.integers(-1060, -940)   # slow dequant path
        else:
            out[b] = f32[b].astype(np.float64)
    return out


def test_encode64_matches_oracle(zb):
    for n, b in enumerate(_blocks64(900, 41)):
        for rate in RATES[n % 3::3]:
            want, _ = oracle.encode_block64(b, rate)
            got = np.zeros(rate, np.uint64)
            zb.zb_encode_block64(np.ascontiguousarray(b), rate, got)
            assert np.array_equal(got, want), (n, rate)


def test_decode64_matches_oracle(zb):
    rng = np.random.default_rng(42)
    blocks = _blocks64(600, 43)
    for n in range(1800):
        rate = int(RATES[n % len(RATES)])
        if n < 600:
            words, _ = oracle.encode_block64(blocks[n], rate)
        else:                  # arbitrary bit patterns (budget ends anywhere)
            words = rng.integers(0, 1 << 63, rate, dtype=np.uint64) * 2 + rng.integers(0, 2, rate, dtype=np.uint64)
            if n % 5 == 0:
                words &= rng.integers(0, 1 << 63, rate, dtype=np.uint64)
                words[0] |= 1
        want, _ = oracle.decode_block64(words, rate)
        got = np.zeros(64)
        zb.zb_decode_block64(words, rate, got)
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), (n, rate)


def _adversarial_ints(n, seed, bits):
    """Negabinary coefficient sets that make the plane coder emit as much as
    possible as early as possible (dense top planes: up to 129 bits for the
    first plane) -- the worst case of the encoder's overlapped shared-memory
    row, where the stream is written over planes already consumed."""
    rng = np.random.default_rng(seed)
    top = (1 << bits) - 1
    out = []
    for b in range(n):
        kind = b % 5
        if kind == 0:
            u = np.full(64, top, dtype=np.uint64)                       # every plane all ones
        elif kind == 1:
            u = rng.integers(0, 1 << 62, 64, dtype=np.uint64) * 4 + rng.integers(0, 4, 64, dtype=np.uint64)
        elif kind == 2:                                                 # top bit set everywhere, rest random
            u = (rng.integers(0, 1 << 62, 64, dtype=np.uint64) | np.uint64(1 << (bits - 1)))
        elif kind == 3:                                                 # alternating dense / empty planes
            u = np.full(64, int("10" * 32, 2) & top, dtype=np.uint64)
        else:                                                           # ones arriving one per plane
            u = np.zeros(64, np.uint64)
            for i in range(64):
                u[i] = np.uint64(1 << max(bits - 1 - i % bits, 0))
        out.append(u & np.uint64(top))
    return out


def _bits_after(words, header, budget):
    """stream bits [header, header + budget) of a row of words, as an int"""
    v = 0
    for i, w in enumerate(words):
        v |= int(w) << (64 * i)
    return (v >> header) & ((1 << budget) - 1)


def _as_int(words):
    v = 0
    for i, w in enumerate(words):
        v |= int(w) << (64 * i)
    return v


@pytest.mark.parametrize("precision", [32, 64])
def test_plane_coder_overlapped_row_worst_cases(zb, precision):
    bits, header = (32, 9) if precision == 32 else (64, 12)
    for n, u in enumerate(_adversarial_ints(200, 51 + precision, bits)):
        for rate in RATES[n % 2::2]:
            budget = 64 * rate - header
            got = np.zeros(rate, np.uint64)
            if precision == 32:
                zb.zb_encode_ints_rows(np.ascontiguousarray(u.astype(np.uint32)), header, rate, got)
                want, _ = oracle.encode_ints(u.astype(np.uint32), budget)
            else:
                zb.zb_encode_ints64_rows(np.ascontiguousarray(u), header, rate, got)
                want, _ = oracle.encode_ints64(u, budget)
            assert _bits_after(got, header, budget) == _as_int(want) & ((1 << budget) - 1), (n, rate)
            assert _as_int(got) & ((1 << header) - 1) == 0
