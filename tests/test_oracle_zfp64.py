"""Pins for the oracle's fp64 fixed-rate coder (oracle/zfp_ref64.c): the
paper's own precision at its rates (32/64, 24/64).
Closed forms, hand derivations and invariants only (zfp itself: unpinned)."""
from fractions import Fraction

import numpy as np
import pytest

import oracle
from paper_2109_05410_b200 import synth


def _blocks64(n, seed):
    rng = np.random.default_rng(seed)
    out = np.zeros((n, 64))
    for b in range(n):
        kind = b % 6
        if kind == 0:
            out[b] = rng.standard_normal(64) * 2.0 ** rng.integers(-900, 900)
        elif kind == 1:
            out[b] = rng.standard_normal(64) * 2.0 ** rng.integers(-1000, 1000, 64)
        elif kind == 2:      # denormal doubles
            out[b] = rng.integers(-(1 << 52), 1 << 52, 64).astype(np.float64) * 2.0 ** -1074
        elif kind == 3:
            out[b] = rng.standard_normal() * 2.0 ** rng.integers(-1074, 1000)
        elif kind == 4:      # smooth
            i, j, k = np.meshgrid(np.arange(4), np.arange(4), np.arange(4), indexing="xy")
            g = rng.standard_normal(4)
            out[b] = (g[0] + g[1] * i + g[2] * j + g[3] * k).reshape(64)
        else:                # fp32 data promoted (the fp32 workload in fp64)
            out[b] = synth.random_blocks(1, seed=int(rng.integers(1 << 30)))[0].astype(np.float64)
    return out


def test_sizes_are_the_fixed_rate_contract():
    for rate in (1, 24, 32, 64):
        w = oracle.zfp_encode64(np.zeros((8, 8, 8)), rate)
        assert w.nbytes == 8 * 8 * rate


def test_constant_one_hand_derived():
    # emax = 1 -> e = 1024, 12 header bits 2e+1 = 0x801; q = 2^61 everywhere, DC only;
    # negabinary(2^61) has bits 61, 62: plane 63 flag 0 (1), plane 62 "1,1,0" (3),
    # plane 61 verbatim 1 + flag 0 (2), planes 60..0 "0,0" (122): 140 bits,
    # word0 = 0x801 | 0x6000 | 0x10000 = 0x16801
    w, used = oracle.encode_block64(np.ones(64), 16)
    assert used == 140 and int(w[0]) == 0x16801 and not w[1:].any()
    # -1.0: negabinary(-2^61) is bit 61 alone: 12 + 1 + 1 + 3 + 122 = 139 bits, 0xc801
    w, used = oracle.encode_block64(-np.ones(64), 16)
    assert used == 139 and int(w[0]) == 0xC801 and not w[1:].any()


def test_zero_blocks():
    for v in (0.0, -0.0):
        w, used = oracle.encode_block64(np.full(64, v), 8)
        assert used == 1 and not w.any()
        x, _ = oracle.decode_block64(w, 8)
        assert not x.view(np.uint64).any()


def test_constants_exact_from_rate_3():
    rng = np.random.default_rng(3)
    vals = list(rng.standard_normal(30) * 2.0 ** rng.integers(-1074, 1000, 30)) + [5e-324, -1.7e308, 1.0]
    for v in vals:
        for rate in (3, 8, 32):
            w, _ = oracle.encode_block64(np.full(64, v), rate)
            x, _ = oracle.decode_block64(w, rate)
            assert (x.view(np.uint64) == np.float64(v).view(np.uint64)).all(), (v, rate)


def test_negabinary64_is_base_minus_two():
    rng = np.random.default_rng(4)
    for x in list(rng.integers(-(1 << 62), 1 << 62, 500)) + [0, 1, -1, 2, -2]:
        u = oracle.int2uint64(int(x))
        assert sum(((u >> i) & 1) * (-2) ** i for i in range(64)) == int(x)
        assert oracle.uint2int64(u) == int(x)
    assert [oracle.int2uint64(v) for v in (0, 1, -1, 2, -2)] == [0, 1, 3, 6, 2]


A = [[4, 4, 4, 4], [5, 1, -1, -5], [-4, 4, 4, -4], [-2, 6, -6, 2]]
B = [[4, 6, -4, -1], [4, 2, 4, 5], [4, -2, 4, -5], [4, -6, -4, 1]]


def test_lifting64_matrices_on_divisible_input():
    rng = np.random.default_rng(5)
    for _ in range(300):
        v = [int(t) * 64 for t in rng.integers(-(1 << 50), 1 << 50, 4)]
        got = oracle.fwd_lift64(v)
        assert [Fraction(int(g)) for g in got] == [sum(Fraction(A[r][c], 16) * v[c] for c in range(4))
                                                  for r in range(4)]
        got = oracle.inv_lift64(v)
        assert [Fraction(int(g)) for g in got] == [sum(Fraction(B[r][c], 4) * v[c] for c in range(4))
                                                  for r in range(4)]


def test_xform64_delta_and_guard_bits():
    q = np.zeros(64, np.int64)
    q[0] = 1 << 61
    got = oracle.fwd_xform64(q).reshape(4, 4, 4).astype(object)
    col = [Fraction(4, 16), Fraction(5, 16), Fraction(-4, 16), Fraction(-2, 16)]
    for k in range(4):
        for j in range(4):
            for i in range(4):
                assert got[k, j, i] == (1 << 61) * col[k] * col[j] * col[i]
    rng = np.random.default_rng(6)
    for _ in range(500):
        q = rng.integers(-(1 << 62) + 1, 1 << 62, 64)
        c = oracle.fwd_xform64(q)
        assert int(np.abs(c.astype(object)).max()) < (1 << 63)


def _closed_form_bits64(u):
    n, total = 0, 0
    for k in range(63, -1, -1):
        x = sum(((int(u[i]) >> k) & 1) << i for i in range(64))
        if n == 64:
            total += 64
            continue
        xs = x >> n
        if xs == 0:
            total += n + 1
            continue
        top = x.bit_length() - 1
        j = bin(xs).count("1")
        total += n + j + (top - n + 1) - (1 if top == 63 else 0) + (1 if top < 63 else 0)
        n = top + 1
    return total


def test_code_length_closed_form_and_lossless_when_it_fits():
    rng = np.random.default_rng(7)
    cases = [rng.integers(0, 1 << 63, 64, dtype=np.uint64) << np.uint64(1) for _ in range(10)]
    for b in _blocks64(24, 8):
        e = oracle.exponent_max64(b)
        if e == -1023:
            continue
        q = oracle.fwd_xform64(oracle.fwd_cast64(b, e))
        cases.append(np.array([oracle.int2uint64(int(q[p])) for p in oracle.perm3()], np.uint64))
    for u in cases:
        want = _closed_form_bits64(u)
        words, used = oracle.encode_ints64(u, 8192)
        assert used == want
        d, _ = oracle.decode_ints64(words, 8192)
        assert np.array_equal(d, u)


def test_embedded_prefix_and_locality():
    for b in _blocks64(60, 9):
        streams = {r: oracle.encode_block64(b, r)[0] for r in (2, 12, 24, 32, 64)}
        rates = sorted(streams)
        for lo, hi in zip(rates, rates[1:]):
            bl = np.unpackbits(streams[lo].view(np.uint8), bitorder="little")
            bh = np.unpackbits(streams[hi].view(np.uint8), bitorder="little")[: 64 * lo]
            assert np.array_equal(bl, bh)
    f = synth.dense(16, 16, 16, seed=2).astype(np.float64)
    w1 = oracle.zfp_encode64(f, 24)
    g = f.copy()
    g[6, 1, 13] += 1.0                                   # block bx=3, by=0, bz=1
    diff = np.nonzero((w1 != oracle.zfp_encode64(g, 24)).reshape(-1, 24).any(axis=1))[0]
    assert diff.tolist() == [3 + 4 * (0 + 4 * 1)]


def test_fidelity_monotone_and_paper_rates():
    f = synth.dense(32, 32, 32, seed=12).astype(np.float64)
    errs = [float(np.abs(oracle.roundtrip64(f, r) - f).max()) for r in (8, 16, 24, 32, 40, 48, 64)]
    assert all(a >= b for a, b in zip(errs, errs[1:])), errs
    # the paper's rates: 32/64 (2:1) and 24/64 keep ~1e-9 / ~1e-7 relative accuracy here
    assert errs[3] < 1e-8 * np.abs(f).max() and errs[2] < 1e-6 * np.abs(f).max()


def test_advance64_raw_equals_plain_fp64_steps():
    u = synth.dense(12, 12, 24, seed=3).astype(np.float64)
    m = synth.layered(12, 12, 24).astype(np.float64)
    a, b = u.copy(), u.copy()
    for _ in range(5):
        a, b = oracle.step_f64(a, b, m), a
    gu, gup = oracle.advance64(u, u, m, 2, (0, 0, 0), 5)
    assert np.array_equal(gu, a) and np.array_equal(gup, b)
