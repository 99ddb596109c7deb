"""Pins for the oracle's ZFP-style fixed-rate coder (oracle/zfp_ref.c).

Nothing here compares the oracle with itself: every expected value is a
closed form, a hand derivation from the format definition,
a mathematical identity, or an invariant the paper's fixed-rate contract
implies ("specify the number of bits to use to preserve a
value").  Bit compatibility with real zfp/cuZFP is UNPINNED (no zfp here).
"""
from fractions import Fraction

import numpy as np
import pytest

import oracle
from paper_2109_05410_b200 import synth

# ----------------------------------------------------------------------------
# size contract (fixed-size pre-allocated buffers)


@pytest.mark.parametrize("shape,rate,nbytes", [
    ((64, 64, 64), 16, 524_288),                  # C1: 4096 blocks * 8 * 16
    ((512, 512, 512), 8, 128 << 20),
    ((512, 512, 512), 16, 256 << 20),
    ((512, 512, 512), 24, 384 << 20),
    ((4, 4, 4), 1, 8),
    ((0, 4, 4), 16, 0),
])
def test_stream_size_closed_form(shape, rate, nbytes):
    nx, ny, nz = shape
    assert oracle.zfp_bytes(nx, ny, nz, rate) == nbytes


def test_encode_output_length_every_rate():
    f = synth.dense(8, 12, 16, seed=3)
    for rate in (1, 2, 7, 8, 16, 24, 33, 64):
        w = oracle.zfp_encode(f, rate)
        assert w.nbytes == (8 // 4) * (12 // 4) * (16 // 4) * 8 * rate


# ----------------------------------------------------------------------------
# hand-derived worked examples (format definition)


def test_zero_and_negative_zero_blocks():
    for v in (0.0, -0.0):
        w, used = oracle.encode_block(np.full(64, v, np.float32), 16)
        assert used == 1 and not w.any()                       # single 0 bit, padding
        x, _ = oracle.decode_block(w, 16)
        assert (x.view(np.uint32) == 0).all()                  # +0.0 exactly


def test_constant_one_hand_derived():
    # 1.0: emax = 1 (1.0 = 0.5 * 2^1), biased 128 -> 9 bits of 2*128+1 = 0x101.
    # q = 2^29 everywhere; lifting of a constant leaves only DC = 2^29.
    # negabinary(2^29) = 0x60000000 (bits 29, 30).  Bit planes:
    #   k=31: group flag 0                      (1 bit)
    #   k=30: flag 1, bit 1, flag 0 -> n = 1    (3 bits: 1,1,0)
    #   k=29: 1 verbatim bit (1), flag 0        (2 bits)
    #   k=28..0: verbatim 0, flag 0             (29 * 2 bits)
    # total 9 + 1 + 3 + 2 + 58 = 73; word0 = 0x101 | 0xC00 | 0x2000 = 0x2D01.
    w, used = oracle.encode_block(np.ones(64, np.float32), 16)
    assert used == 73
    assert int(w[0]) == 0x2D01 and not w[1:].any()


def test_constant_minus_one_hand_derived():
    # -1.0: same exponent; q = -2^29 -> negabinary 0x20000000 (bit 29 only):
    #   k=31, k=30: flag 0 each; k=29: 1,1,0; k=28..0: 0,0 each.
    # total 9 + 1 + 1 + 3 + 58 = 72; word0 = 0x101 | 0x1800 = 0x1901.
    w, used = oracle.encode_block(-np.ones(64, np.float32), 16)
    assert used == 72
    assert int(w[0]) == 0x1901 and not w[1:].any()


def test_constant_blocks_exact_at_every_rate_ge_2():
    # a constant c = f 2^emax gives q = f 2^30 (an integer), DC-only after
    # lifting, and needs at most 9 + 3 + 2*31 = 74 bits <= 128.
    rng = np.random.default_rng(5)
    vals = np.concatenate([rng.standard_normal(40) * 2.0 ** rng.integers(-149, 127, 40),
                           [1e-45, -1e-45, 3.4e38, -3.4e38, 1.17549435e-38]]).astype(np.float32)
    for v in vals:
        for rate in (2, 3, 8, 16, 32, 64):
            w, _ = oracle.encode_block(np.full(64, v, np.float32), rate)
            x, _ = oracle.decode_block(w, rate)
            assert (x.view(np.uint32) == np.float32(v).view(np.uint32)).all(), (v, rate)


def test_budget_exhaustion_deposit_hand_derived():
    # Coefficient 1 holds the top bit: plane 31 = ...010 -> code 1,0,1,0.
    u = np.zeros(64, np.uint32)
    u[1] = 1 << 31
    words, used = oracle.encode_ints(u, 4)
    assert used == 4 and int(words[0]) == 0b0101
    # budget 2: stream "1,0" -> scan stops at n=1, decoder deposits there: exact
    d, _ = oracle.decode_ints(words, 2)
    assert d[1] == 1 << 31 and d.sum() == 1 << 31
    # budget 1: stream "1" -> budget ends before the scan; zfp's decoder
    # deposits the one at n = 0 (SURVEY App. A decoder note)
    d, _ = oracle.decode_ints(words, 1)
    assert d[0] == 1 << 31 and d[1] == 0


# ----------------------------------------------------------------------------
# negabinary: base -2 expansion (closed form)


def _base_minus2_value(u: int) -> int:
    return sum(((u >> i) & 1) * (-2) ** i for i in range(32))


def test_negabinary_values():
    assert [oracle.int2uint(v) for v in (0, 1, -1, 2, -2)] == [0, 1, 3, 6, 2]


def test_negabinary_is_base_minus_two_and_bijective():
    rng = np.random.default_rng(1)
    # |x| < 2^30 keeps the 32-digit base -2 expansion free of wraparound
    for x in list(rng.integers(-(1 << 30), 1 << 30, 2000)) + [0, 1, -1, (1 << 30) - 1, -(1 << 30)]:
        u = oracle.int2uint(int(x))
        assert _base_minus2_value(u) == int(x)
        assert oracle.uint2int(u) == int(x)
    for u in list(rng.integers(0, 1 << 32, 2000, dtype=np.uint64)) + [0, 0xFFFFFFFF, 0xAAAAAAAA]:
        assert oracle.int2uint(oracle.uint2int(int(u))) == int(u)


# ----------------------------------------------------------------------------
# lifting: the non-orthogonal transform it computes exactly on divisible input

A = np.array([[4, 4, 4, 4], [5, 1, -1, -5], [-4, 4, 4, -4], [-2, 6, -6, 2]], dtype=object) / 16
B = np.array([[4, 6, -4, -1], [4, 2, 4, 5], [4, -2, 4, -5], [4, -6, -4, 1]], dtype=object) / 4


def _matvec(M, v):
    return [sum(Fraction(M[r][c]) * int(v[c]) for c in range(4)) for r in range(4)]


def test_lift_matrices_are_inverses():
    for r in range(4):
        for c in range(4):
            s = sum(Fraction(B[r][k]) * Fraction(A[k][c]) for k in range(4))
            assert s == (1 if r == c else 0)


def test_forward_lift_equals_matrix_on_divisible_input():
    rng = np.random.default_rng(2)
    for _ in range(500):
        v = rng.integers(-(1 << 15), 1 << 15, 4) * 64           # no >>1 truncation
        got = oracle.fwd_lift(v)
        assert [Fraction(int(g)) for g in got] == _matvec(A, v)


def test_inverse_lift_equals_matrix_on_divisible_input():
    rng = np.random.default_rng(3)
    for _ in range(500):
        v = rng.integers(-(1 << 15), 1 << 15, 4) * 16
        got = oracle.inv_lift(v)
        assert [Fraction(int(g)) for g in got] == _matvec(B, v)


def test_lift_constant_vector():
    for c in (0, 1, -7, 123456, -(1 << 29), (1 << 29) + 3):
        assert list(oracle.fwd_lift([c] * 4)) == [c, 0, 0, 0]
        assert list(oracle.inv_lift([c, 0, 0, 0])) == [c] * 4


def test_xform_is_separable_x_then_y_then_z():
    # on input divisible by 16^3 the 3-D transform is A applied along every axis
    rng = np.random.default_rng(4)
    Af = np.array([[float(Fraction(a)) for a in row] for row in A])
    for _ in range(50):
        q = (rng.integers(-(1 << 13), 1 << 13, 64) * 4096).astype(np.int64)
        cube = q.reshape(4, 4, 4)                                # [k][j][i]
        want = np.einsum("ai,bj,ck,kji->cba", Af, Af, Af, cube.astype(np.float64))
        got = oracle.fwd_xform(q).reshape(4, 4, 4)
        assert np.array_equal(got.astype(np.float64), want)


def test_xform_delta_is_outer_product_of_first_column():
    q = np.zeros(64, np.int64)
    q[0] = 1 << 29
    got = oracle.fwd_xform(q).reshape(4, 4, 4).astype(np.float64)
    col = np.array([4, 5, -4, -2], np.float64) / 16
    want = (1 << 29) * np.einsum("k,j,i->kji", col, col, col)
    assert np.array_equal(got, want)


def test_forward_lift_worked_example_with_truncation():
    # (3, 1, 4, 1) by hand through the lifting steps of SURVEY App. A:
    #   x += w -> 4; x >>= 1 -> 2; w -= x -> -1
    #   z += y -> 5; z >>= 1 -> 2; y -= z -> -1
    #   x += z -> 4; x >>= 1 -> 2; z -= x -> 0
    #   w += y -> -2; w >>= 1 -> -1; y -= w -> 0
    #   w += y >> 1 -> -1; y -= w >> 1 -> 0 - (-1) = 1
    # (the exact A v = (2.25, 0.4375, 0.25, -1.375): the >>1 truncations matter)
    assert list(oracle.fwd_lift([3, 1, 4, 1])) == [2, 1, 0, -1]
    # e0 impulses: (2,0,0,0) -> (0,2,0,-1), (3,0,0,0) -> (0,2,0,-1),
    # (1,0,0,0) -> 0, (-1,0,0,0) -> (-1,0,1,0)   (same steps by hand)
    assert list(oracle.fwd_lift([2, 0, 0, 0])) == [0, 2, 0, -1]
    assert list(oracle.fwd_lift([3, 0, 0, 0])) == [0, 2, 0, -1]
    assert list(oracle.fwd_lift([1, 0, 0, 0])) == [0, 0, 0, 0]
    assert list(oracle.fwd_lift([-1, 0, 0, 0])) == [-1, 0, 1, 0]


def test_inverse_lift_worked_example_with_truncation():
    # inv of (0, v, 0, 0) by hand: y += w>>1 -> v; w -= y>>1 -> -(v>>1);
    # y += w -> v - (v>>1); w <<= 1; w -= y -> -(v>>1) - v; z += x -> 0 ...
    # = (v + (v>>1), v - (v>>1), -(v - (v>>1)), -(v + (v>>1)))
    for v, want in ((3, [4, 2, -2, -4]), (4, [6, 2, -2, -6]), (2, [3, 1, -1, -3]), (-2, [-3, -1, 1, 3]),
                    (-4, [-6, -2, 2, 6]), (1, [1, 1, -1, -1]), (-1, [-2, 0, 0, 2])):
        assert list(oracle.inv_lift([0, v, 0, 0])) == want, v


def test_forward_xform_axis_order_x_then_y_then_z():
    # A lone value 3 at l = 0 through the 3-D forward transform, by hand, with
    # the 1-D results pinned above (l = i + 4j + 16k):
    #   x (j=k=0):   (3,0,0,0) -> (0,2,0,-1)          at i = 0..3
    #   y (i=1):     (2,0,0,0) -> (0,2,0,-1)          -> l = 5: 2, l = 13: -1
    #     (i=3):     (-1,0,0,0) -> (-1,0,1,0)         -> l = 3: -1, l = 11: 1
    #   z (l=5):     (2,0,0,0) -> (0,2,0,-1)          -> l = 21: 2, l = 53: -1
    #     (l=13):    (-1,0,0,0) -> (-1,0,1,0)         -> l = 13: -1, l = 45: 1
    #     (l=3):     (-1,0,0,0) -> (-1,0,1,0)         -> l = 3: -1, l = 35: 1
    #     (l=11):    (1,0,0,0) -> 0
    q = np.zeros(64, np.int64)
    q[0] = 3
    want = np.zeros(64, np.int64)
    want[[3, 13, 21, 35, 45, 53]] = [-1, -1, 2, 1, 1, -1]
    got = oracle.fwd_xform(q).astype(np.int64)
    assert np.array_equal(got, want)
    # the other order (z, y, x) gives the i <-> k transpose, which differs
    zyx = want.reshape(4, 4, 4).transpose(2, 1, 0).reshape(64)
    assert not np.array_equal(zyx, want)


def test_inverse_xform_axis_order_z_then_y_then_x():
    # A lone coefficient 3 at (i, j, k) = (1, 0, 1), l = 17, through the inverse:
    #   z (i=1, j=0): (0,3,0,0) -> b = (4,2,-2,-4) along k
    #   y (i=1, each k): (b_k,0,0,0) -> constant b_k along j
    #   x (each j, k):  (0,b_k,0,0) -> row_k = inv(0,b_k,0,0) along i:
    #     k=0: (6,2,-2,-6)  k=1: (3,1,-1,-3)  k=2: (-3,-1,1,3)  k=3: (-6,-2,2,6)
    q = np.zeros(64, np.int64)
    q[17] = 3
    rows = np.array([[6, 2, -2, -6], [3, 1, -1, -3], [-3, -1, 1, 3], [-6, -2, 2, 6]], np.int64)
    want = np.repeat(rows[:, None, :], 4, axis=1)          # [k][j][i]
    got = oracle.inv_xform(q).astype(np.int64).reshape(4, 4, 4)
    assert np.array_equal(got, want)
    assert not np.array_equal(want.transpose(2, 1, 0), want)   # x-first would differ


def test_xform_axis_order_fp64_twin():
    # the fp64 codec's int64 lifting runs the same steps in the same axis order
    q = np.zeros(64, np.int64)
    q[0] = 3
    want = np.zeros(64, np.int64)
    want[[3, 13, 21, 35, 45, 53]] = [-1, -1, 2, 1, 1, -1]
    a = q.copy()
    oracle.lib().orc64_fwd_xform(a)
    assert np.array_equal(a, want)
    b = np.zeros(64, np.int64)
    b[17] = 3
    oracle.lib().orc64_inv_xform(b)
    rows = np.array([[6, 2, -2, -6], [3, 1, -1, -3], [-3, -1, 1, 3], [-6, -2, 2, 6]], np.int64)
    assert np.array_equal(b.reshape(4, 4, 4), np.repeat(rows[:, None, :], 4, axis=1))


def test_forward_coefficients_fit_guard_bits():
    # |q| < 2^30 on input, so the transform never wraps (max |coeff| < 2^31)
    rng = np.random.default_rng(6)
    for _ in range(2000):
        q = rng.integers(-(1 << 30) + 1, 1 << 30, 64)
        assert np.abs(oracle.fwd_xform(q).astype(np.int64)).max() < (1 << 31)


# ----------------------------------------------------------------------------
# coefficient order


def test_perm_is_a_sequency_order():
    p = oracle.perm3()
    assert sorted(p.tolist()) == list(range(64))
    i, j, k = p % 4, (p // 4) % 4, p // 16
    s1 = i + j + k
    s2 = i * i + j * j + k * k
    key = list(zip(s1, s2))
    assert key == sorted(key)            # by i+j+k, then by i^2+j^2+k^2


# ----------------------------------------------------------------------------
# embedded group-tested bit-plane coder


def _closed_form_bits(u: np.ndarray) -> int:
    """Unbounded code length from per-plane popcounts and top bits:
    plane k costs n verbatim bits, then 1 bit if nothing new is significant,
    else popcount + (top-n+1) scan bits + a final 0 flag (the scan never
    spends a bit on position 63, and there is no flag once n = 64)."""
    n, total = 0, 0
    for k in range(31, -1, -1):
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


def test_code_length_matches_closed_form():
    rng = np.random.default_rng(7)
    cases = [rng.integers(0, 1 << 32, 64, dtype=np.uint64).astype(np.uint32) for _ in range(30)]
    for b in synth.random_blocks(64, seed=8):
        if oracle.exponent_max(b) == -127:
            continue
        q = oracle.fwd_xform(oracle.fwd_cast(b, oracle.exponent_max(b)))
        cases.append(np.array([oracle.int2uint(int(q[p])) for p in oracle.perm3()], np.uint32))
    z = np.zeros(64, np.uint32); z[63] = 0xFFFFFFFF
    cases += [np.zeros(64, np.uint32), np.full(64, 0xFFFFFFFF, np.uint32), z]
    for u in cases:
        _, used = oracle.encode_ints(u, 64 * 64)
        assert used == _closed_form_bits(u)


def test_integer_stage_lossless_at_rate_34():
    # worst case 31*64 + 64 + 64 + ... <= 2144 < 64*34 - 9 = 2167 bits
    rng = np.random.default_rng(9)
    cases = [rng.integers(0, 1 << 32, 64, dtype=np.uint64).astype(np.uint32) for _ in range(200)]
    cases += [np.full(64, 0xFFFFFFFF, np.uint32), np.full(64, 0xAAAAAAAA, np.uint32),
              np.full(64, 0x55555555, np.uint32)]
    for u in cases:
        words, used = oracle.encode_ints(u, 64 * 34 - 9)
        assert used <= 64 * 34 - 9
        d, used2 = oracle.decode_ints(words, 64 * 34 - 9)
        assert np.array_equal(d, u) and used2 == used


def test_embedded_prefix_property():
    blocks = synth.random_blocks(120, seed=10)
    for b in blocks:
        streams = {r: oracle.encode_block(b, r)[0] for r in (1, 2, 5, 8, 16, 24, 40, 64)}
        rates = sorted(streams)
        for lo, hi in zip(rates, rates[1:]):
            bl = np.unpackbits(streams[lo].view(np.uint8), bitorder="little")
            bh = np.unpackbits(streams[hi].view(np.uint8), bitorder="little")[: 64 * lo]
            assert np.array_equal(bl, bh), (lo, hi)


def test_high_rate_error_bound_and_transform_identity():
    # r >= 34: bit-plane stage lossless, so the result is the transform-only
    # round trip, whose error is a few units of 2^(emax-30) (lifting is not
    # exactly invertible: its >>1 steps drop bits).
    blocks = synth.random_blocks(400, seed=11)
    for b in blocks:
        emax = oracle.exponent_max(b)
        w, _ = oracle.encode_block(b, 34)
        x, _ = oracle.decode_block(w, 34)
        if emax == -127:
            assert not x.view(np.uint32).any()
            continue
        ref = oracle.inv_cast(oracle.inv_xform(oracle.fwd_xform(oracle.fwd_cast(b, emax))), emax)
        assert np.array_equal(x.view(np.uint32), ref.view(np.uint32))
        err = np.abs(x.astype(np.float64) - b.astype(np.float64)).max()
        assert err <= 64 * 2.0 ** (emax - 30) + 2.0 ** (emax - 23)


def test_fidelity_monotone_in_rate_on_smooth_field():
    f = synth.dense(32, 32, 32, seed=12)
    errs = []
    for r in (2, 4, 8, 12, 16, 20, 24, 28, 32):
        g = oracle.roundtrip(f, r)
        errs.append(float(np.abs(g.astype(np.float64) - f).max()))
    assert all(a >= b for a, b in zip(errs, errs[1:])), errs
    assert errs[-1] < 1e-6 * np.abs(f).max()


def test_locality_and_determinism():
    f = synth.dense(16, 16, 16, seed=13)
    w1 = oracle.zfp_encode(f, 12)
    assert np.array_equal(w1, oracle.zfp_encode(f, 12))
    g = f.copy()
    g[5, 9, 2] += 1.0            # block (bx=0, by=2, bz=1)
    w2 = oracle.zfp_encode(g, 12)
    b = 0 + 4 * (2 + 4 * 1)
    diff = np.nonzero((w1 != w2).reshape(-1, 12).any(axis=1))[0]
    assert diff.tolist() == [b]


def test_block_order_and_placement():
    # block b = bx + nbx*(by + nby*bz) occupies words [r*b, r*b + r)
    blocks = synth.random_blocks(2 * 3 * 2, seed=14)
    f = synth.blocks_to_field(blocks, 2, 3, 2)
    w = oracle.zfp_encode(f, 7).reshape(-1, 7)
    for b in range(12):
        assert np.array_equal(w[b], oracle.encode_block(blocks[b], 7)[0])
