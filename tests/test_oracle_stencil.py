"""Pins for the oracle's 25-point leapfrog (oracle/stencil_ref.c).

Closed forms only: Taylor moments of the coefficients, polynomial exactness,
the bit-level impulse response implied by the prescribed fp32 order, the
discrete plane-wave dispersion relation, and the CFL bound (PAPER.md:208,
HALO = 4 at PAPER.md:188; readings R1-R5 in DESIGN.md).
"""
import math
from fractions import Fraction

import numpy as np
import pytest

import oracle
from paper_2109_05410_b200 import synth

CF = [Fraction(-205, 72), Fraction(8, 5), Fraction(-1, 5), Fraction(8, 315), Fraction(-1, 560)]


def f32_round(q: Fraction) -> np.float32:
    """Correctly rounded (RNE) fp32 of an exact rational."""
    c = np.float32(float(q))
    best = c
    for cand in (np.nextafter(c, np.float32(-np.inf)), c, np.nextafter(c, np.float32(np.inf))):
        d, db = abs(Fraction(float(cand)) - q), abs(Fraction(float(best)) - q)
        if d < db or (d == db and (int(np.float32(cand).view(np.uint32)) & 1) == 0):
            best = cand
    return np.float32(best)


def test_coefficients_taylor_moments():
    # second-derivative weights of order 8: moments sum_k c_k (k^p + (-k)^p)
    for p, want in ((0, 0), (2, 2), (4, 0), (6, 0), (8, 0)):
        s = sum(CF[k] * (k ** p + (-k) ** p) for k in range(1, 5))
        if p == 0:
            s += CF[0]
        assert s == want
    assert sum(CF[k] * 2 * k ** 10 for k in range(1, 5)) != 0     # order is exactly 8


def test_coefficients_are_fp32_of_the_rationals():
    c = oracle.default_coeffs()
    for k in range(5):
        assert c[k] == f32_round(CF[k])


def test_cfl_bound_closed_form():
    # S(theta) = c0 + 2 sum c_k cos(k theta) is most negative at theta = pi:
    # S(pi) = -2048/315; leapfrog stable for m * 3 |S| <= 4 -> m <= 105/512
    s_pi = CF[0] + 2 * sum(CF[k] * (-1) ** k for k in range(1, 5))
    assert s_pi == Fraction(-2048, 315)
    assert Fraction(4) / (3 * abs(s_pi)) == Fraction(105, 512)
    th = np.linspace(0, np.pi, 20001)
    S = float(CF[0]) + 2 * sum(float(CF[k]) * np.cos(k * th) for k in range(1, 5))
    assert np.argmin(S) == len(th) - 1


def test_zero_state_is_fixed_point():
    z = np.zeros((12, 12, 12), np.float32)
    out = oracle.step(z, z, synth.layered(12, 12, 12))
    assert not out.view(np.uint32).any()


def test_impulse_response_bit_exact():
    n = 17
    u = np.zeros((n, n, n), np.float32)
    u[8, 8, 8] = 1.0
    up = np.zeros_like(u)
    mval = np.float32(0.15)
    m = np.full_like(u, mval)
    out = oracle.step(u, up, m)
    c = oracle.default_coeffs()
    c0x3 = np.float32(3.0) * c[0]
    want = np.zeros_like(u)
    # centre: L = c0x3, u+ = fmaf(m, c0x3, 2)
    want[8, 8, 8] = f32_round(Fraction(float(mval)) * Fraction(float(c0x3)) + 2)
    for k in range(1, 5):
        arm = mval * c[k]                    # fl32(m * c_k)
        for d in ((k, 0, 0), (-k, 0, 0), (0, k, 0), (0, -k, 0), (0, 0, k), (0, 0, -k)):
            want[8 + d[0], 8 + d[1], 8 + d[2]] = arm
    assert np.array_equal(out, want)
    nz = out != 0
    assert np.array_equal(out[nz].view(np.uint32), want[nz].view(np.uint32))


def test_constant_field_laplacian_zero_away_from_boundary():
    u = np.full((20, 20, 20), np.float32(0.75))
    out = oracle.step(u, u, synth.layered(20, 20, 20))
    inner = out[4:-4, 4:-4, 4:-4]
    assert np.array_equal(inner, u[4:-4, 4:-4, 4:-4])
    assert not np.array_equal(out[0], u[0])          # Dirichlet ghost is felt


def test_quadratic_laplacian_is_six_fp64():
    n = 24
    z, y, x = np.meshgrid(*(np.arange(n, dtype=np.float64) - 11.5,) * 3, indexing="ij")
    u = x * x + y * y + z * z
    m = np.ones_like(u)
    out = oracle.step_f64(u, u, m)              # u+ - u = L(u)
    L = (out - u)[4:-4, 4:-4, 4:-4]
    assert np.abs(L - 6.0).max() < 1e-9


def test_degree8_polynomial_exact_fp64():
    n = 26
    z, y, x = np.meshgrid(*(np.arange(n, dtype=np.float64) / 8 - 1.6,) * 3, indexing="ij")
    u = x ** 8 + 3 * y ** 7 - z ** 6 + x * y * z
    lap = 56 * x ** 6 + 126 * y ** 5 - 30 * z ** 4      # exact, dx = 1/8 folded below
    out = oracle.step_f64(u, u, np.ones_like(u))
    L = (out - u) * 64.0                                   # d^2/dx^2 with dx = 1/8
    assert np.abs(L - lap)[4:-4, 4:-4, 4:-4].max() < 1e-7


def _plane_wave(n, kappa, m, steps, dtype):
    S = lambda th: float(CF[0]) + 2 * sum(float(CF[k]) * math.cos(k * th) for k in range(1, 5))
    cw = 1 + 0.5 * m * sum(S(k) for k in kappa)
    w = math.acos(cw)
    z, y, x = np.meshgrid(*(np.arange(n, dtype=np.float64),) * 3, indexing="ij")
    ph = kappa[0] * x + kappa[1] * y + kappa[2] * z
    u, up = np.cos(ph), np.cos(ph + w)
    exact = np.cos(ph - w * steps)
    return u.astype(dtype), up.astype(dtype), exact


def test_plane_wave_dispersion_fp64():
    n, steps, m = 48, 5, 0.18
    kappa = (0.3, 0.55, 0.9)
    u, up, exact = _plane_wave(n, kappa, m, steps, np.float64)
    mm = np.full_like(u, m)
    for _ in range(steps):
        u, up = oracle.step_f64(u, up, mm), u
    r = 4 * steps                                   # domain of dependence
    assert np.abs(u - exact)[r:-r, r:-r, r:-r].max() < 1e-11


def test_plane_wave_fp32_within_north_star_tolerance():
    n, steps, m = 48, 5, np.float32(0.18)
    kappa = (0.3, 0.55, 0.9)
    u, up, exact = _plane_wave(n, kappa, float(m), steps, np.float32)
    mm = np.full_like(u, m)
    for _ in range(steps):
        u, up = oracle.step(u, up, mm), u
    r = 4 * steps
    err = np.abs(u.astype(np.float64) - exact)[r:-r, r:-r, r:-r].max()
    assert err <= 1e-5 * steps                     # 1e-5 per step (north star)


def test_bounded_energy_under_cfl_and_blowup_above():
    n = 32
    u0 = synth.pulse(n, n, n, sigma=3.0)
    for m, bounded in ((0.2, True), (0.23, False)):
        u, up = u0.copy(), u0.copy()
        mm = np.full_like(u, np.float32(m))
        for _ in range(48 if bounded else 200):
            u, up = oracle.step(u, up, mm), u
        e = float(np.abs(u).max())
        assert (e < 2.0) == bounded, (m, e)


def test_step_planes_restricts_updates():
    n = 16
    u = synth.dense(n, n, n, seed=1)
    up = synth.dense(n, n, n, seed=2)
    m = synth.layered(n, n, n)
    full = oracle.step(u, up, m)
    out = np.full_like(u, np.float32(7.0))
    lib = oracle.lib()
    lib.orc_step_planes(u, up, m, out, n, n, n, oracle.default_coeffs(), 5, 11)
    assert np.array_equal(out[5:11], full[5:11])
    assert (out[:5] == 7).all() and (out[11:] == 7).all()
