"""Pins of the oracle against the fixtures in tests/golden/ (values printed in
the paper, or fixed by a textbook / the format definition, each cited in its
file).  CPU only; nothing here comes from the CUDA path."""
from fractions import Fraction

import numpy as np
import pytest

import oracle
from golden_io import keyvals, table
from paper_2109_05410_b200 import synth


# ---------------------------------------------------------------- stencil weights
def _fd8():
    rows = table("fd8_second_derivative.txt")
    assert [int(r[0]) for r in rows] == [0, 1, 2, 3, 4]
    return [Fraction(int(r[1]), int(r[2])) for r in rows]


def test_fd8_fixture_is_an_order8_second_derivative():
    # sanity of the fixture itself: exact on x^2 (gives 2), zero on x^0, x^4,
    # x^6, x^8; nonzero on x^10 (order exactly 8)
    c = _fd8()
    mom = lambda p: (c[0] if p == 0 else 0) + sum(c[k] * (k ** p + (-k) ** p) for k in range(1, 5))
    assert [mom(p) for p in (0, 2, 4, 6, 8)] == [0, 2, 0, 0, 0]
    assert mom(10) != 0


def test_oracle_coefficients_are_the_textbook_weights():
    c = _fd8()
    got32 = oracle.default_coeffs()
    for k in range(5):
        # fp32 weights are the rationals rounded once (reading R2)
        want = np.float32(float(c[k]))
        assert abs(Fraction(float(got32[k])) - c[k]) <= abs(Fraction(float(want)) - c[k])
        assert got32[k] == want
        assert oracle.C64[k] == float(c[k])


def test_stencil_has_25_points():
    # the oracle's impulse response touches exactly 1 + 3*2*HALO points
    halo = keyvals("paper_table1.txt")["halo"]
    n = 16
    z = np.zeros((n, n, n), np.float32)
    u = z.copy()
    u[8, 8, 8] = 1.0
    out = oracle.step(u, z, np.ones((n, n, n), np.float32) * np.float32(0.1))
    nz = np.argwhere(out != 0)
    assert len(nz) == 1 + 3 * 2 * halo == 25
    assert np.abs(nz - 8).max() == halo
    assert (np.count_nonzero(nz - 8, axis=1) <= 1).all()     # axis-aligned arms only


# ---------------------------------------------------------------- Table 1
def test_table1_entire_data_size():
    t = keyvals("paper_table1.txt")
    assert t["datasets"] == t["read_write"] + t["write_only"] + t["read_only"]
    side = t["interior"] + 2 * t["halo"]
    total = t["datasets"] * t["dtype_bytes"] * side ** 3
    # the printed "46 GB" is the GiB figure truncated (46.53 GiB; 49.9e9 bytes)
    assert int(total / 2 ** 30) == t["entire_size_gb"]
    assert round(total / 1e9) != t["entire_size_gb"]


def test_table1_transfer_roles_match_the_schedule():
    # two read-write fields go up and down, the read-only field only up, the
    # write-only one never moves: the oracle's region emulator
    # counts exactly these bytes, raw, per sweep
    t = keyvals("paper_table1.txt")
    nx, ny, nz, T, P, n = 8, 8, 64, 2, 16, 4
    u = synth.dense(nx, ny, nz, seed=3)
    _, _, st = oracle.ooc_emulate(u, u, synth.layered(nx, ny, nz), T, P, 1, (0, 0, 0), n)
    field = 4 * nx * ny * nz
    sweeps = n // T
    assert st["h2d"] == sweeps * (t["read_write"] + t["read_only"]) * field
    assert st["d2h"] == sweeps * t["read_write"] * field


# ---------------------------------------------------------------- Section 5 schedule
def test_sec5_step_grid_and_sampling():
    s = keyvals("paper_sec5_schedule.txt")
    grid = list(range(s["steps_first"], s["steps_last"] + 1, s["steps_increment"]))
    assert len(grid) == 9 and grid[-1] == s["steps_last"]
    # every sampled step ends a sweep of T = 12 steps
    assert all(g % s["temporal_blocking"] == 0 for g in grid)
    # 100 points on each of the 1152 interior planes
    assert s["points_per_plane"] * keyvals("paper_table1.txt")["interior"] == s["sampled_points"]
    assert s["rates"] == [32, 24] and s["rate_denominator"] == 64


def _paper_decomposition(nx=8, ny=8):
    s, t = keyvals("paper_sec5_schedule.txt"), keyvals("paper_table1.txt")
    nz, D, T = t["interior"], s["divisions"], s["temporal_blocking"]
    P = nz // D
    assert P * D == nz and P >= 2 * t["halo"] * T          # 144 planes, halo 48 each side
    return nx, ny, nz, T, P


@pytest.mark.parametrize("rates", [(0, 0, 0), (16, 0, 16), (16, 16, 16)])
def test_paper_decomposition_ooc_equals_reduced_schedule(rates):
    # the paper's own z decomposition (1152 planes, 8 blocks, T = 12) with
    # small x/y: the literal region emulator equals the reduced schedule
    nx, ny, nz, T, P = _paper_decomposition()
    u = synth.dense(nx, ny, nz, seed=31)
    up = (u * np.float32(0.97)).astype(np.float32)
    m = synth.layered(nx, ny, nz)
    n = 2 * T
    if rates == (0, 0, 0):
        ru, rup = oracle.advance(u, up, m, T, rates, n)
    else:
        ru, rup = oracle.run(u, up, m, T, rates, n)
    eu, eup, st = oracle.ooc_emulate(u, up, m, T, P, 1, rates, n)
    assert np.array_equal(eu.view(np.uint32), ru.view(np.uint32))
    assert np.array_equal(eup.view(np.uint32), rup.view(np.uint32))
    assert st["halo"] == 0


# ---------------------------------------------------------------- codec worked examples
def test_constant_block_encodings():
    for value, rate, used_want, w0 in table("zfp_constant_blocks.txt"):
        w, used = oracle.encode_block(np.full(64, float(value), np.float32), int(rate))
        assert used == int(used_want)
        assert int(w[0]) == int(w0, 16) and not w[1:].any()
        x, _ = oracle.decode_block(w, int(rate))
        assert (x == np.float32(value)).all()
