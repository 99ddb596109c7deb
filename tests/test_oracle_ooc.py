"""Pins for the reduction SURVEY 8(c) c.0: the paper's out-of-core schedule
with separate compression (Fig. 4) and region sharing
(Fig. 3) equals in-core steps with a whole-field round trip
after every sweep.  The literal region emulator (oracle/ooc_emul.c) and the
reduced schedule (orc_advance) are written independently; they must agree bit
for bit, for every valid (T, P, G), and the byte counts must equal the closed
forms of region sharing.
"""
import numpy as np
import pytest

import oracle
from paper_2109_05410_b200 import synth


def _fields(nx, ny, nz, seed):
    u = synth.dense(nx, ny, nz, seed=seed)
    up = (u * np.float32(0.97)).astype(np.float32)
    return u, up, synth.layered(nx, ny, nz)


CASES = [
    # nx, ny, nz, T, P, G, nsteps
    (8, 8, 48, 1, 8, 1, 5),
    (8, 12, 96, 3, 24, 1, 7),         # T does not divide nsteps
    (12, 8, 96, 2, 16, 2, 6),
    (8, 8, 96, 2, 16, 3, 4),
    (8, 8, 64, 2, 16, 1, 0),          # step(0) == set_field round trip only
    (8, 8, 32, 4, 32, 1, 8),          # D = 1
]


@pytest.mark.parametrize("nx,ny,nz,T,P,G,n", CASES)
def test_raw_ooc_equals_in_core(nx, ny, nz, T, P, G, n):
    u, up, m = _fields(nx, ny, nz, 21)
    ru, rup = oracle.advance(u, up, m, T, (0, 0, 0), n)
    eu, eup, _ = oracle.ooc_emulate(u, up, m, T, P, G, (0, 0, 0), n)
    assert np.array_equal(eu.view(np.uint32), ru.view(np.uint32))
    assert np.array_equal(eup.view(np.uint32), rup.view(np.uint32))


@pytest.mark.parametrize("nx,ny,nz,T,P,G,n", CASES)
@pytest.mark.parametrize("rates", [(16, 16, 16), (8, 12, 24), (0, 16, 8)])
def test_compressed_ooc_equals_round_trip_schedule(nx, ny, nz, T, P, G, n, rates):
    u, up, m = _fields(nx, ny, nz, 22)
    ru, rup = oracle.run(u, up, m, T, rates, n)
    eu, eup, _ = oracle.ooc_emulate(u, up, m, T, P, G, rates, n)
    assert np.array_equal(eu.view(np.uint32), ru.view(np.uint32))
    assert np.array_equal(eup.view(np.uint32), rup.view(np.uint32))


def test_raw_ooc_matches_plain_steps():
    # raw path: no round trips at all -> plain repeated oracle steps
    u, up, m = _fields(8, 8, 48, 23)
    a, b = u.copy(), up.copy()
    for _ in range(6):
        a, b = oracle.step(a, b, m), a
    eu, eup, _ = oracle.ooc_emulate(u, up, m, 3, 24, 1, (0, 0, 0), 6)
    assert np.array_equal(eu, a) and np.array_equal(eup, b)


@pytest.mark.parametrize("rates", [(0, 0, 0), (16, 16, 16)])
def test_temporal_block_cone_nan_poison(rates):
    u, up, m = _fields(8, 8, 96, 24)
    a = oracle.ooc_emulate(u, up, m, 3, 24, 2, rates, 9, poison=False)
    b = oracle.ooc_emulate(u, up, m, 3, 24, 2, rates, 9, poison=True)
    assert np.array_equal(a[0].view(np.uint32), b[0].view(np.uint32))
    assert np.array_equal(a[1].view(np.uint32), b[1].view(np.uint32))
    assert np.isfinite(b[0]).all()


@pytest.mark.parametrize("G", [1, 2])
@pytest.mark.parametrize("rates", [(0, 0, 0), (16, 8, 24)])
def test_region_sharing_byte_accounting(G, rates):
    nx, ny, nz, T, P, n = 8, 12, 96, 2, 16, 6
    u, up, m = _fields(nx, ny, nz, 25)
    _, _, st = oracle.ooc_emulate(u, up, m, T, P, G, rates, n)
    sweeps = -(-n // T)
    stored = [oracle.zfp_bytes(nx, ny, nz, r) if r else 4 * nx * ny * nz for r in rates]
    # every region of every field is uploaded exactly once per sweep
    assert st["h2d"] == sweeps * sum(stored)
    # read-write regions downloaded once per sweep; the read-only one never
    assert st["d2h"] == sweeps * (stored[0] + stored[1])
    h = 4 * T
    per = [oracle.zfp_bytes(nx, ny, h, r) if r else 4 * nx * ny * h for r in rates]
    # per boundary: h planes of u, u- both ways every sweep; m once, both ways
    assert st["halo"] == (G - 1) * (2 * sweeps * (per[0] + per[1]) + 2 * per[2])
    # naive halo transfer would upload block +- h every time (Fig. 1b); region
    # sharing (Fig. 3) uploads every plane once: it saves 2h planes per
    # internal block boundary per field per sweep
    D = nz // G // P
    naive_planes = G * (D * P + 2 * h * (D - 1))
    assert naive_planes - nz == G * (D - 1) * 2 * h


# ----------------------------------------------------------------------------
# the paper's own precision (fp64; rates 32/64 and 24/64,
# PAPER.md:213-215): the literal emulator instantiated in fp64
# (oracle/ooc_emul64.c) pins the reduced fp64 schedule orc64_advance at
# rates > 0, which no closed form reaches.

def _fields64(nx, ny, nz, seed):
    u = synth.dense(nx, ny, nz, seed=seed).astype(np.float64)
    up = u * 0.97
    return u, up, synth.layered(nx, ny, nz).astype(np.float64)


@pytest.mark.parametrize("nx,ny,nz,T,P,G,n", CASES)
@pytest.mark.parametrize("rates", [(32, 32, 32), (0, 24, 24), (0, 32, 0), (16, 40, 8)])
def test_compressed_ooc_equals_round_trip_schedule_fp64(nx, ny, nz, T, P, G, n, rates):
    u, up, m = _fields64(nx, ny, nz, 24)
    ru, rup = oracle.run64(u, up, m, T, rates, n)
    eu, eup, st = oracle.ooc_emulate64(u, up, m, T, P, G, rates, n)
    assert np.array_equal(eu.view(np.uint64), ru.view(np.uint64))
    assert np.array_equal(eup.view(np.uint64), rup.view(np.uint64))
    if n:
        # rate r: 8r bytes per 4^3 block, raw: 8 B per value
        rb = [(nx // 4) * (ny // 4) * 8 * r if r else nx * ny * 4 * 8 for r in rates]   # per block-row
        sweeps = -(-n // T)
        assert st["h2d"] == sweeps * sum(rb[f] * nz // 4 for f in range(3))
        assert st["d2h"] == sweeps * sum(rb[f] * nz // 4 for f in range(2))


def test_fp64_emulator_poisoned_cone_and_paper_decomposition():
    # NaN outside the valid cone changes nothing; the paper's D = 8, T = 12 shape
    u, up, m = _fields64(8, 8, 8 * 96, 25)
    rates = (0, 24, 24)                                 # the paper's code 4
    ru, rup = oracle.run64(u, up, m, 12, rates, 24)
    eu, eup, _ = oracle.ooc_emulate64(u, up, m, 12, 96, 1, rates, 24, poison=True)
    assert np.array_equal(eu.view(np.uint64), ru.view(np.uint64))
    assert np.array_equal(eup.view(np.uint64), rup.view(np.uint64))


def test_fp64_raw_schedule_is_plain_fp64_steps():
    u, up, m = _fields64(8, 8, 48, 26)
    a, b = u.copy(), up.copy()
    for _ in range(5):
        nxt = np.empty_like(a)
        oracle.lib().orc_step_f64(a, b, m, nxt, 8, 8, 48, oracle.C64)
        a, b = nxt, a
    eu, eup, _ = oracle.ooc_emulate64(u, up, m, 2, 16, 1, (0, 0, 0), 5)
    assert np.array_equal(eu, a) and np.array_equal(eup, b)
