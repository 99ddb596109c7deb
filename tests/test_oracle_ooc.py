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
