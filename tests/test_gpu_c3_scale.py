"""Parity at the scale the metric is quoted on (4096-wide
planes streamed out of core), which the small grids of the other tests never
reach: 4096 x 4096 x 256 with P = 128, T = 4, so every device slab holds
4096^2 x (P + 8T) = 2.68e9 > 2^31 values per field (64-bit indexing), the
stencil runs 4096-wide rows with a ragged last tile (4096 = 273 x 15 + 1 rows),
the codec 1M ZFP blocks per block-row, and the host store is 25.8 GB of pinned
memory shared by all runs (oocz_create_ex).

The oracle cannot step the whole grid, so it runs on a sub-box around each
sampled point: the reduced schedule is local -- a value
depends only on inputs within 4 cells per step plus one ZFP block (4 cells) per
round trip -- so on a box whose cut faces lie farther than that from the point
(and whose z / x / y origin is 4-aligned, so its ZFP blocks are the grid's),
the oracle gives the whole-grid value.  Points cover block boundaries (z = P
+- 1), the z ends of the domain, the x / y Dirichlet ghosts, the last (ragged)
stencil tile row, and seeded random positions.  The inputs are generated on
the GPU (synth.dense_torch / layered_torch) and checked against synth here."""
import numpy as np
import pytest

import oracle
from paper_2109_05410_b200 import synth
from gpu_util import Z

pytestmark = pytest.mark.gpu

N, NZ, T, RATE, SEED = 4096, 256, 4, 16, 2
SWEEPS = 2
NSTEPS = SWEEPS * T
R = 4 * NSTEPS + 4 * (SWEEPS + 1) + 8       # dependence radius (steps + round trips) + margin


def _points():
    rng = np.random.default_rng(20261017)
    pts = [(int(rng.integers(0, N)), int(rng.integers(0, N)), int(rng.integers(0, NZ))) for _ in range(16)]
    pts += [(1000, 2000, 127), (1000, 2000, 128), (7, 4090, 129), (4095, 3, 0), (0, 0, NZ - 1),
            (2048, 4095, 64), (2048, 4094, 200), (4095, 4095, 255), (3, 1111, 255), (2222, 0, 128),
            (17, 4095, 131), (4094, 2047, 1), (1234, 4089, 96), (3333, 15, 160), (5, 5, 124), (4090, 4090, 132)]
    return pts


def _set_fields(z, ctx):
    import torch
    for z0 in range(0, NZ, 16):
        d = synth.dense_torch(N, N, NZ, SEED, z0, z0 + 16)
        z.oocz_set_field_planes(ctx, z.OOCZ_U, z0, d)
        z.oocz_set_field_planes(ctx, z.OOCZ_UPREV, z0, d)
        z.oocz_set_field_planes(ctx, z.OOCZ_M, z0, synth.layered_torch(N, N, NZ, z0, z0 + 16))
        del d
    torch.cuda.synchronize()


def _oracle_at(x, y, zz):
    lo = [max(0, (c - R) // 4 * 4) for c in (x, y, zz)]
    hi = [min(n, ((c + R) // 4 + 1) * 4) for c, n in zip((x, y, zz), (N, N, NZ))]
    u = synth.dense(N, N, NZ, SEED, lo[2], hi[2], lo[1], hi[1], lo[0], hi[0])
    m = synth.layered(N, N, NZ, lo[2], hi[2], lo[1], hi[1], lo[0], hi[0])
    ou, oup = oracle.run(u, u, m, T, (RATE,) * 3, NSTEPS)
    i = (zz - lo[2], y - lo[1], x - lo[0])
    return ou[i], oup[i]


@pytest.fixture(scope="module")
def expected():
    return {p: _oracle_at(*p) for p in _points()}


@pytest.fixture(scope="module")
def arena():
    z = Z()
    cfg = z.oocz_default_config(N, N, NZ, tb=T, block_planes=128, rate=[RATE] * 3)
    need = z.oocz_host_store_bytes(cfg, 1)
    p = z.oocz_host_alloc(need)
    yield p, need
    z.oocz_host_free(p)


def test_gpu_generators_match_synth_at_4096():
    import torch
    for z0 in (0, 124, NZ - 4):
        d = synth.dense_torch(N, N, NZ, SEED, z0, z0 + 4).cpu().numpy()
        m = synth.layered_torch(N, N, NZ, z0, z0 + 4).cpu().numpy()
        assert np.array_equal(d.view(np.uint32), synth.dense(N, N, NZ, seed=SEED, z0=z0, z1=z0 + 4).view(np.uint32))
        assert np.array_equal(m.view(np.uint32), synth.layered(N, N, NZ, z0=z0, z1=z0 + 4).view(np.uint32))
    torch.cuda.empty_cache()


@pytest.mark.parametrize("name,opts", [
    ("paper_faithful", dict(block_planes=128)),                                   # D = 2, slab 2.68e9 values
    ("serpentine_m_resident", dict(block_planes=64, serpentine=1, m_resident=1, slots=7)),   # m_full 4.8e9 values
    ("serpentine_m_hbm", dict(block_planes=64, serpentine=1, m_hbm=1, slots=20, slab_sets=1)),  # the headline schedule
    ("hbm_store_one_set", dict(block_planes=128, store=1, slab_sets=1)),
])
def test_c3_scale_sampled_parity(name, opts, expected, arena):
    import torch
    z = Z()
    cfg = z.oocz_default_config(N, N, NZ, tb=T, rate=[RATE] * 3, **opts)
    torch.cuda.empty_cache()
    if opts.get("store", 0) == 0:
        ctx = z.oocz_create_ex(cfg, 0, 1, None, 0, arena[0], arena[1])
    else:
        ctx = z.oocz_create(cfg, 0, 1, None, 0)
    try:
        _set_fields(z, ctx)
        z.oocz_step(ctx, NSTEPS)                 # one call: the oracle's schedule
        st = z.oocz_get_stats(ctx)
        assert st["sweeps"] == SWEEPS
        rows = {}
        bad = []
        for (x, y, zz), (wu, wup) in expected.items():
            zb = zz // 4 * 4
            if zb not in rows:
                rows[zb] = (z.oocz_get_field_planes(ctx, z.OOCZ_U, zb, np.empty((4, N, N), np.float32)),
                            z.oocz_get_field_planes(ctx, z.OOCZ_UPREV, zb, np.empty((4, N, N), np.float32)))
            gu, gup = rows[zb][0][zz - zb, y, x], rows[zb][1][zz - zb, y, x]
            if not (np.float32(gu).view(np.uint32) == np.float32(wu).view(np.uint32) and
                    np.float32(gup).view(np.uint32) == np.float32(wup).view(np.uint32)):
                bad.append(((x, y, zz), float(gu), float(wu), float(gup), float(wup)))
        assert not bad, (name, bad[:5])
        assert len(expected) >= 32
    finally:
        z.oocz_destroy(ctx)
