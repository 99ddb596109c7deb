"""Resident blocks (cfg.resident_blocks = K): a host-store context keeps the
compressed rows of z-blocks 0 .. K-1 in HBM and streams the rest.  The
placement changes where bytes live, never what is computed, so every case is
bit-exact against the oracle's reduced schedule; the host link carries only the
streamed blocks' rows."""
import numpy as np
import pytest

from gpu_util import Z, bits
from test_gpu_engine import CASES, _fields, _run_oracle

pytestmark = pytest.mark.gpu


def _cfg(z, nx, ny, nz, T, P, rates, K, **kw):
    return z.oocz_default_config(nx, ny, nz, tb=T, block_planes=P, rate=list(rates), store=z.OOCZ_STORE_HOST,
                                 resident_blocks=K, **kw)


def _ks(D):
    return sorted({1, max(D - 1, 1), D})


@pytest.mark.parametrize("serpentine,m_resident,slots", [(0, 0, 2), (1, 1, 3), (1, 0, 2), (0, 1, 3)])
@pytest.mark.parametrize("nx,ny,nz,T,P,rates,calls", CASES)
def test_resident_blocks_match_oracle(nx, ny, nz, T, P, rates, calls, serpentine, m_resident, slots):
    z = Z()
    u, up, m = _fields(nx, ny, nz, 5)
    wa, wb = _run_oracle(u, up, m, T, rates, calls)
    for K in _ks(nz // P):
        cfg = _cfg(z, nx, ny, nz, T, P, rates, K, serpentine=serpentine, m_resident=m_resident, slots=slots)
        with z.Stepper(cfg) as s:
            s.set(u, up, m)
            for n in calls:
                s.step(n)
            assert np.array_equal(bits(s.get(z.OOCZ_U)), bits(wa)), K
            assert np.array_equal(bits(s.get(z.OOCZ_UPREV)), bits(wb)), K


@pytest.mark.parametrize("K", [0, 1, 2, 3, 4])
def test_resident_blocks_host_bytes(K):
    """Ascending sweeps: per sweep the H2D bytes are the streamed fields' rows of
    planes [K P, S) and the D2H bytes u's and u-'s rows of the same planes; the
    pinned host store holds just those rows."""
    z = Z()
    nx, ny, nz, T, P, rates = 32, 32, 128, 2, 32, (16, 12, 8)
    u, up, m = _fields(nx, ny, nz, 9)
    cfg = _cfg(z, nx, ny, nz, T, P, rates, K)
    row = [nx // 4 * ny // 4 * 8 * r for r in rates]          # bytes of one 4-plane row per field
    streamed = (nz - K * P) // 4
    with z.Stepper(cfg) as s:
        s.set(u, up, m)
        st0 = s.stats()
        s.step(3 * T)
        st = s.stats()
        assert st["sweeps"] - st0["sweeps"] == 3
        assert st["h2d_bytes"] - st0["h2d_bytes"] == 3 * streamed * sum(row)
        assert st["d2h_bytes"] - st0["d2h_bytes"] == 3 * streamed * (row[0] + row[1])
        assert st["host_bytes_pinned"] == streamed * sum(row)
        wa, wb = _run_oracle(u, up, m, T, rates, [3 * T])
        assert np.array_equal(bits(s.get(z.OOCZ_U)), bits(wa))
        assert np.array_equal(bits(s.get(z.OOCZ_UPREV)), bits(wb))


def test_resident_blocks_planes_and_checkpoint_across_the_boundary():
    """z-range set / get that straddle the resident / streamed boundary, and a
    checkpoint (save_store / load_store) of a hybrid store restored into a
    host-only context: the same stream bytes, the same steps."""
    z = Z()
    nx, ny, nz, T, P, rates = 24, 20, 96, 2, 24, (16, 16, 16)
    u, up, m = _fields(nx, ny, nz, 13)
    cfg = _cfg(z, nx, ny, nz, T, P, rates, 2)                # rows of planes [0, 48) in HBM
    ref = _cfg(z, nx, ny, nz, T, P, rates, 0)
    with z.Stepper(cfg) as s, z.Stepper(ref) as r:
        for f, a in ((z.OOCZ_U, u), (z.OOCZ_UPREV, up), (z.OOCZ_M, m)):
            for z0, n in ((0, 40), (40, 16), (56, 40)):          # [40, 56) straddles plane 48
                z.oocz_set_field_planes(s.ctx, f, z0, a[z0:z0 + n])
            z.oocz_set_field(r.ctx, f, a)
        for f in (z.OOCZ_U, z.OOCZ_UPREV, z.OOCZ_M):
            assert np.array_equal(z.oocz_save_store(s.ctx, f), z.oocz_save_store(r.ctx, f))
        s.step(5)
        r.step(5)
        got = np.empty((32, ny, nx), np.float32)
        z.oocz_get_field_planes(s.ctx, z.OOCZ_U, 32, got)      # [32, 64) straddles plane 48
        assert np.array_equal(bits(got), bits(r.get(z.OOCZ_U)[32:64]))
        saved = [z.oocz_save_store(s.ctx, f) for f in (z.OOCZ_U, z.OOCZ_UPREV, z.OOCZ_M)]
        for f, b in zip((z.OOCZ_U, z.OOCZ_UPREV, z.OOCZ_M), saved):
            assert np.array_equal(b, z.oocz_save_store(r.ctx, f))
    with z.Stepper(ref) as t, z.Stepper(_cfg(z, nx, ny, nz, T, P, rates, 3, m_resident=1)) as h:
        for ctx in (t.ctx, h.ctx):
            for f, b in zip((z.OOCZ_U, z.OOCZ_UPREV, z.OOCZ_M), saved):
                z.oocz_load_store(ctx, f, b)
        t.step(4)
        h.step(4)
        assert np.array_equal(bits(h.get(z.OOCZ_U)), bits(t.get(z.OOCZ_U)))
        assert np.array_equal(bits(h.get(z.OOCZ_UPREV)), bits(t.get(z.OOCZ_UPREV)))


@pytest.mark.parametrize("precision,cone", [(32, 1), (64, 0), (64, 1)])
def test_resident_blocks_fp64_and_trapezoid_cone(precision, cone):
    """The paper's own schedule (trapezoid cone, ascending, m streamed) and the fp64
    path with resident blocks: bit-exact against the matching oracle."""
    import oracle
    z = Z()
    nx, ny, nz, T, P = 24, 20, 96, 2, 24
    rates = (32, 24, 24) if precision == 64 else (16, 12, 16)
    u, up, m = _fields(nx, ny, nz, 17)
    calls = [5, 4]
    if precision == 64:
        u, up, m = (a.astype(np.float64) for a in (u, up, m))
        a, b, mm = oracle.roundtrip64(u, rates[0]), oracle.roundtrip64(up, rates[1]), oracle.roundtrip64(m, rates[2])
        for n in calls:
            a, b = oracle.advance64(a, b, mm, T, rates, n)
        view = np.uint64
    else:
        a, b = _run_oracle(u, up, m, T, rates, calls)
        view = np.uint32
    for K in (1, 3):
        cfg = _cfg(z, nx, ny, nz, T, P, rates, K, precision=precision, cone=cone)
        with z.Stepper(cfg) as s:
            s.set(u, up, m)
            for n in calls:
                s.step(n)
            assert np.array_equal(s.get(z.OOCZ_U).view(view), a.view(view)), K
            assert np.array_equal(s.get(z.OOCZ_UPREV).view(view), b.view(view)), K


@pytest.mark.parametrize("world,K", [(2, 1), (2, 4), (4, 1), (4, 2)])
def test_resident_blocks_partitioned_group(world, K):
    """z-partitioned (in-process local group, compressed halos) with the first K
    blocks of every rank resident: each rank's halo rows come from HBM (top) and
    the host (bottom) as placed; bit-identical to the oracle."""
    z = Z()
    nx, ny, nz, T, P, rates = 32, 24, 128, 2, 16, (16, 12, 16)
    u, up, m = _fields(nx, ny, nz, 23)
    cfg = _cfg(z, nx, ny, nz, T, P, rates, K, serpentine=int(world == 2), m_resident=int(K == 1))
    ctxs = z.oocz_create_local_group(cfg, world)
    S = nz // world
    try:
        for r, c in enumerate(ctxs):
            for f, a in ((z.OOCZ_U, u), (z.OOCZ_UPREV, up), (z.OOCZ_M, m)):
                z.oocz_set_field(c, f, a[r * S:(r + 1) * S])
        z.oocz_step_local_group(ctxs, 7)
        gu = np.concatenate([z.oocz_get_field(c, z.OOCZ_U, np.empty((S, ny, nx), np.float32)) for c in ctxs])
        gup = np.concatenate([z.oocz_get_field(c, z.OOCZ_UPREV, np.empty((S, ny, nx), np.float32)) for c in ctxs])
    finally:
        for c in ctxs:
            z.oocz_destroy(c)
    ou, oup = _run_oracle(u, up, m, T, rates, [7])
    assert np.array_equal(bits(gu), bits(ou))
    assert np.array_equal(bits(gup), bits(oup))


def test_resident_blocks_auto_takes_what_the_budget_leaves():
    """resident_blocks = -1: the largest K whose rows fit the device budget beside
    everything else (here a budget of the K = 0 need plus 2.5 blocks of rows:
    K = 2), reported by oocz_get_config; results unchanged."""
    z = Z()
    nx, ny, nz, T, P, rates = 32, 32, 128, 2, 32, (16, 12, 8)
    u, up, m = _fields(nx, ny, nz, 29)
    per_block = sum(nx // 4 * ny // 4 * 8 * r for r in rates) * (P // 4)
    with z.Stepper(_cfg(z, nx, ny, nz, T, P, rates, 0)) as s0:
        need0 = s0.stats()["device_bytes_used"]
    cfg = _cfg(z, nx, ny, nz, T, P, rates, -1, device_bytes=need0 + per_block * 5 // 2)
    with z.Stepper(cfg) as s:
        assert z.oocz_get_config(s.ctx).resident_blocks == 2
        assert s.stats()["device_bytes_used"] == need0 + 2 * per_block
        s.set(u, up, m)
        s.step(5)
        wa, wb = _run_oracle(u, up, m, T, rates, [5])
        assert np.array_equal(bits(s.get(z.OOCZ_U)), bits(wa))
        assert np.array_equal(bits(s.get(z.OOCZ_UPREV)), bits(wb))
    with z.Stepper(_cfg(z, nx, ny, nz, T, P, rates, -1)) as s:     # the whole free HBM: every block
        assert z.oocz_get_config(s.ctx).resident_blocks == nz // P


def test_resident_blocks_with_a_caller_arena():
    """oocz_create_ex with resident blocks: the arena must hold only the streamed
    rows (oocz_host_store_bytes of the config); one byte less is OOCZ_ECAPACITY and
    leaves nothing behind; the exact size steps bit-exactly."""
    z = Z()
    nx, ny, nz, T, P, rates = 32, 24, 96, 2, 24, (16, 12, 16)
    u, up, m = _fields(nx, ny, nz, 31)
    cfg = _cfg(z, nx, ny, nz, T, P, rates, 2)
    need = z.oocz_host_store_bytes(cfg, 1)
    assert need < z.oocz_host_store_bytes(_cfg(z, nx, ny, nz, T, P, rates, 0), 1)
    arena = z.oocz_host_alloc(need)
    try:
        with pytest.raises(z.OoczError) as e:
            z.oocz_create_ex(cfg, 0, 1, None, 0, arena, need - 1)
        assert e.value.status == z.OOCZ_ECAPACITY
        ctx = z.oocz_create_ex(cfg, 0, 1, None, 0, arena, need)
        try:
            for f, a in ((z.OOCZ_U, u), (z.OOCZ_UPREV, up), (z.OOCZ_M, m)):
                z.oocz_set_field(ctx, f, a)
            z.oocz_step(ctx, 6)
            wa, wb = _run_oracle(u, up, m, T, rates, [6])
            assert np.array_equal(bits(z.oocz_get_field(ctx, z.OOCZ_U, np.empty_like(u))), bits(wa))
            assert np.array_equal(bits(z.oocz_get_field(ctx, z.OOCZ_UPREV, np.empty_like(u))), bits(wb))
        finally:
            z.oocz_destroy(ctx)
    finally:
        z.oocz_host_free(arena)


@pytest.mark.parametrize("K,serpentine,slots", [(0, 1, 5), (1, 1, 3), (0, 0, 2), (2, 1, 7)])
def test_m_hbm_matches_oracle_and_moves_no_m_bytes(K, serpentine, slots):
    """m_hbm = 1: m's compressed stream lives in HBM whole and is decoded per block
    (never crossing the host link), u and u- placed as resident_blocks says:
    bit-exact, and the H2D bytes carry no m rows."""
    z = Z()
    nx, ny, nz, T, P, rates = 32, 24, 96, 2, 16, (16, 12, 8)
    u, up, m = _fields(nx, ny, nz, 37)
    calls = [7, 4]
    cfg = _cfg(z, nx, ny, nz, T, P, rates, K, serpentine=serpentine, slots=slots, m_hbm=1)
    ref = _cfg(z, nx, ny, nz, T, P, rates, K, serpentine=serpentine, slots=slots, m_resident=1)
    with z.Stepper(cfg) as s, z.Stepper(ref) as r:
        for st in (s, r):
            st.set(u, up, m)
            for n in calls:
                st.step(n)
        wa, wb = _run_oracle(u, up, m, T, rates, calls)
        assert np.array_equal(bits(s.get(z.OOCZ_U)), bits(wa))
        assert np.array_equal(bits(s.get(z.OOCZ_UPREV)), bits(wb))
        # m decoded once (m_resident) or read in HBM (m_hbm): the same host traffic
        assert s.stats()["h2d_bytes"] == r.stats()["h2d_bytes"]
        assert s.stats()["d2h_bytes"] == r.stats()["d2h_bytes"]
        assert np.array_equal(bits(s.get(z.OOCZ_M)), bits(r.get(z.OOCZ_M)))
