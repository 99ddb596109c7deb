"""Set / read back a field by z-ranges (oocz_set_field_planes /
oocz_get_field_planes): the calls that let slabs larger than host memory be
initialised and sampled.  Setting in chunks stores exactly the
bytes a whole-field set stores, so the run equals the oracle bit for bit."""
import numpy as np
import pytest

import oracle
from paper_2109_05410_b200 import synth
from gpu_util import Z, bits

pytestmark = pytest.mark.gpu


def _fields(nx, ny, nz):
    u = synth.dense(nx, ny, nz, seed=21)
    return u, (u * np.float32(0.9)).astype(np.float32), synth.layered(nx, ny, nz)


@pytest.mark.parametrize("store,m_resident,chunk", [(0, 0, 8), (1, 0, 12), (0, 1, 20), (1, 1, 4)])
def test_chunked_set_equals_whole_set_and_oracle(store, m_resident, chunk):
    import torch
    z = Z()
    nx, ny, nz, T, P, rates = 40, 24, 96, 2, 24, (16, 12, 8)
    u, up, m = _fields(nx, ny, nz)
    cfg = z.oocz_default_config(nx, ny, nz, tb=T, block_planes=P, rate=list(rates), store=store,
                                m_resident=m_resident)
    with z.Stepper(cfg) as a:
        a.set(u, up, m)
        whole = [z.oocz_save_store(a.ctx, f) for f in range(3)]
    with z.Stepper(cfg) as b:
        # u from host chunks, u- from device chunks, m in reverse order
        for z0 in range(0, nz, chunk):
            z.oocz_set_field_planes(b.ctx, z.OOCZ_U, z0, u[z0:z0 + chunk])
            z.oocz_set_field_planes(b.ctx, z.OOCZ_UPREV, z0, torch.from_numpy(up[z0:z0 + chunk].copy()).cuda())
        for z0 in reversed(range(0, nz, chunk)):
            z.oocz_set_field_planes(b.ctx, z.OOCZ_M, z0, m[z0:z0 + chunk])
        torch.cuda.synchronize()
        for f in range(3):
            assert np.array_equal(z.oocz_save_store(b.ctx, f), whole[f])
        b.step(7)
        gu = b.get(z.OOCZ_U)
        # read back by ranges, to host and to device
        parts = [z.oocz_get_field_planes(b.ctx, z.OOCZ_U, z0, np.empty((min(chunk, nz - z0), ny, nx), np.float32))
                 for z0 in range(0, nz, chunk)]
        assert np.array_equal(bits(np.concatenate(parts)), bits(gu))
        d = torch.empty((8, ny, nx), dtype=torch.float32, device="cuda")
        z.oocz_get_field_planes(b.ctx, z.OOCZ_U, 16, d)
        assert np.array_equal(bits(d.cpu().numpy()), bits(gu[16:24]))
    ou, _ = oracle.run(u, up, m, T, rates, 7)
    assert np.array_equal(bits(gu), bits(ou))


def test_plane_range_errors_and_partial_state():
    z = Z()
    nx, ny, nz = 16, 16, 32
    u, up, m = _fields(nx, ny, nz)
    cfg = z.oocz_default_config(nx, ny, nz, tb=2, block_planes=16, rate=[16, 16, 16])
    with z.Stepper(cfg) as s:
        with pytest.raises(z.OoczError) as e:
            z.oocz_set_field_planes(s.ctx, z.OOCZ_U, 2, u[2:10])
        assert e.value.status == z.OOCZ_EALIGN
        with pytest.raises(z.OoczError) as e:
            z.oocz_set_field_planes(s.ctx, z.OOCZ_U, 28, u[:8])
        assert e.value.status == z.OOCZ_EINVAL
        z.oocz_set_field_planes(s.ctx, z.OOCZ_U, 0, u[:16])
        z.oocz_set_field(s.ctx, z.OOCZ_UPREV, up)
        z.oocz_set_field(s.ctx, z.OOCZ_M, m)
        with pytest.raises(z.OoczError) as e:            # u's rows [16, 32) never set
            z.oocz_step(s.ctx, 2)
        assert e.value.status == z.OOCZ_ESTATE
        with pytest.raises(z.OoczError) as e:
            z.oocz_get_field_planes(s.ctx, z.OOCZ_U, 0, np.empty((4, ny, nx), np.float32))
        assert e.value.status == z.OOCZ_ESTATE
        z.oocz_set_field_planes(s.ctx, z.OOCZ_U, 16, u[16:])
        before = [z.oocz_save_store(s.ctx, f) for f in range(3)]
        bad = u[16:24].copy()
        bad[3, 2, 1] = np.nan
        with pytest.raises(z.OoczError) as e:            # a rejected call changes nothing
            z.oocz_set_field_planes(s.ctx, z.OOCZ_U, 16, bad)
        assert e.value.status == z.OOCZ_ENONFINITE
        for f in range(3):
            assert np.array_equal(z.oocz_save_store(s.ctx, f), before[f])
        z.oocz_step(s.ctx, 2)                            # the old field still steps, bit for bit
        got = s.get(z.OOCZ_U)
    want, _ = oracle.run(u, up, m, 2, (16, 16, 16), 2)
    assert np.array_equal(bits(got), bits(want))


@pytest.mark.parametrize("store,m_resident", [(0, 0), (1, 1)])
def test_rejected_set_field_leaves_state_unchanged(store, m_resident):
    """SURVEY 8(b) "A failed validation leaves the state unchanged": a set_field
    rejected for NaN (u), or for m out of range (negative, above m_max, or a
    round trip RT(m) above m_max) keeps the previous field, which then steps
    bit-exactly like the oracle."""
    z = Z()
    nx, ny, nz, T, P, rates = 24, 16, 32, 2, 16, (16, 12, 2)
    u, up, m = _fields(nx, ny, nz)
    cfg = z.oocz_default_config(nx, ny, nz, tb=T, block_planes=P, rate=list(rates), store=store,
                                m_resident=m_resident)
    mmax = z.oocz_cfl_limit(z.default_coeffs())
    with z.Stepper(cfg) as s:
        s.set(u, up, m)
        before = [z.oocz_save_store(s.ctx, f) for f in range(3)]
        bad_u = u.copy()
        bad_u[5, 3, 2] = np.inf
        bad_neg = m.copy()
        bad_neg[1, 1, 1] = -1e-3
        bad_big = m.copy()
        bad_big[7, 2, 9] = np.float32(mmax * 1.01)
        # every value <= m_max, but rate 2 cannot hold the block: its round trip
        # overshoots the bound (what the stencil would read)
        edge = np.full_like(m, np.float32(mmax))
        edge[::2, ::2, ::2] = 0.0
        cases = [(z.OOCZ_U, bad_u, z.OOCZ_ENONFINITE), (z.OOCZ_M, bad_neg, z.OOCZ_ECFL),
                 (z.OOCZ_M, bad_big, z.OOCZ_ECFL)]
        if oracle.roundtrip(edge, rates[2]).max() > mmax:
            cases.append((z.OOCZ_M, edge, z.OOCZ_ECFL))
        for f, a, code in cases:
            with pytest.raises(z.OoczError) as e:
                z.oocz_set_field(s.ctx, f, a)
            assert e.value.status == code, (f, code)
            for g in range(3):
                assert np.array_equal(z.oocz_save_store(s.ctx, g), before[g])
        assert len(cases) == 4
        s.step(3)
        got = s.get(z.OOCZ_U)
    want, _ = oracle.run(u, up, m, T, rates, 3)
    assert np.array_equal(bits(got), bits(want))


def test_chunked_set_fp64():
    """The paper's precision through the plane-range calls."""
    z = Z()
    nx, ny, nz, T, P, rates = 24, 20, 48, 2, 16, (32, 24, 40)
    u, up, m = (a.astype(np.float64) for a in _fields(nx, ny, nz))
    cfg = z.oocz_default_config(nx, ny, nz, tb=T, block_planes=P, rate=list(rates), precision=64)
    with z.Stepper(cfg) as s:
        for z0 in range(0, nz, 8):
            for f, a in ((z.OOCZ_U, u), (z.OOCZ_UPREV, up), (z.OOCZ_M, m)):
                z.oocz_set_field_planes(s.ctx, f, z0, a[z0:z0 + 8])
        s.step(5)
        got = np.concatenate([z.oocz_get_field_planes(s.ctx, z.OOCZ_U, z0, np.empty((8, ny, nx), np.float64))
                              for z0 in range(0, nz, 8)])
    want, _ = oracle.run64(u, up, m, T, rates, 5)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
