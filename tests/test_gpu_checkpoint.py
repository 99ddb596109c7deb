"""Checkpoint / restore of the compressed store: a run
interrupted at a sweep boundary, saved, loaded into a fresh context and
continued is bit-identical to the uninterrupted run; a decode->re-encode
"checkpoint" of the fields is not (ZFP round trips are not idempotent)."""
import numpy as np
import pytest

import oracle
from paper_2109_05410_b200 import synth
from gpu_util import Z, bits

pytestmark = pytest.mark.gpu


def _fields(nx, ny, nz):
    u = synth.dense(nx, ny, nz, seed=11)
    return u, (u * np.float32(0.95)).astype(np.float32), synth.layered(nx, ny, nz)


@pytest.mark.parametrize("store,m_resident,rates", [(0, 0, (8, 8, 8)), (1, 0, (12, 16, 8)), (0, 1, (8, 0, 12))])
def test_checkpoint_continues_bit_for_bit(store, m_resident, rates):
    z = Z()
    nx, ny, nz, T, P = 32, 24, 64, 2, 16
    u, up, m = _fields(nx, ny, nz)
    cfg = z.oocz_default_config(nx, ny, nz, tb=T, block_planes=P, rate=list(rates), store=store,
                                m_resident=m_resident)
    with z.Stepper(cfg) as a:
        a.set(u, up, m)
        a.step(10)
        want_u, want_up = a.get(z.OOCZ_U), a.get(z.OOCZ_UPREV)
    with z.Stepper(cfg) as b:
        b.set(u, up, m)
        b.step(4)
        saved = [z.oocz_save_store(b.ctx, f) for f in (z.OOCZ_U, z.OOCZ_UPREV, z.OOCZ_M)]
    assert [s.nbytes for s in saved] == [oracle.zfp_bytes(nx, ny, nz, r) if r else 4 * nx * ny * nz
                                         for r in rates]
    with z.Stepper(cfg) as c:
        for f, s in zip((z.OOCZ_U, z.OOCZ_UPREV, z.OOCZ_M), saved):
            z.oocz_load_store(c.ctx, f, s)
        c.step(6)
        got_u, got_up = c.get(z.OOCZ_U), c.get(z.OOCZ_UPREV)
    assert np.array_equal(bits(got_u), bits(want_u))
    assert np.array_equal(bits(got_up), bits(want_up))


def test_load_rejects_wrong_size_and_field():
    z = Z()
    cfg = z.oocz_default_config(16, 16, 32, tb=2, block_planes=16, rate=[16, 16, 16])
    with z.Stepper(cfg) as s:
        with pytest.raises(z.OoczError):
            z.oocz_load_store(s.ctx, z.OOCZ_U, np.zeros(7, np.uint8))
        with pytest.raises(z.OoczError):
            z.oocz_save_store(s.ctx, z.OOCZ_U)          # never set
        assert z.oocz_store_bytes(s.ctx, 5) == 0
