"""fp64 path (the paper's own precision; its rates 32/64 and
24/64) vs the fp64 oracle: codec streams bit-exact, stencil
bit-exact (prescribed order, R5 in fp64), the out-of-core stepper
bit-exact against the reduced schedule c.0 in fp64 (oracle.run64)."""
import numpy as np
import pytest

import oracle
from paper_2109_05410_b200 import synth
from gpu_util import Z, to_dev

pytestmark = pytest.mark.gpu


def b64(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


def _dense64(nx, ny, nz, seed):
    """fp64 workload: the DENSE field plus a term below fp32 resolution, so all
    52 mantissa bits carry information."""
    f = synth.dense(nx, ny, nz, seed=seed).astype(np.float64)
    fine = synth.uniforms(seed + 7, nx * ny * nz).reshape(nz, ny, nx) - 0.5
    return f + fine * 2.0 ** -30


def _fields64():
    rb = synth.random_blocks(5 * 3 * 7, seed=41).astype(np.float64)
    wide = np.random.default_rng(3).standard_normal((4, 8, 1032)) * 2.0 ** np.random.default_rng(4).integers(
        -1000, 1000, (4, 8, 1032))
    return {
        "dense64": _dense64(48, 36, 20, 1),
        "pulse": synth.pulse(64, 64, 64, sigma=4.0).astype(np.float64),
        "layered": synth.layered(40, 24, 16).astype(np.float64),
        "adversarial": synth.blocks_to_field(rb, 5, 3, 7),
        "wide_range": wide,                                     # 258 blocks, exponents across fp64
        "denormal": np.random.default_rng(5).integers(-(1 << 52), 1 << 52, (8, 8, 12)) * 2.0 ** -1074,
        "zeros": np.zeros((8, 8, 8)),
    }


def gpu_encode64(f, rate):
    import torch
    z = Z()
    nz, ny, nx = f.shape
    n = z.oocz_zfp_bytes(nx, ny, nz, rate) // 8
    out = torch.empty(max(n, 1), dtype=torch.int64, device="cuda")
    z.oocz_zfp_encode_f64(to_dev(np.ascontiguousarray(f, np.float64)), nx, ny, nz, rate, out,
                          torch.cuda.current_stream())
    torch.cuda.synchronize()
    return out.cpu().numpy().view(np.uint64)[:n]


def gpu_decode64(words, shape, rate):
    import torch
    z = Z()
    nz, ny, nx = shape
    out = torch.empty(shape, dtype=torch.float64, device="cuda")
    z.oocz_zfp_decode_f64(to_dev(np.ascontiguousarray(words, np.uint64).view(np.int64)), nx, ny, nz, rate, out,
                          torch.cuda.current_stream())
    torch.cuda.synchronize()
    return out.cpu().numpy()


@pytest.mark.parametrize("rate", [1, 8, 16, 24, 32, 48, 64])
def test_encode64_bit_exact(rate):
    for name, f in _fields64().items():
        want = oracle.zfp_encode64(f, rate)
        got = gpu_encode64(f, rate)
        bad = np.nonzero(got != want)[0]
        assert bad.size == 0, (name, rate, bad[:5])


@pytest.mark.parametrize("rate", [1, 12, 24, 32, 64])
def test_decode64_bit_exact(rate):
    for name, f in _fields64().items():
        words = oracle.zfp_encode64(f, rate)
        want = oracle.zfp_decode64(words, f.shape, rate)
        got = gpu_decode64(words, f.shape, rate)
        assert np.array_equal(b64(got), b64(want)), (name, rate)


@pytest.mark.parametrize("rate", [3, 24, 41, 64])
def test_decode64_arbitrary_streams(rate):
    rng = np.random.default_rng(rate)
    shape = (12, 16, 20)
    n = oracle.zfp_bytes(20, 16, 12, rate) // 8
    for trial in range(4):
        words = rng.integers(0, 1 << 63, n, dtype=np.uint64) * 2 + rng.integers(0, 2, n, dtype=np.uint64)
        if trial % 2:
            words &= rng.integers(0, 1 << 63, n, dtype=np.uint64)
            words |= np.uint64(1)
        want = oracle.zfp_decode64(words, shape, rate)
        got = gpu_decode64(words, shape, rate)
        assert np.array_equal(b64(got), b64(want)), (rate, trial)


def _state64(nx, ny, nz, seed):
    return _dense64(nx, ny, nz, seed), 0.5 * _dense64(nx, ny, nz, seed + 100), synth.layered(nx, ny, nz).astype(np.float64)


@pytest.mark.parametrize("shape,n", [((64, 64, 64), 1), ((136, 10, 37), 3), ((12, 20, 9), 2), ((4, 4, 4), 1),
                                     ((264, 20, 30), 4)])
def test_stencil64_bit_exact(shape, n):
    import torch
    z = Z()
    nx, ny, nz = shape
    u, up, m = _state64(nx, ny, nz, 9)
    a, b = u, up
    for _ in range(n):
        a, b = oracle.step_f64(a, b, m), a
    du, dup, dm = to_dev(u), to_dev(up), to_dev(m)
    z.oocz_stencil_steps_f64(du, dup, dm, nx, ny, nz, z.default_coeffs64(), n, torch.cuda.current_stream())
    torch.cuda.synchronize()
    assert np.array_equal(b64(du.cpu().numpy()), b64(a))
    assert np.array_equal(b64(dup.cpu().numpy()), b64(b))


@pytest.mark.parametrize("z0,z1,zv0,zv1", [(4, 28, 0, 32), (8, 20, 4, 24), (0, 32, 0, 32), (12, 13, 10, 16)])
def test_stencil64_cone_limited(z0, z1, zv0, zv1):
    import torch
    z = Z()
    nx, ny, nz = 40, 24, 32
    u, up, m = _state64(nx, ny, nz, 11)
    uz = u.copy()
    uz[:zv0] = 0
    uz[zv1:] = 0
    want = up.copy()
    want[z0:z1] = oracle.step_f64(uz, up, m)[z0:z1]
    du, dup, dm = to_dev(u), to_dev(up), to_dev(m)
    z.oocz_stencil_step_planes_f64(du, dup, dm, nx, ny, nz, z.default_coeffs64(), z0, z1, zv0, zv1,
                                   torch.cuda.current_stream())
    torch.cuda.synchronize()
    assert np.array_equal(b64(dup.cpu().numpy()), b64(want))


CASES64 = [
    # nx, ny, nz, T, P, rates, calls
    (64, 64, 64, 2, 32, (32, 32, 32), [10]),          # C1 shape at the paper's 2:1 rate
    (32, 24, 64, 2, 16, (24, 24, 24), [7]),           # paper's 24/64
    (40, 16, 96, 3, 24, (0, 16, 40), [7, 2]),         # raw + mixed, split calls
    (136, 12, 64, 2, 16, (64, 0, 12), [6]),           # ragged tiles
]


def _run64_gpu(u, up, m, T, P, rates, store, calls, m_resident=0, serpentine=0, **kw):
    z = Z()
    nz, ny, nx = u.shape
    cfg = z.oocz_default_config(nx, ny, nz, tb=T, block_planes=P, rate=list(rates), store=store,
                                precision=64, m_resident=m_resident, serpentine=serpentine, **kw)
    with z.Stepper(cfg) as s:
        s.set(u, up, m)
        for n in calls:
            s.step(n)
        return s.get(z.OOCZ_U), s.get(z.OOCZ_UPREV), s.stats()


def _run64_oracle(u, up, m, T, rates, calls):
    a, b, mm = (oracle.roundtrip64(x, r) for x, r in zip((u, up, m), rates))
    for n in calls:
        a, b = oracle.advance64(a, b, mm, T, rates, n)
    return a, b


@pytest.mark.parametrize("store,m_resident,serp", [(0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1), (1, 1, 1)])
@pytest.mark.parametrize("nx,ny,nz,T,P,rates,calls", CASES64)
def test_stepper64_matches_oracle(store, m_resident, serp, nx, ny, nz, T, P, rates, calls):
    u, up, m = _state64(nx, ny, nz, 3)
    gu, gup, st = _run64_gpu(u, up, m, T, P, rates, store, calls, m_resident, serp)
    ou, oup = _run64_oracle(u, up, m, T, rates, calls)
    assert np.array_equal(b64(gu), b64(ou)) and np.array_equal(b64(gup), b64(oup))
    if store == 0 and not serp:
        stored = [oracle.zfp_bytes(nx, ny, nz, r) if r else 8 * nx * ny * nz for r in rates]
        nf = 2 if m_resident else 3
        assert st["h2d_bytes"] == st["sweeps"] * sum(stored[:nf])


@pytest.mark.parametrize("world", [2, 4])
def test_partitioned64_bit_identical(world):
    z = Z()
    nx, ny, nz, T, P, rates = 32, 24, 128, 2, 16, (32, 24, 0)
    u, up, m = _state64(nx, ny, nz, 5)
    cfg = z.oocz_default_config(nx, ny, nz, tb=T, block_planes=P, rate=list(rates), store=0, precision=64)
    ctxs = z.oocz_create_local_group(cfg, world)
    S = nz // world
    try:
        for r, c in enumerate(ctxs):
            for f, a in ((z.OOCZ_U, u), (z.OOCZ_UPREV, up), (z.OOCZ_M, m)):
                z.oocz_set_field(c, f, a[r * S:(r + 1) * S])
        z.oocz_step_local_group(ctxs, 7)
        gu = np.concatenate([z.oocz_get_field(c, z.OOCZ_U, np.empty((S, ny, nx))) for c in ctxs])
        gup = np.concatenate([z.oocz_get_field(c, z.OOCZ_UPREV, np.empty((S, ny, nx))) for c in ctxs])
    finally:
        for c in ctxs:
            z.oocz_destroy(c)
    ou, oup = _run64_oracle(u, up, m, T, rates, [7])
    assert np.array_equal(b64(gu), b64(ou)) and np.array_equal(b64(gup), b64(oup))


def test_set_field64_checks():
    z = Z()
    nx, ny, nz = 16, 16, 32
    u, up, m = _state64(nx, ny, nz, 6)
    cfg = z.oocz_default_config(nx, ny, nz, tb=2, block_planes=16, rate=[32, 32, 32], precision=64)
    with z.Stepper(cfg) as s:
        bad = u.copy()
        bad[1, 2, 3] = np.inf
        with pytest.raises(z.OoczError) as ei:
            z.oocz_set_field(s.ctx, z.OOCZ_U, bad)
        assert ei.value.status == z.OOCZ_ENONFINITE
        lim = z.oocz_cfl_limit_f64(z.default_coeffs64())
        with pytest.raises(z.OoczError) as ei:
            z.oocz_set_field(s.ctx, z.OOCZ_M, np.full_like(m, np.nextafter(lim, 1.0)))
        assert ei.value.status == z.OOCZ_ECFL
        s.set(u, up, m)
        assert np.array_equal(b64(s.get(z.OOCZ_U)), b64(oracle.roundtrip64(u, 32)))


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_stencil_ring_release_stress(dtype):
    """Regression for a measured WAR race: a ring slot released while the
    consumer's shared-memory loads were still in flight (stencil
    "slot release").  Ragged last y-tiles made it visible in fp64 as wrong
    neighbours in ~10% of launches; 40 launches per shape must all be exact."""
    import torch
    z = Z()
    for (nx, ny, nz) in [(136, 10, 37), (264, 20, 30)]:
        if dtype == "f64":
            u, up, m = _state64(nx, ny, nz, 9)
            want = oracle.step_f64(u, up, m)
            fn, c = z.oocz_stencil_step_planes_f64, z.default_coeffs64()
        else:
            u, up, m = (a.astype(np.float32) for a in _state64(nx, ny, nz, 9))
            want = oracle.step(u, up, m)
            fn, c = z.oocz_stencil_step_planes, z.default_coeffs()
        du, dm = to_dev(u), to_dev(m)
        for _ in range(40):
            dup = to_dev(up)
            fn(du, dup, dm, nx, ny, nz, c, 0, nz, 0, nz, torch.cuda.current_stream())
            torch.cuda.synchronize()
            assert np.array_equal(dup.cpu().numpy(), want), (nx, ny, nz)


def test_random_configurations64_bit_exact(seed=64):
    """48 seeded random configurations in the paper's precision (fp64, rates
    raw / 1..64, every orchestration option) against the fp64 oracle."""
    rng = np.random.default_rng(seed)
    for case in range(48):
        T = int(rng.integers(1, 4))
        P = int(rng.choice([q for q in (8, 12, 16, 20, 24) if q >= 8 * T]))
        nz = P * int(rng.integers(1, 4))
        nx, ny = 4 * int(rng.integers(2, 10)), 4 * int(rng.integers(1, 7))
        rates = tuple(int(rng.choice([0, 1, 7, 16, 24, 32, 41, 64])) for _ in range(3))
        store = int(rng.integers(0, 2))
        kw = dict(slots=int(rng.integers(2, 4)), slab_sets=int(rng.choice([0, 1, 3])))
        serp, mres = int(rng.integers(0, 2)), int(rng.integers(0, 2))
        calls = [int(x) for x in rng.integers(1, 3 * T + 2, size=int(rng.integers(1, 3)))]
        u, up, m = _state64(nx, ny, nz, 500 + case)
        gu, gup, _ = _run64_gpu(u, up, m, T, P, rates, store, calls, mres, serp, **kw)
        ou, oup = _run64_oracle(u, up, m, T, rates, calls)
        assert np.array_equal(b64(gu), b64(ou)) and np.array_equal(b64(gup), b64(oup)), \
            (nx, ny, nz, T, P, rates, store, serp, mres, kw, calls)



@pytest.mark.parametrize("rates", [(32, 0, 0), (0, 0, 32), (24, 0, 24)])
def test_paper_codes_in_paper_decomposition64(rates):
    """The paper's four codes (uncompressed; one read-write
    dataset at 32/64; the read-only dataset at 32/64; one read-write and the
    read-only dataset at 24/64) in fp64, on the paper's z decomposition
    (tests/golden/: 1152 planes, 8 divisions, T = 12) with a small x/y extent."""
    from golden_io import keyvals
    s, t = keyvals("paper_sec5_schedule.txt"), keyvals("paper_table1.txt")
    nz, T = t["interior"], s["temporal_blocking"]
    P = nz // s["divisions"]
    nx, ny = 16, 12
    u, up, m = _state64(nx, ny, nz, 5)
    gu, gup, st = _run64_gpu(u, up, m, T, P, rates, 0, [2 * T])
    ou, oup = _run64_oracle(u, up, m, T, rates, [2 * T])
    assert np.array_equal(b64(gu), b64(ou)) and np.array_equal(b64(gup), b64(oup))
