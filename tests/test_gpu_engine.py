"""End-to-end parity of the out-of-core stepper (oocz_create / set_field /
step / get_field) vs the oracle's reduced schedule: in-core
steps plus a whole-field round trip after every sweep.  Bar: bit-exact."""
import numpy as np
import pytest

import oracle
from paper_2109_05410_b200 import synth
from gpu_util import Z, bits

pytestmark = pytest.mark.gpu


def _fields(nx, ny, nz, seed, kind="dense"):
    if kind == "pulse":
        u = synth.pulse(nx, ny, nz, sigma=4.0)
        up = u.copy()
    else:
        u = synth.dense(nx, ny, nz, seed=seed)
        up = (synth.dense(nx, ny, nz, seed=seed + 1) * np.float32(0.9)).astype(np.float32)
    return u, up, synth.layered(nx, ny, nz)


def _run_gpu(u, up, m, T, P, rates, store, calls, slots=2, profile=0, serpentine=0, m_resident=0, slab_sets=0,
             cone=0, resident_blocks=0):
    z = Z()
    nz, ny, nx = u.shape
    cfg = z.oocz_default_config(nx, ny, nz, tb=T, block_planes=P, rate=list(rates), store=store,
                                slots=slots, profile=profile, serpentine=serpentine, m_resident=m_resident,
                                slab_sets=slab_sets, cone=cone, resident_blocks=resident_blocks)
    with z.Stepper(cfg) as s:
        s.set(u, up, m)
        for n in calls:
            s.step(n)
        return s.get(z.OOCZ_U), s.get(z.OOCZ_UPREV), s.stats(), (z.oocz_get_events(s.ctx) if profile else None)


def _run_oracle(u, up, m, T, rates, calls):
    a = oracle.roundtrip(u, rates[0])
    b = oracle.roundtrip(up, rates[1])
    mm = oracle.roundtrip(m, rates[2])
    for n in calls:
        a, b = oracle.advance(a, b, mm, T, rates, n)
    return a, b


CASES = [
    # nx, ny, nz, T, P, rates, calls
    (64, 64, 64, 2, 32, (16, 16, 16), [10]),          # C1 shape (BASELINE configs[0])
    (32, 24, 64, 2, 16, (0, 0, 0), [10]),             # raw
    (40, 16, 96, 3, 24, (8, 12, 24), [7]),            # mixed rates, n mod T != 0
    (24, 28, 48, 1, 8, (16, 0, 4), [3, 2]),           # split calls
    (32, 32, 32, 4, 32, (16, 16, 16), [8]),           # D = 1
    (136, 12, 64, 2, 16, (24, 24, 24), [6]),          # ragged CTA tiles
]


@pytest.mark.parametrize("slab_sets", [1, 2, 3])
@pytest.mark.parametrize("serpentine", [0, 1])
@pytest.mark.parametrize("store", [0, 1])
@pytest.mark.parametrize("nx,ny,nz,T,P,rates,calls", CASES)
def test_stepper_matches_oracle(store, serpentine, slab_sets, nx, ny, nz, T, P, rates, calls):
    u, up, m = _fields(nx, ny, nz, 3)
    gu, gup, st, _ = _run_gpu(u, up, m, T, P, rates, store, calls, serpentine=serpentine, slab_sets=slab_sets)
    ou, oup = _run_oracle(u, up, m, T, rates, calls)
    assert np.array_equal(bits(gu), bits(ou))
    assert np.array_equal(bits(gup), bits(oup))


def test_c1_config_bit_exact_and_byte_accounting():
    """BASELINE configs[0]: 64^3, 2 z-blocks, rate 16, 10 steps (PULSE + LAYERED)."""
    u, up, m = _fields(64, 64, 64, 0, kind="pulse")
    rates = (16, 16, 16)
    gu, gup, st, evs = _run_gpu(u, up, m, 2, 32, rates, 0, [10], profile=1)
    ou, oup = _run_oracle(u, up, m, 2, rates, [10])
    assert np.array_equal(bits(gu), bits(ou)) and np.array_equal(bits(gup), bits(oup))
    stored = oracle.zfp_bytes(64, 64, 64, 16)
    assert st["sweeps"] == 5
    assert st["h2d_bytes"] == 5 * 3 * stored         # region sharing: every plane once per sweep
    assert st["d2h_bytes"] == 5 * 2 * stored         # m is never written back
    assert st["kernel_launches"] > 0
    _audit(evs)


def _audit(evs):
    """SPEC.md:285-286 StageEvent invariants: per block h2d <= decode <= stencil
    <= encode <= d2h in start order; no two events on one lane overlap."""
    assert evs
    by_lane = {}
    for e in evs:
        assert e["end_ms"] >= e["start_ms"]
        by_lane.setdefault(e["lane"], []).append(e)
    for lane, es in by_lane.items():
        es.sort(key=lambda e: e["start_ms"])
        for a, b in zip(es, es[1:]):
            assert b["start_ms"] >= a["end_ms"] - 1e-3, (lane, a, b)
    order = [0, 1, 2, 3, 4]
    blocks = {}
    for e in evs:
        blocks.setdefault((e["sweep"], e["block"]), {}).setdefault(e["stage"], e)
    for key, stg in blocks.items():
        starts = [stg[s]["start_ms"] for s in order if s in stg]
        assert starts == sorted(starts), key


@pytest.mark.parametrize("slab_sets", [2, 3])
@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("rates", [(16, 16, 16), (0, 0, 0), (8, 24, 12)])
def test_partitioned_group_bit_identical_to_single(world, rates, slab_sets):
    """z-partitioned run (halos exchanged in compressed form) == world 1 == oracle."""
    z = Z()
    nx, ny, nz, T, P = 32, 24, 128, 2, 16
    u, up, m = _fields(nx, ny, nz, 5)
    cfg = z.oocz_default_config(nx, ny, nz, tb=T, block_planes=P, rate=list(rates), store=0, slab_sets=slab_sets)
    ctxs = z.oocz_create_local_group(cfg, world)
    S = nz // world
    try:
        for r, c in enumerate(ctxs):
            for f, a in ((z.OOCZ_U, u), (z.OOCZ_UPREV, up), (z.OOCZ_M, m)):
                z.oocz_set_field(c, f, a[r * S:(r + 1) * S])
        z.oocz_step_local_group(ctxs, 7)
        gu = np.concatenate([z.oocz_get_field(c, z.OOCZ_U, np.empty((S, ny, nx), np.float32)) for c in ctxs])
        gup = np.concatenate([z.oocz_get_field(c, z.OOCZ_UPREV, np.empty((S, ny, nx), np.float32)) for c in ctxs])
        halo = sum(z.oocz_get_stats(c)["halo_bytes"] for c in ctxs)
    finally:
        for c in ctxs:
            z.oocz_destroy(c)
    ou, oup = _run_oracle(u, up, m, T, rates, [7])
    assert np.array_equal(bits(gu), bits(ou))
    assert np.array_equal(bits(gup), bits(oup))
    h = 4 * T
    per = [oracle.zfp_bytes(nx, ny, h, r) if r else 4 * nx * ny * h for r in rates]
    sweeps = 4
    assert halo == (world - 1) * 2 * (sweeps * (per[0] + per[1]) + per[2])


def test_set_get_round_trip_and_errors():
    z = Z()
    nx, ny, nz = 16, 16, 32
    u, up, m = _fields(nx, ny, nz, 6)
    cfg = z.oocz_default_config(nx, ny, nz, tb=2, block_planes=16, rate=[12, 12, 12])
    with z.Stepper(cfg) as s:
        with pytest.raises(z.OoczError) as ei:
            s.step(1)                                   # fields not set
        assert ei.value.status == z.OOCZ_ESTATE
        bad = u.copy()
        bad[3, 4, 5] = np.nan
        with pytest.raises(z.OoczError) as ei:
            z.oocz_set_field(s.ctx, z.OOCZ_U, bad)
        assert ei.value.status == z.OOCZ_ENONFINITE
        with pytest.raises(z.OoczError) as ei:
            z.oocz_set_field(s.ctx, z.OOCZ_M, np.full_like(m, 0.21))   # > 105/512
        assert ei.value.status == z.OOCZ_ECFL
        with pytest.raises(z.OoczError) as ei:
            z.oocz_set_field(s.ctx, z.OOCZ_M, -m)
        assert ei.value.status == z.OOCZ_ECFL
        s.set(u, up, m)
        assert np.array_equal(bits(s.get(z.OOCZ_U)), bits(oracle.roundtrip(u, 12)))
        assert np.array_equal(bits(s.get(z.OOCZ_M)), bits(oracle.roundtrip(m, 12)))
        s.step(0)
        assert np.array_equal(bits(s.get(z.OOCZ_UPREV)), bits(oracle.roundtrip(up, 12)))


def test_slots_and_many_sweeps_pipelined():
    """Deep pipelines across many sweeps (cross-sweep hazards) stay exact."""
    u, up, m = _fields(32, 32, 128, 7)
    for slots in (2, 3, 5):
        gu, gup, _, _ = _run_gpu(u, up, m, 2, 16, (16, 16, 16), 0, [40], slots=slots)
        ou, oup = _run_oracle(u, up, m, 2, (16, 16, 16), [40])
        assert np.array_equal(bits(gu), bits(ou)) and np.array_equal(bits(gup), bits(oup)), slots


@pytest.mark.parametrize("store", [0, 1])
@pytest.mark.parametrize("nx,ny,nz,T,P,rates,calls", [CASES[0], CASES[2], CASES[3], CASES[4]])
def test_m_resident_matches_oracle(store, nx, ny, nz, T, P, rates, calls):
    """Orchestration beyond the paper: m decoded once and
    kept in HBM -- same bits, and no m bytes on the host link."""
    z = Z()
    u, up, m = _fields(nx, ny, nz, 3)
    cfg = z.oocz_default_config(nx, ny, nz, tb=T, block_planes=P, rate=list(rates), store=store, m_resident=1)
    with z.Stepper(cfg) as s:
        s.set(u, up, m)
        for n in calls:
            s.step(n)
        gu, gup, st = s.get(z.OOCZ_U), s.get(z.OOCZ_UPREV), s.stats()
    ou, oup = _run_oracle(u, up, m, T, rates, calls)
    assert np.array_equal(bits(gu), bits(ou)) and np.array_equal(bits(gup), bits(oup))
    if store == 0:
        stored = [oracle.zfp_bytes(nx, ny, nz, r) if r else 4 * nx * ny * nz for r in rates]
        assert st["h2d_bytes"] == st["sweeps"] * (stored[0] + stored[1])


@pytest.mark.parametrize("world", [2, 4])
def test_m_resident_partitioned_group(world):
    z = Z()
    nx, ny, nz, T, P, rates = 32, 24, 128, 2, 16, (16, 12, 8)
    u, up, m = _fields(nx, ny, nz, 5)
    cfg = z.oocz_default_config(nx, ny, nz, tb=T, block_planes=P, rate=list(rates), store=0, m_resident=1)
    ctxs = z.oocz_create_local_group(cfg, world)
    S = nz // world
    try:
        for r, c in enumerate(ctxs):
            for f, a in ((z.OOCZ_U, u), (z.OOCZ_UPREV, up), (z.OOCZ_M, m)):
                z.oocz_set_field(c, f, a[r * S:(r + 1) * S])
        z.oocz_step_local_group(ctxs, 7)
        gu = np.concatenate([z.oocz_get_field(c, z.OOCZ_U, np.empty((S, ny, nx), np.float32)) for c in ctxs])
    finally:
        for c in ctxs:
            z.oocz_destroy(c)
    ou, _ = _run_oracle(u, up, m, T, rates, [7])
    assert np.array_equal(bits(gu), bits(ou))


def _serpentine_bytes(D, P, h, T, calls, slots, nf, row):
    """Host-link bytes of serpentine sweeps, modelled from the rule (DESIGN.md
    R22): a read-unit part is decoded from a staging slot when the block that
    encoded it is at most `slots` blocks back in the sequence; the last
    nkeep = min(D, (slots + 1) // 2) blocks before each turn skip their D2H (their
    rows are read from their slots after the turn); m rows (nf == 3) always
    cross, except at a turn."""
    S = D * P
    nkeep = min(D, (slots + 1) // 2)
    h2d = d2h = 0
    seq, last = 0, [-1] * D
    for n in calls:
        k = -(-n // T)
        for s_ in range(k):
            asc = s_ % 2 == 0
            for kk in range(D):
                i = kk if asc else D - 1 - kk
                turn = s_ > 0 and kk == 0
                keep = s_ < k - 1 and kk >= D - nkeep
                if asc:
                    rd0, rd1 = (0 if i == 0 else i * P + h), min((i + 1) * P + h, S)
                    nb = min(i + 1, D - 1)
                    parts = [(rd0, min(rd1, (i + 1) * P), i), ((i + 1) * P, rd1, nb)]
                else:
                    rd0, rd1 = max(i * P - h, 0), (S if i == D - 1 else (i + 1) * P - h)
                    nb = max(i - 1, 0)
                    parts = [(rd0, i * P, nb), (max(rd0, i * P), rd1, i)]
                for z0, z1, owner in parts:
                    if z1 <= z0:
                        continue
                    on_dev = last[owner] >= 0 and seq <= last[owner] + slots
                    for f in range(nf):
                        if f == 2:
                            h2d += 0 if turn else (z1 - z0) // 4 * row[2]
                        elif not on_dev:
                            h2d += (z1 - z0) // 4 * row[f]
                last[i] = seq
                if not keep:
                    d2h += (P // 4) * (row[0] + row[1])
                seq += 1
        last = [x if x >= 0 else -1 for x in last]
    return h2d, d2h


@pytest.mark.parametrize("slab_sets", [1, 2, 3, 4])
@pytest.mark.parametrize("m_resident", [0, 1])
@pytest.mark.parametrize("slots", [2, 3, 5])
@pytest.mark.parametrize("D,calls", [(4, [12]), (3, [5, 7]), (1, [9]), (2, [4, 4, 1]), (6, [14, 3])])
def test_serpentine_bit_exact_and_bytes(D, calls, slots, m_resident, slab_sets):
    """Serpentine sweeps (R22): same bits as the oracle, and exactly the
    host-link bytes of the schedule's model: the block at each turn never crosses
    the link, and with slots >= 3 the rows of recent blocks are decoded from the
    staging slots instead of crossing twice."""
    nx, ny, T, P, rates = 32, 24, 2, 16, (16, 12, 8)
    nz = D * P
    u, up, m = _fields(nx, ny, nz, 11)
    gu, gup, st, evs = _run_gpu(u, up, m, T, P, rates, 0, calls, slots=slots, profile=1, serpentine=1,
                                m_resident=m_resident, slab_sets=slab_sets)
    ou, oup = _run_oracle(u, up, m, T, rates, calls)
    assert np.array_equal(bits(gu), bits(ou)) and np.array_equal(bits(gup), bits(oup))
    row = [oracle.zfp_bytes(nx, ny, 4, r) for r in rates]
    nf = 2 if m_resident else 3
    h2d, d2h = _serpentine_bytes(D, P, 4 * T, T, calls, slots, nf, row)
    assert st["h2d_bytes"] == h2d
    assert st["d2h_bytes"] == d2h
    _audit(evs)


@pytest.mark.parametrize("world", [2, 4])
def test_serpentine_partitioned_group(world):
    z = Z()
    nx, ny, nz, T, P, rates = 32, 24, 128, 2, 16, (16, 12, 8)
    u, up, m = _fields(nx, ny, nz, 5)
    cfg = z.oocz_default_config(nx, ny, nz, tb=T, block_planes=P, rate=list(rates), store=0, serpentine=1)
    ctxs = z.oocz_create_local_group(cfg, world)
    S = nz // world
    try:
        for r, c in enumerate(ctxs):
            for f, a in ((z.OOCZ_U, u), (z.OOCZ_UPREV, up), (z.OOCZ_M, m)):
                z.oocz_set_field(c, f, a[r * S:(r + 1) * S])
        z.oocz_step_local_group(ctxs, 9)
        gu = np.concatenate([z.oocz_get_field(c, z.OOCZ_U, np.empty((S, ny, nx), np.float32)) for c in ctxs])
        gup = np.concatenate([z.oocz_get_field(c, z.OOCZ_UPREV, np.empty((S, ny, nx), np.float32)) for c in ctxs])
    finally:
        for c in ctxs:
            z.oocz_destroy(c)
    ou, oup = _run_oracle(u, up, m, T, rates, [9])
    assert np.array_equal(bits(gu), bits(ou)) and np.array_equal(bits(gup), bits(oup))


@pytest.fixture(scope="module")
def c2_state():
    """BASELINE configs[1] at full size: the bench's 512^3 DENSE(1) / LAYERED
    workload, and the oracle's result after 2 sweeps (T = 4, rate 16)."""
    n = 512
    u = synth.dense(n, n, n, seed=1)
    m = synth.layered(n, n, n)
    ou, oup = oracle.run(u, u, m, 4, (16, 16, 16), 8)
    return u, m, ou, oup


@pytest.mark.parametrize("store,opts", [
    (1, dict(m_resident=1)),                                  # bench value path
    (0, dict(serpentine=1, m_resident=1, slots=4)),           # bench e2e path (C2)
    (0, dict(serpentine=1, m_resident=1, slots=3)),           # 3 slots: 2 kept blocks per turn
    (0, dict()),                                              # the paper-faithful schedule
])
def test_c2_full_size_bench_configs_bit_exact(c2_state, store, opts):
    """The bench's own launch configurations (512^3, P = 128, T = 4, rate 16) for
    2 sweeps -- covering a serpentine turn -- equal the oracle bit for bit over
    the whole field."""
    u, m, ou, oup = c2_state
    z = Z()
    cfg = z.oocz_default_config(512, 512, 512, tb=4, block_planes=128, rate=[16, 16, 16], store=store, **opts)
    with z.Stepper(cfg) as s:
        s.set(u, u, m)
        s.step(8)
        gu, gup = s.get(z.OOCZ_U), s.get(z.OOCZ_UPREV)
    assert np.array_equal(bits(gu), bits(ou))
    assert np.array_equal(bits(gup), bits(oup))


@pytest.mark.parametrize("store", [0, 1])
def test_extreme_rates(store):
    """Rate 1 (the smallest: 8 bytes per 4^3 block) and rate 64 (more bits than
    the raw value) through the whole stepper, mixed with raw."""
    nx, ny, nz, T, P = 32, 16, 48, 2, 16
    u, up, m = _fields(nx, ny, nz, 9)
    for rates in ((1, 64, 0), (64, 1, 2)):
        gu, gup, _, _ = _run_gpu(u, up, m, T, P, rates, store, [6], serpentine=1, m_resident=1, slots=3)
        ou, oup = _run_oracle(u, up, m, T, rates, [6])
        assert np.array_equal(bits(gu), bits(ou)) and np.array_equal(bits(gup), bits(oup)), rates


@pytest.mark.parametrize("seed", [2024, 7, 99])
def test_random_configurations_bit_exact(seed):
    """96 seeded random configurations of everything the stepper accepts --
    grid shape, T, P, per-field rates (raw to 64), store location, slots,
    slab sets, serpentine, m resident, resident blocks (host store), split calls --
    against the oracle.  (This test found the separate-encode-stream race.)"""
    rng = np.random.default_rng(seed)
    for case in range(96):
        T = int(rng.integers(1, 4))
        h = 4 * T
        P = int(rng.choice([q for q in (8, 12, 16, 20, 24, 32) if q >= 2 * h]))
        D = int(rng.integers(1, 5))
        nz = P * D
        nx, ny = 4 * int(rng.integers(2, 12)), 4 * int(rng.integers(1, 8))
        rates = tuple(int(rng.choice([0, 1, 3, 8, 12, 16, 24, 33, 64])) for _ in range(3))
        store = int(rng.integers(0, 2))
        opts = dict(slots=int(rng.integers(2, 5)), slab_sets=int(rng.choice([0, 1, 2, 3, 4])),
                    serpentine=int(rng.integers(0, 2)), m_resident=int(rng.integers(0, 2)))
        calls = [int(x) for x in rng.integers(1, 3 * T + 2, size=int(rng.integers(1, 4)))]
        if store == 0:      # (its own generator: the draws above stay those of earlier rounds)
            opts["resident_blocks"] = int(np.random.default_rng(1000 * seed + case).integers(0, D + 1))
        u, up, m = _fields(nx, ny, nz, 100 + case)
        gu, gup, _, _ = _run_gpu(u, up, m, T, P, rates, store, calls, **opts)
        ou, oup = _run_oracle(u, up, m, T, rates, calls)
        cfg = (nx, ny, nz, T, P, rates, store, opts, calls)
        assert np.array_equal(bits(gu), bits(ou)) and np.array_equal(bits(gup), bits(oup)), cfg


def test_random_partitioned_configurations_bit_exact(seed=4242):
    """24 seeded random z-partitioned runs (in-process local group of 2-4 ranks,
    compressed halos) with every orchestration option: equal to the oracle,
    i.e. to world 1, bit for bit."""
    z = Z()
    rng = np.random.default_rng(seed)
    for case in range(24):
        world = int(rng.choice([2, 3, 4]))
        T = int(rng.integers(1, 3))
        P = int(rng.choice([q for q in (8, 12, 16) if q >= 8 * T]))
        S = P * int(rng.integers(1, 3))
        nz = S * world
        nx, ny = 4 * int(rng.integers(2, 9)), 4 * int(rng.integers(1, 6))
        rates = tuple(int(rng.choice([0, 3, 12, 16, 33])) for _ in range(3))
        opts = dict(store=int(rng.integers(0, 2)), slots=int(rng.integers(2, 4)),
                    slab_sets=int(rng.choice([0, 1, 3])), serpentine=int(rng.integers(0, 2)),
                    m_resident=int(rng.integers(0, 2)))
        n = int(rng.integers(1, 3 * T + 2))
        u, up, m = _fields(nx, ny, nz, 700 + case)
        cfg = z.oocz_default_config(nx, ny, nz, tb=T, block_planes=P, rate=list(rates), **opts)
        ctxs = z.oocz_create_local_group(cfg, world)
        try:
            for r, c in enumerate(ctxs):
                for f, a in ((z.OOCZ_U, u), (z.OOCZ_UPREV, up), (z.OOCZ_M, m)):
                    z.oocz_set_field(c, f, a[r * S:(r + 1) * S])
            z.oocz_step_local_group(ctxs, n)
            gu = np.concatenate([z.oocz_get_field(c, z.OOCZ_U, np.empty((S, ny, nx), np.float32)) for c in ctxs])
            gup = np.concatenate([z.oocz_get_field(c, z.OOCZ_UPREV, np.empty((S, ny, nx), np.float32)) for c in ctxs])
        finally:
            for c in ctxs:
                z.oocz_destroy(c)
        ou, oup = _run_oracle(u, up, m, T, rates, [n])
        assert np.array_equal(bits(gu), bits(ou)) and np.array_equal(bits(gup), bits(oup)), \
            (world, nx, ny, nz, T, P, rates, opts, n)


@pytest.mark.parametrize("serpentine,m_resident", [(0, 0), (1, 1)])
@pytest.mark.parametrize("rates", [(0, 0, 0), (16, 0, 16), (16, 16, 16)])
def test_paper_decomposition_bit_exact(rates, serpentine, m_resident):
    """The paper's own z decomposition (tests/golden/: 1152 interior planes,
    8 divisions, T = 12) with a small x/y extent."""
    from golden_io import keyvals
    s, t = keyvals("paper_sec5_schedule.txt"), keyvals("paper_table1.txt")
    nz, T = t["interior"], s["temporal_blocking"]
    P = nz // s["divisions"]
    nx, ny = 32, 24
    u, up, m = _fields(nx, ny, nz, 77)
    gu, gup, st, _ = _run_gpu(u, up, m, T, P, rates, 0, [2 * T], serpentine=serpentine, m_resident=m_resident)
    ou, oup = _run_oracle(u, up, m, T, rates, [2 * T])
    assert np.array_equal(bits(gu), bits(ou)) and np.array_equal(bits(gup), bits(oup))
    assert st["sweeps"] == 2


@pytest.mark.parametrize("slab_sets", [1, 2, 3])
@pytest.mark.parametrize("nx,ny,nz,T,P,rates,calls", CASES + [
    (64, 64, 64, 2, 32, (16, 16, 16), [10, 10, 3, 10]),     # cached graphs reused, a partial sweep
    (32, 32, 128, 1, 8, (12, 0, 8), [40]),                  # 40 sweeps: three chunks of <= 16
])
def test_graphs_bit_exact(nx, ny, nz, T, P, rates, calls, slab_sets):
    """cfg.graphs = 1 (store in HBM): the captured-and-replayed sweeps give the
    eager path's bits, call after call, and count the same kernel launches."""
    u, up, m = _fields(nx, ny, nz, 11)
    z = Z()
    launches = []
    outs = []
    for graphs in (0, 1):
        cfg = z.oocz_default_config(nx, ny, nz, tb=T, block_planes=P, rate=list(rates), store=1,
                                    slab_sets=slab_sets, graphs=graphs)
        with z.Stepper(cfg) as s:
            s.set(u, up, m)
            l0 = z.oocz_kernel_launch_count()
            for n in calls:
                s.step(n)
            launches.append(z.oocz_kernel_launch_count() - l0)
            st = s.stats()
            outs.append((s.get(z.OOCZ_U), s.get(z.OOCZ_UPREV), st["sweeps"]))
    ou, oup = _run_oracle(u, up, m, T, rates, calls)
    for gu, gup, _ in outs:
        assert np.array_equal(bits(gu), bits(ou)) and np.array_equal(bits(gup), bits(oup))
    assert outs[0][2] == outs[1][2] and launches[0] == launches[1]


def test_graphs_ignored_where_not_eligible():
    """Host store (or serpentine / profile): graphs = 1 falls back to the eager
    path, same bits."""
    nx, ny, nz, T, P, rates = 32, 24, 64, 2, 16, (16, 16, 16)
    u, up, m = _fields(nx, ny, nz, 12)
    z = Z()
    cfg = z.oocz_default_config(nx, ny, nz, tb=T, block_planes=P, rate=list(rates), store=0, graphs=1,
                                serpentine=1, slots=3)
    with z.Stepper(cfg) as s:
        s.set(u, up, m)
        s.step(7)
        gu = s.get(z.OOCZ_U)
    ou, _ = _run_oracle(u, up, m, T, rates, [7])
    assert np.array_equal(bits(gu), bits(ou))


@pytest.mark.parametrize("nx,ny,nz,T,P,calls", [(32, 24, 96, 3, 24, [7]), (24, 16, 64, 2, 16, [4, 3]),
                                                (16, 16, 128, 4, 32, [8])])
def test_parallelogram_updates_every_cell_once_per_step(nx, ny, nz, T, P, calls):
    """Reading R26: every block updates exactly P planes per step (parallelogram
    tiles, mirrored in the descending sweeps of serpentine runs), so one step of
    the whole grid costs the stencil 16 B per cell and no more, where the paper's
    trapezoid cone costs (P + 2h - 8s) planes per block.  Bit-exact against the
    oracle either way."""
    u, up, m = _fields(nx, ny, nz, 13)
    rates = (16, 16, 16)
    ou, oup = _run_oracle(u, up, m, T, rates, calls)
    pb = nx * ny * 4
    stencil_bytes = {}
    for serp in (0, 1):
        gu, gup, st, evs = _run_gpu(u, up, m, T, P, rates, 1, calls, profile=1, serpentine=serp)
        assert np.array_equal(bits(gu), bits(ou)) and np.array_equal(bits(gup), bits(oup))
        # events of the last call only
        stencil_bytes[serp] = sum(e["bytes"] for e in evs if e["stage"] == 2)
    last = calls[-1]
    for serp in (0, 1):                                     # read u, u-, m, write u+ once per cell and step
        assert stencil_bytes[serp] == 4 * nz * pb * last


@pytest.mark.parametrize("nx,ny,nz,T,P,calls", [(32, 24, 96, 3, 24, [7]), (24, 16, 64, 2, 16, [4, 3]),
                                                (16, 16, 128, 4, 32, [8])])
def test_paper_trapezoid_cone_bit_exact_and_its_cost(nx, ny, nz, T, P, calls):
    """cone = 1: the paper's own temporal-blocking shape,
    block i updates [iP - h + 4s, (i+1)P + h - 4s) in step s, recomputing the
    overlap.  Same bits as the oracle (and as the parallelogram tiles), in both
    sweep directions, and the stencil's algorithmic bytes are exactly the cone's:
    sum over blocks and steps of the cone's planes clipped to the grid."""
    u, up, m = _fields(nx, ny, nz, 14)
    rates = (16, 16, 16)
    ou, oup = _run_oracle(u, up, m, T, rates, calls)
    pb = nx * ny * 4
    h, D = 4 * T, nz // P
    last = calls[-1]
    for serp in (0, 1):
        for store in (0, 1):
            gu, gup, st, evs = _run_gpu(u, up, m, T, P, rates, store, calls, profile=1, serpentine=serp, cone=1,
                                        m_resident=serp)
            assert np.array_equal(bits(gu), bits(ou)) and np.array_equal(bits(gup), bits(oup)), (serp, store)
            got = sum(e["bytes"] for e in evs if e["stage"] == 2)
            want = 0
            done = 0
            while done < last:
                ts = min(T, last - done)
                for i in range(D):
                    for step in range(1, ts + 1):
                        z0, z1 = max(i * P - h + 4 * step, 0), min((i + 1) * P + h - 4 * step, nz)
                        want += 16 * (z1 - z0) * nx * ny
                done += ts
            assert got == want, (serp, store, got, want)


def test_random_configurations_cone_bit_exact(seed=77):
    """48 seeded random configurations with the paper's trapezoid cone."""
    rng = np.random.default_rng(seed)
    for case in range(48):
        T = int(rng.integers(1, 4))
        P = int(rng.choice([q for q in (8, 12, 16, 20, 24, 32) if q >= 8 * T]))
        nz = P * int(rng.integers(1, 5))
        nx, ny = 4 * int(rng.integers(2, 12)), 4 * int(rng.integers(1, 8))
        rates = tuple(int(rng.choice([0, 3, 8, 16, 24, 64])) for _ in range(3))
        store = int(rng.integers(0, 2))
        opts = dict(slots=int(rng.integers(2, 5)), slab_sets=int(rng.choice([0, 1, 2, 3])),
                    serpentine=int(rng.integers(0, 2)), m_resident=int(rng.integers(0, 2)))
        calls = [int(x) for x in rng.integers(1, 3 * T + 2, size=int(rng.integers(1, 3)))]
        u, up, m = _fields(nx, ny, nz, 300 + case)
        gu, gup, _, _ = _run_gpu(u, up, m, T, P, rates, store, calls, cone=1, **opts)
        ou, oup = _run_oracle(u, up, m, T, rates, calls)
        assert np.array_equal(bits(gu), bits(ou)) and np.array_equal(bits(gup), bits(oup)), \
            (nx, ny, nz, T, P, rates, store, opts, calls)


@pytest.mark.parametrize("precision", [32, 64])
@pytest.mark.parametrize("calls", [[8], [5, 2], [1, 1, 3]])
def test_raw_device_store_steps_in_core(precision, calls):
    """Raw fields with the store in HBM step in core: one whole-grid stencil
    launch per step, the time levels swapping by pointer, no copies -- bit-exact
    against the oracle (and so against the block schedule), with the stencil's
    16 B per cell-update as the only recorded traffic."""
    import oracle as O
    z = Z()
    nx, ny, nz, T, P = 40, 24, 96, 3, 24
    u, up, m = _fields(nx, ny, nz, 41)
    if precision == 64:
        u, up, m = (a.astype(np.float64) for a in (u, up, m))
        a, b = u, up
        for n in calls:
            a, b = O.advance64(a, b, m, T, (0, 0, 0), n)
        view = np.uint64
    else:
        a, b = _run_oracle(u, up, m, T, (0, 0, 0), calls)
        view = np.uint32
    cfg = z.oocz_default_config(nx, ny, nz, tb=T, block_planes=P, rate=[0, 0, 0], store=1, profile=1,
                                precision=precision, m_resident=1)
    with z.Stepper(cfg) as s:
        s.set(u, up, m)
        l0 = s.stats()["kernel_launches"]
        for n in calls:
            s.step(n)
        st = s.stats()
        assert st["kernel_launches"] - l0 == sum(calls)
        assert st["h2d_bytes"] == st["d2h_bytes"] == 0
        evs = z.oocz_get_events(s.ctx)
        assert {e["stage"] for e in evs} == {2}                          # stencil
        assert sum(e["bytes"] for e in evs) == 4 * nz * nx * ny * (8 if precision == 64 else 4) * calls[-1]
        assert np.array_equal(s.get(z.OOCZ_U).view(view), a.view(view))
        assert np.array_equal(s.get(z.OOCZ_UPREV).view(view), b.view(view))
