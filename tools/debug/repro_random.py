import sys, os
_R = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))); sys.path.insert(0, os.path.join(_R, 'tests')); sys.path.insert(0, _R)
os.chdir('/root/repo')
import numpy as np
import test_gpu_engine as E
from gpu_util import bits
rng = np.random.default_rng(2024)
for case in range(96):
    T = int(rng.integers(1, 4)); h = 4 * T
    P = int(rng.choice([q for q in (8, 12, 16, 20, 24, 32) if q >= 2 * h]))
    D = int(rng.integers(1, 5)); nz = P * D
    nx, ny = 4 * int(rng.integers(2, 12)), 4 * int(rng.integers(1, 8))
    rates = tuple(int(rng.choice([0, 1, 3, 8, 12, 16, 24, 33, 64])) for _ in range(3))
    store = int(rng.integers(0, 2))
    opts = dict(slots=int(rng.integers(2, 5)), slab_sets=int(rng.choice([0, 2, 3, 4])),
                serpentine=int(rng.integers(0, 2)), m_resident=int(rng.integers(0, 2)))
    calls = [int(x) for x in rng.integers(1, 3 * T + 2, size=int(rng.integers(1, 4)))]
    u, up, m = E._fields(nx, ny, nz, 100 + case)
    gu, gup, _, _ = E._run_gpu(u, up, m, T, P, rates, store, calls, **opts)
    ou, oup = E._run_oracle(u, up, m, T, rates, calls)
    ok = np.array_equal(bits(gu), bits(ou)) and np.array_equal(bits(gup), bits(oup))
    if not ok:
        print("FAIL case", case, (nx, ny, nz, T, P, rates, store, opts, calls), flush=True)
        # isolate
        for key in ("slots", "slab_sets", "serpentine", "m_resident"):
            for val in ({"slots": [2, 3, 4], "slab_sets": [0, 3, 4], "serpentine": [0, 1], "m_resident": [0, 1]}[key]):
                o2 = dict(opts); o2[key] = val
                g2, gp2, _, _ = E._run_gpu(u, up, m, T, P, rates, store, calls, **o2)
                ok2 = np.array_equal(bits(g2), bits(ou)) and np.array_equal(bits(gp2), bits(oup))
                print("  ", key, val, "ok" if ok2 else "FAIL", flush=True)
        for st in (0, 1):
            g2, gp2, _, _ = E._run_gpu(u, up, m, T, P, rates, st, calls, **opts)
            print("   store", st, np.array_equal(bits(g2), bits(ou)) and np.array_equal(bits(gp2), bits(oup)))
        for c2 in ([sum(calls)], [calls[0]]):
            g2, gp2, _, _ = E._run_gpu(u, up, m, T, P, rates, store, c2, **opts)
            o2u, o2p = E._run_oracle(u, up, m, T, rates, c2)
            print("   calls", c2, np.array_equal(bits(g2), bits(o2u)) and np.array_equal(bits(gp2), bits(o2p)))
        bad = np.nonzero(bits(gu) != bits(ou)); print("   u mismatches", len(bad[0]), "planes", sorted(set(bad[0].tolist()))[:20])
        bad = np.nonzero(bits(gup) != bits(oup)); print("   up mismatches", len(bad[0]), "planes", sorted(set(bad[0].tolist()))[:20])
        break
print("done")
