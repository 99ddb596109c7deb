"""Find the first call / sweep where the racing configuration diverges."""
import os
import sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "tests"))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import oracle  # noqa: E402
import test_gpu_engine as E  # noqa: E402
from gpu_util import Z, bits  # noqa: E402

z = Z()
nx, ny, nz, T, P, rates = 40, 16, 80, 2, 20, (64, 3, 12)
u, up, m = E._fields(nx, ny, nz, 152)
for store in (1, 0):
    for calls in ([2] * 8, [1] * 8, [3] * 6, [4, 7]):
        first = {}
        for rep in range(15):
            cfg = z.oocz_default_config(nx, ny, nz, tb=T, block_planes=P, rate=list(rates), store=store, slots=4)
            a = oracle.roundtrip(u, rates[0]); b = oracle.roundtrip(up, rates[1]); mm = oracle.roundtrip(m, rates[2])
            with z.Stepper(cfg) as s:
                s.set(u, up, m)
                for k, n in enumerate(calls):
                    s.step(n)
                    a, b = oracle.advance(a, b, mm, T, rates, n)
                    gu, gup = s.get(z.OOCZ_U), s.get(z.OOCZ_UPREV)
                    if not (np.array_equal(bits(gu), bits(a)) and np.array_equal(bits(gup), bits(b))):
                        bu = sorted(set(np.nonzero(bits(gu) != bits(a))[0].tolist()))
                        bp = sorted(set(np.nonzero(bits(gup) != bits(b))[0].tolist()))
                        key = (k, tuple(bu[:1] + bu[-1:]), tuple(bp[:1] + bp[-1:]))
                        first[key] = first.get(key, 0) + 1
                        break
        print("store", store, "calls", calls, "first divergences (call, u planes, u- planes): count", first, flush=True)
