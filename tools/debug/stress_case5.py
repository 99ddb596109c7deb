"""In a racing run, which stored words differ from the oracle's stream?"""
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
shown = 0
for rep in range(60):
    cfg = z.oocz_default_config(nx, ny, nz, tb=T, block_planes=P, rate=list(rates), store=1, slots=2)
    a = oracle.roundtrip(u, rates[0]); b = oracle.roundtrip(up, rates[1]); mm = oracle.roundtrip(m, rates[2])
    with z.Stepper(cfg) as s:
        s.set(u, up, m)
        for k in range(4):
            s.step(2)
            a_prev = a
            a, b = oracle.advance(a, b, mm, T, rates, 2)
            st = z.oocz_save_store(s.ctx, 0).view(np.uint64)
            # the oracle's stream of u: advance() ends with the round trip, so encode its pre-RT field
            # by re-running the last sweep without the round trip is not available; compare decoded instead
            gu = s.get(z.OOCZ_U)
            if not np.array_equal(bits(gu), bits(a)):
                want = oracle.zfp_encode(a, rates[0])      # a is RT'd: re-encoding an RT'd field is not
                # idempotent in general, so compare per 4^3 block which blocks decode differently
                nb = (nx // 4) * (ny // 4) * (nz // 4)
                ga = gu.reshape(nz // 4, 4, ny // 4, 4, nx // 4, 4).transpose(0, 2, 4, 1, 3, 5).reshape(nb, 64)
                oa = a.reshape(nz // 4, 4, ny // 4, 4, nx // 4, 4).transpose(0, 2, 4, 1, 3, 5).reshape(nb, 64)
                badb = np.nonzero((bits(ga) != bits(oa)).any(1))[0]
                print("rep", rep, "call", k, "bad blocks", badb.tolist()[:40], "of", nb,
                      "values per bad block", [(int((bits(ga[i]) != bits(oa[i])).sum())) for i in badb[:10]], flush=True)
                rate = rates[0]
                for bblk in badb[:3]:
                    w = st[bblk * rate:(bblk + 1) * rate]
                    print("   block", int(bblk), "stored words[0:3]", [hex(int(x)) for x in w[:3]], flush=True)
                shown += 1
                break
    if shown >= 4:
        break
print("done")
