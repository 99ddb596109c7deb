"""Profile the racing configuration: does any encode start before its own
block's stencil ends, or any stencil start before the previous encode of its
slab set ends?"""
import os
import sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "tests"))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import test_gpu_engine as E  # noqa: E402
from gpu_util import bits  # noqa: E402

nx, ny, nz, T, P, rates = 40, 16, 80, 2, 20, (64, 3, 12)
u, up, m = E._fields(nx, ny, nz, 152)
calls = [4, 7]
ou, oup = E._run_oracle(u, up, m, T, rates, calls)
for rep in range(30):
    gu, gup, st, evs = E._run_gpu(u, up, m, T, P, rates, 0, calls, slots=4, profile=1)
    ok = np.array_equal(bits(gu), bits(ou))
    by = {}
    for e in evs:
        by.setdefault((e["sweep"], e["block"]), {}).setdefault(e["stage"], []).append(e)
    viol = []
    for key, stg in by.items():
        if 2 in stg and 3 in stg:
            s_end = max(x["end_ms"] for x in stg[2]); e_start = min(x["start_ms"] for x in stg[3])
            if e_start < s_end - 1e-4:
                viol.append(("enc-before-stencil-end", key, round(s_end - e_start, 4)))
        if 1 in stg and 2 in stg:
            d_end = max(x["end_ms"] for x in stg[1]); s_start = min(x["start_ms"] for x in stg[2])
            if s_start < d_end - 1e-4:
                viol.append(("stencil-before-decode-end", key, round(d_end - s_start, 4)))
    # global block order (sweep-major) and cross-block reuse of slab sets (2) and slots (4)
    order = sorted(by)
    span = lambda stg, k, f: (f(x["start_ms"] for x in stg[k]), f(x["end_ms"] for x in stg[k]))
    for a in range(len(order)):
        sa = by[order[a]]
        for b2 in range(a + 1, min(a + 5, len(order))):
            sb = by[order[b2]]
            d = b2 - a
            if d % 2 == 0 and 3 in sa:          # same slab set: decode(b) after encode(a)
                enc_end = max(x["end_ms"] for x in sa[3])
                for st_ in (1, 6, 2):
                    if st_ in sb:
                        st_start = min(x["start_ms"] for x in sb[st_])
                        if st_start < enc_end - 1e-4:
                            viol.append(("set-reuse", order[a], order[b2], st_, round(enc_end - st_start, 4)))
    print("rep", rep, "ok" if ok else "MISMATCH", viol[:6], flush=True)
