"""Block height P at C2 (512^3, T = 4, rate 16, headline schedules): value (store
in HBM) and e2e (host store), alternating, best of 2 each.  Smaller P means more
blocks per call (shorter pipeline fill / drain on the host link) but a larger
stencil cone per block ((P + 2h - 8s) planes per step s)."""
import json
import os
import sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2109_05410_b200 import oocz as Z  # noqa: E402

torch.cuda.set_device(0)
fields = bench.make_fields_c2()
cells = bench.NX * bench.NY * bench.NZ * bench.T * 10
ps = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "64,128,256").split(",")]
res = {}
for rep in range(2):
    for p in ps:
        for label, store, opt in (("value", 1, dict(m_resident=1)),
                                  ("e2e", 0, dict(serpentine=1, m_resident=1, slots=3))):
            dev_s, st, evs, launches, ctx = bench.run_mode_c2(Z, store, (16,) * 3, fields, 0, 10, 3, 0,
                                                          block_planes=p, **opt)
            Z.oocz_destroy(ctx)
            key = f"P{p}_{label}"
            res[key] = max(res.get(key, 0.0), round(cells / dev_s / 1e9, 1))
print(json.dumps(res), flush=True)
