"""Share of the value path's device time per stage and lane (profile = 1, C2, store in
HBM, m resident, 10 sweeps): how much the C_i and parallelogram strip copies cost."""
import collections
import os
import sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2109_05410_b200 import oocz as Z  # noqa: E402

torch.cuda.set_device(0)
fields = bench.make_fields_c2()
dev_s, st, evs, launches, ctx = bench.run_mode_c2(Z, 1, (16,) * 3, fields, 0, 10, 3, 1, m_resident=1)
Z.oocz_destroy(ctx)
lanes = {0: "h2d", 1: "compute", 2: "d2h", 3: "comm", 4: "decode", 5: "encode"}
agg = collections.Counter()
for e in evs:
    agg[(Z.STAGES.get(e["stage"], e["stage"]), lanes.get(e["lane"], e["lane"]))] += e["end_ms"] - e["start_ms"]
print("span ms %.2f" % (dev_s * 1e3))
for k, v in sorted(agg.items(), key=lambda t: -t[1]):
    print("%-22s %8.2f ms" % ("/".join(k), v))
