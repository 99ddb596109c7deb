"""C2 value path (bench.run_mode_c2, store in HBM, m resident): eager vs graphs,
alternating, 4 rounds."""
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
res = {"eager": [], "graph": []}
for _ in range(4):
    for g in (0, 1):
        dev_s, st, evs, launches, ctx = bench.run_mode_c2(Z, 1, (16,) * 3, fields, 0, 10, 3, 0,
                                                      m_resident=1, graphs=g)
        Z.oocz_destroy(ctx)
        res["graph" if g else "eager"].append(round(cells / dev_s / 1e9, 1))
print(json.dumps(res), flush=True)
