"""C3 headline schedule (serpentine + m resident) out of core vs staging slots:
more slots keep more recently encoded blocks' rows on the device across a
serpentine turn, so fewer read units cross H2D (R22)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2109_05410_b200 import oocz as Z  # noqa: E402

torch.cuda.set_device(0)
nx = ny = bench.C3N
nz = bench.C3Z
cfg16 = Z.oocz_default_config(nx, ny, nz, tb=bench.T, block_planes=64, rate=[16] * 3)
need = Z.oocz_host_store_bytes(cfg16, 1)
arena_p = Z.oocz_host_alloc(need)
try:
    for slots in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "3,4,5,6").split(",")]:
        try:
            mode = sys.argv[2] if len(sys.argv) > 2 else "mres"
            opt = (dict(P=64, serpentine=1, m_hbm=1, slots=slots, gen_chunk=4) if mode == "mhbm" else
                   dict(P=64, serpentine=1, m_hbm=1, slots=slots, gen_chunk=4, slab_sets=1) if mode == "mhbm1" else
                   dict(P=64, serpentine=1, m_resident=1, slots=slots, gen_chunk=4 if slots >= 5 else 16))
            r = bench.run_c3(Z, f"slots{slots}_{mode}", nx, ny, nz, (16,) * 3, opt, (arena_p, need), 0, 1, None, 0,
                             4, 2, None)
            print(json.dumps({"slots": slots, "mode": mode, "G": round(r["cups"] / 1e9, 2), "h2d_GB": round(r["h2d_per_sweep"] / 1e9, 2),
                              "d2h_GB": round(r["d2h_per_sweep"] / 1e9, 2), "h2d_GBps": round(r["h2d_GBps"], 2),
                              "d2h_GBps": round(r["d2h_GBps"], 2), "device_GB": round(r["device_bytes"] / 1e9, 1)}),
                  flush=True)
        except Exception as e:
            print(json.dumps({"slots": slots, "error": str(e)[:200]}), flush=True)
finally:
    Z.oocz_host_free(arena_p)
