"""e2e of the out-of-core path vs staging slots and schedule (C2, rate 16)."""
import os
import sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2109_05410_b200 import oocz as Z  # noqa: E402

torch.cuda.set_device(0)
fields = bench.make_fields_c2()
cells = bench.NX * bench.NY * bench.NZ * bench.T * 10
for serp, mres in ((0, 0), (1, 0), (0, 1), (1, 1)):
    for slots in (2, 3, 4):
        dev_s, st, evs, launches, ctx = bench.run_mode_c2(Z, 0, (16, 16, 16), fields, 0, 10, 3, 0,
                                                      m_resident=mres, serpentine=serp, slots=slots)
        Z.oocz_destroy(ctx)
        sw = st["sweeps"]
        print(f"serp={serp} mres={mres} slots={slots}: e2e {cells / dev_s / 1e9:.1f} G  "
              f"h2d {st['h2d_bytes'] / sw / 1e6:.0f} MB d2h {st['d2h_bytes'] / sw / 1e6:.0f} MB per sweep, "
              f"{st['h2d_bytes'] / dev_s / 1e9:.1f} / {st['d2h_bytes'] / dev_s / 1e9:.1f} GB/s", flush=True)
