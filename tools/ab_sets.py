"""value (store in HBM) and e2e (pinned host store) vs slab sets and staging
slots, headline schedule (serpentine + m resident), C2 at rate 16 and raw."""
import os
import sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2109_05410_b200 import oocz as Z  # noqa: E402

torch.cuda.set_device(0)
fields = bench.make_fields_c2()
cells = bench.NX * bench.NY * bench.NZ * bench.T * 10
for rates in ((16, 16, 16), (0, 0, 0)):
    for store in (1, 0):
        for sets in (2, 3, 4):
            for slots in ((2, 3) if store == 0 else (2,)):
                dev_s, st, evs, launches, ctx = bench.run_mode_c2(Z, store, rates, fields, 0, 10, 3, 0, m_resident=1, serpentine=1, slots=slots,
                                                              slab_sets=sets)
                Z.oocz_destroy(ctx)
                print(f"rates={rates[0]} store={'dev' if store else 'host'} sets={sets} slots={slots}: "
                      f"{cells / dev_s / 1e9:.1f} G cell-updates/s", flush=True)
