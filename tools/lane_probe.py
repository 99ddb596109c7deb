"""Per-kernel device time inside the pipelined sweep (profile = 1 events on the
library's streams) for one schedule, next to the same kernels alone on a
slab of the same shape: which kernel slows down when they share the GPU.

  OOCZ_LIB=... python tools/lane_probe.py [c3hbm|c2hbm]
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2109_05410_b200 import oocz as Z  # noqa: E402
from paper_2109_05410_b200 import synth  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "c3hbm"
torch.cuda.set_device(0)
if which == "c3hbm":
    nx, nz, P = 4096, 1536, 96
    r = bench.run_c3(Z, which, nx, nx, nz, (16,) * 3, {"P": P, "store": 1, "slab_sets": 1}, None, 0, 1, None, 0,
                     2, 2, None, profile=1)
    evs = r["evs"]
    cells = nx * nx * nz * 4 * 2
    dev_s = r["device_s"]
else:
    fields = bench.make_fields_c2()
    dev_s, st, evs, launches, ctx = bench.run_mode_c2(Z, 1, (16,) * 3, fields, 0, 4, 3, 1, m_resident=1)
    Z.oocz_destroy(ctx)
    nx, P = 512, 128
    cells = 512 ** 3 * 4 * 4
table = bench.kernel_table(evs)
out = {"schedule": which, "G_cell_updates_per_s": round(cells / dev_s / 1e9, 1), "span_ms": round(dev_s * 1e3, 1),
       "in_pipeline": {k: {"ms": round(v[0], 1), "launches": v[2], "avg_ms": round(v[0] / v[2], 3)} for k, v in table.items()},
       "lanes": bench.lanes_summary(evs)}
# the same kernels alone: one block's slab (P + 2h planes), L2 flushed between
planes = P + 32
if which == "c3hbm":
    u = synth.dense_torch(nx, nx, 1536, 2, 0, planes)
    m = synth.layered_torch(nx, nx, 1536, 0, planes)
else:
    u = torch.from_numpy(np.ascontiguousarray(fields[0][:planes])).cuda()
    m = torch.from_numpy(np.ascontiguousarray(fields[2][:planes])).cuda()
up = u.clone()
dec = torch.empty_like(u)
words = torch.empty(Z.oocz_zfp_bytes(nx, nx, planes, 16) // 8, dtype=torch.int64, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream()


def med(fn, reps=5):
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn()
        b.record(s)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts) // 2]


own = P                                  # the encoder codes the own planes; the decoder the read unit
out["alone_per_launch_ms"] = {
    "encode": round(med(lambda: Z.oocz_zfp_encode(u, nx, nx, own, 16, words, s)), 3),
    "decode": round(med(lambda: Z.oocz_zfp_decode(words, nx, nx, own, 16, dec, s)), 3),
    "stencil": round(med(lambda: Z.oocz_stencil_step_planes(u, up, m, nx, nx, planes, Z.default_coeffs(), 16,
                                                            16 + P, 0, planes, s)), 3),
}
print(json.dumps(out), flush=True)
