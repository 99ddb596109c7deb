"""Feasibility probe for on-chip (L2) temporal blocking:
the same stencil launch on a slab that stays resident in the 126 MB L2
(warm, no flush) vs the same slab after an L2 flush (cold).  The warm time is
what a step fed from L2 could run at, i.e. the ceiling of fusing steps through
L2."""
import os
import sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2109_05410_b200 import oocz as Z  # noqa: E402
from paper_2109_05410_b200 import synth  # noqa: E402

s = torch.cuda.current_stream()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for (nx, ny, planes) in ((512, 512, 24), (512, 512, 32), (256, 512, 48), (512, 512, 160)):
    u = torch.from_numpy(synth.dense(nx, ny, planes, seed=1)).cuda()
    m = torch.from_numpy(synth.layered(nx, ny, planes)).cuda()
    up = u.clone()
    res = {}
    for mode in ("cold", "warm"):
        ts = []
        for _ in range(30):
            if mode == "cold":
                flush.zero_()
            else:   # touch the three fields so they are L2-resident
                Z.oocz_stencil_step_planes(u, up, m, nx, ny, planes, Z.default_coeffs(), 4, planes - 4, 0, planes, s)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            Z.oocz_stencil_step_planes(u, up, m, nx, ny, planes, Z.default_coeffs(), 4, planes - 4, 0, planes, s)
            b.record(s)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ts.sort()
        cells = nx * ny * (planes - 8)
        res[mode] = ts[len(ts) // 2]
        print(f"{nx}x{ny}x{planes} ({3 * nx * ny * planes * 4 / 2**20:.0f} MiB) {mode}: {res[mode] * 1e3:.1f} us, "
              f"{cells / res[mode] / 1e6:.0f} G cell-updates/s, {16 * cells / res[mode] / 1e6:.0f} GB/s algorithmic",
              flush=True)
    print(f"   warm/cold = {res['warm'] / res['cold']:.3f}")
