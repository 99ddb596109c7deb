"""Time the isolated fp32 / fp64 stencil (one C2 slab, L2 flushed, CUDA events)."""
import os
import sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2109_05410_b200 import oocz as Z, synth  # noqa: E402

n, planes = 512, 160
u = torch.from_numpy(synth.dense(n, n, n, seed=1, z0=0, z1=planes)).cuda()
m = torch.from_numpy(synth.layered(n, n, n, z0=0, z1=planes)).cuda()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream()
upd = n * n * (planes - 8)
for name, uu, mm, fn, c, b in (("f32", u, m, Z.oocz_stencil_step_planes, Z.default_coeffs(), 16),
                               ("f64", u.double(), m.double(), Z.oocz_stencil_step_planes_f64, Z.default_coeffs64(), 32)):
    up = uu.clone()
    ts = []
    for _ in range(15):
        flush.zero_()
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn(uu, up, mm, n, n, planes, c, 4, planes - 4, 0, planes, s)
        e.record(s)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(e))
    t = sorted(ts)[len(ts) // 2] / 1e3
    print(name, "ms %.4f" % (t * 1e3), "GB/s %.0f" % (b * upd / t / 1e9))
