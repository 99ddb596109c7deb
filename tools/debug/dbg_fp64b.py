"""Debug: for mismatching fp64 stencil cells, find which value substituted for an
OOB (zero) y-neighbour would explain the difference, and where that value lives."""
import sys
import numpy as np
import torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import oracle
from paper_2109_05410_b200 import oocz as z
from test_gpu_fp64 import _state64

def dev(a): return torch.from_numpy(np.ascontiguousarray(a)).cuda()
c = oracle.C64
lib = sys.argv[1] if len(sys.argv) > 1 else ""
for (nx, ny, nz) in [(136, 10, 37), (136, 12, 24), (264, 20, 30)]:
    u, up, m = _state64(nx, ny, nz, 9)
    want = oracle.step_f64(u, up, m)
    shown = 0
    for r in range(30):
        du, dup, dm = dev(u), dev(up), dev(m)
        z.oocz_stencil_step_planes_f64(du, dup, dm, nx, ny, nz, z.default_coeffs64(), 0, nz, 0, nz, None)
        torch.cuda.synchronize()
        g = dup.cpu().numpy()
        bad = np.argwhere(g != want)
        if not len(bad):
            continue
        print((nx, ny, nz), "rep", r, "nbad", len(bad), "rows", sorted(set(bad[:, 1].tolist())),
              "planes", sorted(set(bad[:, 0].tolist())))
        for (zz, yy, xx) in bad[:3]:
            diff = g[zz, yy, xx] - want[zz, yy, xx]
            L = diff / m[zz, yy, xx]
            cands = []
            for d in range(1, 5):
                v = L / c[d]
                # search u for v (same x), relative 1e-6
                hit = np.argwhere(np.abs(u[:, :, xx] - v) <= 1e-6 * max(abs(v), 1e-30))
                cands.append((d, float(v), [tuple(map(int, h)) for h in hit[:3]]))
            print("   cell", (int(zz), int(yy), int(xx)), "diff %.3e" % diff, cands)
        shown += 1
        if shown >= 3:
            break
