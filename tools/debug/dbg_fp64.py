"""Debug: repeat the fp64 stencil vs the oracle and print where mismatches sit."""
import collections
import sys
import numpy as np
import torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import oracle
from paper_2109_05410_b200 import oocz as z
from test_gpu_fp64 import _state64

def dev(a): return torch.from_numpy(np.ascontiguousarray(a)).cuda()
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
for (nx, ny, nz, n) in [(136, 10, 37, 1), (136, 12, 24, 1), (264, 20, 30, 1), (64, 64, 64, 1)]:
    u, up, m = _state64(nx, ny, nz, 9)
    want = oracle.step_f64(u, up, m)
    nbad = 0
    where = collections.Counter()
    for r in range(reps):
        du, dup, dm = dev(u), dev(up), dev(m)
        z.oocz_stencil_steps_f64(du, dup, dm, nx, ny, nz, z.default_coeffs64(), n, torch.cuda.current_stream())
        torch.cuda.synchronize()
        g = du.cpu().numpy()
        bad = np.argwhere(g != want)
        if len(bad):
            nbad += 1
            for (zz, yy, xx) in bad[:200]:
                where[(int(zz), int(yy), int(xx) // 4 * 4)] += 1
            if nbad <= 2:
                k = tuple(bad[0])
                print("   rep", r, "nbad", len(bad), "first", k, "got %r want %r up %r u %r" % (g[k], want[k], up[k], u[k]))
    print((nx, ny, nz), "failing reps", nbad, "/", reps, "top cells", where.most_common(8))
