"""Stress the stencil on a ragged geometry, alone and next to a concurrent
kernel on another stream, against the oracle."""
import os
import sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import oracle  # noqa: E402
from paper_2109_05410_b200 import oocz as Z  # noqa: E402
from paper_2109_05410_b200 import synth  # noqa: E402

for (nx, ny, nz, z0, z1, zv0, zv1) in ((40, 16, 36, 8, 28, 0, 28), (40, 16, 36, 4, 28, 0, 28),
                                        (136, 31, 40, 4, 36, 0, 40), (64, 16, 36, 8, 28, 0, 28)):
    u = synth.dense(nx, ny, nz, seed=3)
    up = (synth.dense(nx, ny, nz, seed=4) * np.float32(0.5)).astype(np.float32)
    m = synth.layered(nx, ny, nz)
    want = oracle.step(u[zv0:zv1], up[zv0:zv1], m[zv0:zv1])
    du, dm = torch.from_numpy(u).cuda(), torch.from_numpy(m).cuda()
    side = torch.cuda.Stream()
    big = torch.empty(64 << 20, device="cuda")
    ef = torch.from_numpy(synth.dense(512, 512, 64, seed=5)).cuda()
    ew = torch.empty(Z.oocz_zfp_bytes(512, 512, 64, 16) // 8, dtype=torch.int64, device="cuda")
    for mode in ("alone", "concurrent", "with_encode", "with_decode"):
        bad = 0
        for rep in range(300):
            dup = torch.from_numpy(up).cuda()
            torch.cuda.synchronize()
            if mode == "concurrent":
                with torch.cuda.stream(side):
                    for _ in range(3):
                        big.mul_(1.0001)
            if mode == "with_encode":
                for _ in range(2):
                    Z.oocz_zfp_encode(ef, 512, 512, 64, 16, ew, side)
            if mode == "with_decode":
                for _ in range(2):
                    Z.oocz_zfp_decode(ew, 512, 512, 64, 16, ef, side)
            Z.oocz_stencil_step_planes(du, dup, dm, nx, ny, nz, Z.default_coeffs(), z0, z1, zv0, zv1,
                                       torch.cuda.current_stream())
            torch.cuda.synchronize()
            got = dup.cpu().numpy()
            if not np.array_equal(got[z0:z1].view(np.uint32), want[z0 - zv0:z1 - zv0].view(np.uint32)):
                bad += 1
        print((nx, ny, nz, z0, z1), mode, "bad launches", bad, "of 300", flush=True)
