"""Encode (rates 64, 3) on one stream next to a stencil on another, on disjoint
buffers shaped like the racing engine case; check both results each time."""
import os
import sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import oracle  # noqa: E402
from paper_2109_05410_b200 import oocz as Z  # noqa: E402
from paper_2109_05410_b200 import synth  # noqa: E402

nx, ny, L = 40, 16, 36
u = synth.dense(nx, ny, L, seed=3); up = (u * np.float32(0.7)).astype(np.float32); m = synth.layered(nx, ny, L)
want_st = oracle.step(u[0:28], up[0:28], m[0:28])
# two cone-limited steps as the engine runs them: step 1 on [4, 28) into up, step 2 on [8, 28) into u
u1 = up.copy(); u1[4:28] = want_st[4:28]
want2 = oracle.step(u1[0:28], u[0:28], m[0:28])
e_in = synth.dense(nx, ny, 20, seed=9)
want_e64 = oracle.zfp_encode(e_in, 64)
want_e3 = oracle.zfp_encode(e_in, 3)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
du, dm = torch.from_numpy(u).cuda(), torch.from_numpy(m).cuda()
de = torch.from_numpy(e_in).cuda()
w64 = torch.empty(Z.oocz_zfp_bytes(nx, ny, 20, 64) // 8, dtype=torch.int64, device="cuda")
w3 = torch.empty(Z.oocz_zfp_bytes(nx, ny, 20, 3) // 8, dtype=torch.int64, device="cuda")
bad_s = bad_e = 0
for rep in range(2000):
    dup = torch.from_numpy(up).cuda()
    du2 = du.clone()
    w64.zero_(); w3.zero_()
    torch.cuda.synchronize()
    Z.oocz_zfp_encode(de, nx, ny, 20, 64, w64, s1)
    Z.oocz_zfp_encode(de, nx, ny, 20, 3, w3, s1)
    Z.oocz_stencil_step_planes(du2, dup, dm, nx, ny, L, Z.default_coeffs(), 4, 28, 0, 28, s2)
    Z.oocz_stencil_step_planes(dup, du2, dm, nx, ny, L, Z.default_coeffs(), 8, 28, 0, 28, s2)
    torch.cuda.synchronize()
    got = dup.cpu().numpy(); got2 = du2.cpu().numpy()
    if not (np.array_equal(got[4:28].view(np.uint32), want_st[4:28].view(np.uint32)) and
            np.array_equal(got2[8:28].view(np.uint32), want2[8:28].view(np.uint32))):
        bad_s += 1
    if not (np.array_equal(w64.cpu().numpy().view(np.uint64), want_e64) and
            np.array_equal(w3.cpu().numpy().view(np.uint64), want_e3)):
        bad_e += 1
print("bad stencil", bad_s, "bad encode", bad_e, "of 2000", flush=True)
