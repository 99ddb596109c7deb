"""Launch each hot kernel on the C2 workload a few times (for ncu captures)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2109_05410_b200 import oocz as Z  # noqa: E402
from paper_2109_05410_b200 import synth  # noqa: E402

n = int(os.environ.get("N", "512"))                # 4096: a C3 plane (DENSE(2), generated on the GPU)
planes = int(os.environ.get("PLANES", "160"))      # one slab: P + 2h
rate = int(os.environ.get("RATE", "16"))
if n == 512:
    u = torch.from_numpy(synth.dense(n, n, n, seed=1, z0=0, z1=planes)).cuda()
    m = torch.from_numpy(synth.layered(n, n, n, z0=0, z1=planes)).cuda()
else:
    u = synth.dense_torch(n, n, 1536, 2, 0, planes)
    m = synth.layered_torch(n, n, 1536, 0, planes)
up = u.clone()
words = torch.empty(Z.oocz_zfp_bytes(n, n, planes, rate) // 8, dtype=torch.int64, device="cuda")
out = torch.empty_like(u)
s = torch.cuda.current_stream()
for _ in range(int(os.environ.get("REPS", "3"))):
    Z.oocz_zfp_encode(u, n, n, planes, rate, words, s)
    Z.oocz_zfp_decode(words, n, n, planes, rate, out, s)
    Z.oocz_stencil_step_planes(u, up, m, n, n, planes, Z.default_coeffs(), 4, planes - 4, 0, planes, s)
torch.cuda.synchronize()
print("done")

if os.environ.get("F64", "0") == "1":
    r64 = int(os.environ.get("RATE64", "32"))
    u64, m64 = u.double(), m.double()
    up64, out64 = u64.clone(), torch.empty_like(u64)
    w64 = torch.empty(Z.oocz_zfp_bytes(n, n, planes, r64) // 8, dtype=torch.int64, device="cuda")
    for _ in range(int(os.environ.get("REPS", "3"))):
        Z.oocz_zfp_encode_f64(u64, n, n, planes, r64, w64, s)
        Z.oocz_zfp_decode_f64(w64, n, n, planes, r64, out64, s)
        Z.oocz_stencil_step_planes_f64(u64, up64, m64, n, n, planes, Z.default_coeffs64(), 4, planes - 4, 0,
                                       planes, s)
    torch.cuda.synchronize()
    print("done f64")
