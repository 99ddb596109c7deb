"""CUDA-event timing of each hot kernel on one C2 slab (P + 2h = 160 planes of 512^2)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2109_05410_b200 import oocz as Z  # noqa: E402
from paper_2109_05410_b200 import synth  # noqa: E402

n, planes = 512, int(os.environ.get("PLANES", "160"))
res = {}
u = torch.from_numpy(synth.dense(n, n, n, seed=1, z0=0, z1=planes)).cuda()
m = torch.from_numpy(synth.layered(n, n, n, z0=0, z1=planes)).cuda()
up = u.clone()
out = torch.empty_like(u)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream()
cells = n * n * planes


def timeit(fn, reps=20):
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn()
        b.record(s)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


for rate in (8, 16, 24):
    words = torch.empty(Z.oocz_zfp_bytes(n, n, planes, rate) // 8, dtype=torch.int64, device="cuda")
    te = timeit(lambda: Z.oocz_zfp_encode(u, n, n, planes, rate, words, s))
    td = timeit(lambda: Z.oocz_zfp_decode(words, n, n, planes, rate, out, s))
    cb = cells // 64 * 8 * rate
    res[f"encode_r{rate}"] = {"ms": te, "Gvalues/s": cells / te / 1e6, "alg_GB/s": (4 * cells + cb) / te / 1e6}
    res[f"decode_r{rate}"] = {"ms": td, "Gvalues/s": cells / td / 1e6, "alg_GB/s": (4 * cells + cb) / td / 1e6}
upd = n * n * (planes - 8)
tsn = timeit(lambda: Z.oocz_stencil_step_planes(u, up, m, n, n, planes, Z.default_coeffs(), 4, planes - 4, 0,
                                                planes, s))
res["stencil"] = {"ms": tsn, "Gcells/s": upd / tsn / 1e6, "alg_GB/s": 16 * upd / tsn / 1e6}
print(json.dumps(res, indent=1))
