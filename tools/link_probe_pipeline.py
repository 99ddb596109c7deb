"""Why the pipeline's copies run below the 1 GiB probe on some boxes: H2D and
D2H at once out of / into a large pinned arena at scattered offsets (like the
store), with one stream per direction vs two, and with a stencil kernel
streaming HBM on a third stream meanwhile.

  python tools/link_probe_pipeline.py [arena_GB]
"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2109_05410_b200 import oocz as Z  # noqa: E402
from paper_2109_05410_b200 import synth  # noqa: E402
from cuda.bindings import runtime as rt  # noqa: E402

GB = float(sys.argv[1]) if len(sys.argv) > 1 else 96.0
nbytes = int(GB * 1e9) // (2 << 20) * (2 << 20)
chunk = 2 << 30
H2D, D2H = rt.cudaMemcpyKind.cudaMemcpyHostToDevice, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost
arena = Z.oocz_host_alloc(nbytes)
dev = torch.empty(2 * chunk, dtype=torch.uint8, device="cuda")
streams = [torch.cuda.Stream() for _ in range(4)]
n = 4096
u = synth.dense_torch(n, n, 1536, 2, 0, 40)
m = synth.layered_torch(n, n, 1536, 0, 40)
up = u.clone()
ks = torch.cuda.Stream()
offs = [int(i * (nbytes // 2 - chunk) / 5) // 4096 * 4096 for i in range(6)]


d2d_a = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
d2d_b = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")


def run(per_dir: int, kernels: bool, d2d: bool = False):
    rates = []
    for off in offs:
        torch.cuda.synchronize()
        if d2d:                  # device-to-device copies on the copy engines meanwhile
            with torch.cuda.stream(ks):
                for _ in range(40):
                    d2d_b.copy_(d2d_a, non_blocking=True)
        if kernels:
            with torch.cuda.stream(ks):
                for _ in range(6):
                    Z.oocz_stencil_step_planes(u, up, m, n, n, 40, Z.default_coeffs(), 4, 36, 0, 40, ks)
        ev0 = torch.cuda.Event(enable_timing=True)
        ev0.record(streams[0])
        for s in streams:
            s.wait_event(ev0)
        part = chunk // per_dir
        for i in range(per_dir):
            sh, sd = streams[i], streams[2 + i] if per_dir == 2 else streams[1]
            rt.cudaMemcpyAsync(dev.data_ptr() + i * part, arena + off + i * part, part, H2D, sh.cuda_stream)
            rt.cudaMemcpyAsync(arena + nbytes // 2 + off + i * part, dev.data_ptr() + chunk + i * part, part, D2H,
                               sd.cuda_stream)
        ends = []
        for s in streams[:2 * per_dir] if per_dir == 2 else streams[:2]:
            e = torch.cuda.Event(enable_timing=True)
            e.record(s)
            ends.append(e)
        torch.cuda.synchronize()
        ms = max(ev0.elapsed_time(e) for e in ends)
        rates.append(chunk / (ms / 1e3) / 1e9)
    return round(sum(rates) / len(rates), 2)


out = {"arena_GB": GB}
for per_dir in (1, 2):
    for kern in (False, True):
        out[f"streams_per_dir={per_dir} kernels={kern}"] = run(per_dir, kern)
out["streams_per_dir=1 d2d copies"] = run(1, False, True)
Z.oocz_host_free(arena)
print(json.dumps(out))
