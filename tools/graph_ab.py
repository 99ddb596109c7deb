"""Eager vs CUDA-graph sweeps (cfg.graphs) with the store in HBM: C1 (64^3, 2
z-blocks, T = 2, rate 16, BASELINE configs[0]) and other sizes; device time per
sweep from the library's events, best of 3 calls of 20 sweeps after a warm-up
call (which also captures the graph)."""
import json
import os
import sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2109_05410_b200 import oocz as Z  # noqa: E402
from paper_2109_05410_b200 import synth  # noqa: E402

torch.cuda.set_device(0)
res = {}
for (n, P, T) in ((64, 32, 2), (128, 32, 4), (256, 64, 4), (512, 128, 4)):
    u = synth.dense(n, n, n, seed=1)
    m = synth.layered(n, n, n)
    for graphs in (0, 1):
        cfg = Z.oocz_default_config(n, n, n, tb=T, block_planes=P, rate=[16] * 3, store=1, graphs=graphs,
                                    m_resident=1)
        ctx = Z.oocz_create(cfg)
        try:
            for f, a in ((Z.OOCZ_U, u), (Z.OOCZ_UPREV, u), (Z.OOCZ_M, m)):
                Z.oocz_set_field(ctx, f, a)
            Z.oocz_step(ctx, 20 * T)
            best = 1e30
            for _ in range(3):
                Z.oocz_step(ctx, 20 * T)
                best = min(best, Z.oocz_get_stats(ctx)["last_step_device_ms"] / 20)
        finally:
            Z.oocz_destroy(ctx)
        key = f"{n}^3 P{P} T{T} {'graph' if graphs else 'eager'}"
        res[key] = {"us_per_sweep": round(best * 1e3, 1), "G_cell_updates_per_s": round(n ** 3 * T / (best / 1e3) / 1e9, 2)}
        print(key, res[key], flush=True)
print(json.dumps(res))
