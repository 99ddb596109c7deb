#!/usr/bin/env python3
"""C5 precision sweep (BASELINE.json configs[4]; Fig. 7).

1024^3 fp32, PULSE(sigma 8) wavefield with u- = u, LAYERED m, T = 4, P = 128.
One context per rate (8, 12, 16, 24 on all three fields) plus the uncompressed
one, stepped together to 4,320 steps; every 480 steps (the paper's step grid,
PAPER.md:217) each compressed u^t is compared with the uncompressed u^t:
normwise max|a-b|/max|b| and the paper's mean point-wise |a-b|/|b| over 100
seeded points per plane (102,400 points; |b| < 1e-30 skipped, counted).

The stores are kept in HBM (same results bit for bit as the host store: the
out-of-core schedule does not change the arithmetic, tests/test_gpu_engine.py).
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2109_05410_b200 import oocz as Z  # noqa: E402
from paper_2109_05410_b200 import synth  # noqa: E402
import bench  # noqa: E402  (rel_errors)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--steps", type=int, default=4320)
    ap.add_argument("--every", type=int, default=480)
    ap.add_argument("--rates", default="8,12,16,24")
    ap.add_argument("--out", default="gpurun_out/drift_c5.json")
    args = ap.parse_args()
    n = args.n
    rates = [int(r) for r in args.rates.split(",")]
    t0 = time.time()
    u = synth.pulse(n, n, n, sigma=8.0)
    m = synth.layered(n, n, n)
    ctxs = {}
    for r in [0] + rates:
        cfg = Z.oocz_default_config(n, n, n, tb=4, block_planes=128, rate=[r] * 3, store=Z.OOCZ_STORE_DEVICE)
        c = Z.oocz_create(cfg)
        for f, a in ((Z.OOCZ_U, u), (Z.OOCZ_UPREV, u), (Z.OOCZ_M, m)):
            Z.oocz_set_field(c, f, a)
        ctxs[r] = c
    del u, m
    rows = []
    done = 0
    buf_ref = np.empty((n, n, n), np.float32)
    buf = np.empty((n, n, n), np.float32)
    while done < args.steps:
        k = min(args.every, args.steps - done)
        times = {}
        for r, c in ctxs.items():
            Z.oocz_step(c, k)
            times[r] = Z.oocz_get_stats(c)["last_step_device_ms"]
        done += k
        Z.oocz_get_field(ctxs[0], Z.OOCZ_U, buf_ref)
        row = {"steps": done, "ref_max_abs": float(np.abs(buf_ref).max())}
        for r in rates:
            Z.oocz_get_field(ctxs[r], Z.OOCZ_U, buf)
            e = bench.rel_errors(buf, buf_ref)
            row[f"r{r}"] = {"normwise_max": e["normwise_max"], "mean_pointwise": e["mean_pointwise"],
                            "skipped": e["skipped"], "mean_pointwise_significant": e["mean_pointwise_significant"],
                            "significant_points": e["significant_points"],
                            "cell_updates_per_s": n ** 3 * k / (times[r] / 1e3)}
        row["raw_cell_updates_per_s"] = n ** 3 * k / (times[0] / 1e3)
        rows.append(row)
        print(json.dumps(row), flush=True)
    for c in ctxs.values():
        Z.oocz_destroy(c)
    res = {"config": f"C5: {n}^3 fp32, PULSE(8) + LAYERED, T=4, P=128, rates {rates} vs uncompressed",
           "points_per_plane": 100, "rows": rows, "wall_s": round(time.time() - t0, 1),
           "paper_context": "mean point-wise rel. error between 1e-6 and 1e-7 after 4,320 steps, fp64, "
                            "rate 24/64 (PAPER.md:247)"}
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    with open(args.out, "w") as fh:
        json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main()
