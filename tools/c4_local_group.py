"""C4's z-partitioned protocol at C3 scale on ONE GPU: the 4096 x 4096 x 1536
grid split over `world` in-process contexts (the local group: the same
compressed-halo protocol as NCCL, with device copies), each rank streaming its
own slab out of core from its own pinned store; the result compared bit for bit
with world = 1 on sampled planes (a partitioned run equals world = 1 because the
halos are the round-tripped bytes a single GPU would decode).  Throughput here
is not C4's (the ranks share one GPU and one host link).

  python tools/c4_local_group.py [--world 2] [--sweeps 2]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2109_05410_b200 import oocz as Z  # noqa: E402
from paper_2109_05410_b200 import synth  # noqa: E402


def run(world, args, planes):
    n, nz = 4096, 1536
    # (m streamed: two ranks' resident m would not fit one GPU's HBM)
    cfg = Z.oocz_default_config(n, n, nz, tb=4, block_planes=args.P, rate=[16] * 3, serpentine=1, slots=2,
                                slab_sets=args.sets if world > 1 else 0)
    S = nz // world
    ctxs = Z.oocz_create_local_group(cfg, world) if world > 1 else [Z.oocz_create(cfg)]
    try:
        for r, c in enumerate(ctxs):
            for z0 in range(0, S, 16):
                d = synth.dense_torch(n, n, nz, 2, r * S + z0, r * S + z0 + 16)
                Z.oocz_set_field_planes(c, Z.OOCZ_U, z0, d)
                Z.oocz_set_field_planes(c, Z.OOCZ_UPREV, z0, d)
                del d
                Z.oocz_set_field_planes(c, Z.OOCZ_M, z0, synth.layered_torch(n, n, nz, r * S + z0, r * S + z0 + 16))
        torch.cuda.synchronize()
        step = (lambda k: Z.oocz_step_local_group(ctxs, k)) if world > 1 else (lambda k: Z.oocz_step(ctxs[0], k))
        t0 = time.perf_counter()
        step(4 * args.sweeps)
        host_s = time.perf_counter() - t0
        st = [Z.oocz_get_stats(c) for c in ctxs]
        got = []
        for zg in planes:                      # global planes -> (rank, local plane)
            r, zl = zg // S, zg % S
            got.append(Z.oocz_get_field_planes(ctxs[r], Z.OOCZ_U, zl, np.empty((4, n, n), np.float32)))
        return {"world": world, "host_s": round(host_s, 2),
                "halo_bytes": int(sum(s["halo_bytes"] for s in st)),
                "h2d_bytes": int(sum(s["h2d_bytes"] for s in st))}, np.concatenate(got)
    finally:
        for c in ctxs:
            Z.oocz_destroy(c)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--world", type=int, default=2)
    ap.add_argument("--sweeps", type=int, default=2)
    ap.add_argument("--P", type=int, default=64)
    ap.add_argument("--sets", type=int, default=0, help="slab sets per rank (0: the library default)")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    S = 1536 // args.world
    # planes on both sides of every rank boundary, and inside
    planes = sorted({0, 764, 1532} | {b + o for b in range(S, 1536, S) for o in (-8, -4, 0, 4)})
    a, ua = run(1, args, planes)
    b, ub = run(args.world, args, planes)
    same = bool(np.array_equal(ua.view(np.uint32), ub.view(np.uint32)))
    print(json.dumps({"grid": [4096, 4096, 1536], "P": args.P, "steps": 4 * args.sweeps, "planes_compared": planes,
                      "values_compared": int(ua.size), "bit_identical": same, "world1": a, f"world{args.world}": b}))


if __name__ == "__main__":
    main()
