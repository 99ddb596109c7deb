"""Per-sweep drain of the z-partitioned pipeline, measured on ONE GPU with the
in-process local group (the same halo protocol as NCCL, device copies).

A: OOCZ_HALO_ONE_GROUP=1 -- both halo directions in one exchange on one
   stream, the round-1 protocol (each rank's first block of a sweep waits for
   the neighbours' LAST blocks of the previous sweep in both directions);
B: the per-direction protocol (halo.h): each direction completes on its own.
With ascending sweeps block 0 still needs the upper neighbour's last block
(inherent); serpentine sweeps make every halo a product of the neighbour's
FIRST block of the previous sweep.  world = 1 on the same grid is the bound.

  python tools/halo_drain.py [--nz 1024] [--sweeps 6] [--store 0]
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2109_05410_b200 import oocz as Z  # noqa: E402
from paper_2109_05410_b200 import synth  # noqa: E402


def run(world, one_group, opts, u, m, args):
    os.environ["OOCZ_HALO_ONE_GROUP"] = "1" if one_group else "0"
    nx = ny = args.n
    nz = args.nz
    cfg = Z.oocz_default_config(nx, ny, nz, tb=4, block_planes=args.P, rate=[16] * 3, store=args.store, **opts)
    S = nz // world
    ctxs = Z.oocz_create_local_group(cfg, world) if world > 1 else [Z.oocz_create(cfg)]
    try:
        for r, c in enumerate(ctxs):
            for f, a in ((Z.OOCZ_U, u), (Z.OOCZ_UPREV, u), (Z.OOCZ_M, m)):
                Z.oocz_set_field(c, f, np.ascontiguousarray(a[r * S:(r + 1) * S]))
        step = (lambda n: Z.oocz_step_local_group(ctxs, n)) if world > 1 else (lambda n: Z.oocz_step(ctxs[0], n))
        step(4 * 2)
        best = 0.0
        for _ in range(args.reps):
            step(4 * args.sweeps)
            ms = max(Z.oocz_get_stats(c)["last_step_device_ms"] for c in ctxs)
            best = max(best, nx * ny * nz * 4 * args.sweeps / (ms / 1e3))
        got = Z.oocz_get_field(ctxs[-1], Z.OOCZ_U, np.empty((S, ny, nx), np.float32))
        return best, got
    finally:
        for c in ctxs:
            Z.oocz_destroy(c)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=512)
    ap.add_argument("--nz", type=int, default=1024)
    ap.add_argument("--P", type=int, default=128)
    ap.add_argument("--sweeps", type=int, default=6)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--store", type=int, default=0)
    args = ap.parse_args()
    u = synth.dense(args.n, args.n, args.nz, seed=1)
    m = synth.layered(args.n, args.n, args.nz)
    res = {"grid": [args.n, args.n, args.nz], "P": args.P, "store": "device" if args.store else "host",
           "unit": "G cell-updates/s (device-timed, max over the group's contexts)"}
    for sname, opts in (("ascending", {}), ("serpentine+m_resident", dict(serpentine=1, m_resident=1, slots=3))):
        w1, ref = run(1, False, opts, u, m, args)
        a, ga = run(2, True, opts, u, m, args)
        b, gb = run(2, False, opts, u, m, args)
        S = args.nz // 2
        same = bool(np.array_equal(ga.view(np.uint32), gb.view(np.uint32)))
        res[sname] = {"world1": round(w1 / 1e9, 2), "world2_one_group": round(a / 1e9, 2),
                      "world2_per_direction": round(b / 1e9, 2), "per_direction_over_one_group": round(b / a, 3),
                      "bit_identical_protocols": same}
        print(sname, res[sname], flush=True)
        del ref
    print(json.dumps(res))


if __name__ == "__main__":
    main()
