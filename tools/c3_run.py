"""BASELINE configs[2]: the 4096 x 4096 x 1536 fp32 wavefield,
previous wavefield and velocity model (3 x 103 GB raw = 309 GB, more than the
183 GB of HBM and the 196 GB of host RAM) streamed out of core on ONE B200 at
ZFP rate 16 (a 154.6 GB pinned compressed store), P = 192 (8 z-blocks), T = 4.

Inputs are generated on the GPU in z-chunks (the DENSE(2) / LAYERED recipes of
synth.py, same fp64 operations, so the values are bit-identical to synth's --
checked on two chunks) and compressed with oocz_set_field_planes; nothing of
full size ever exists in host memory except the pinned compressed store.
Timing: W warm-up sweeps, then K sweeps device-timed on the library's streams.
Parity: the run's u at sampled points vs the CPU oracle on a sub-box around
each point (the cone of the 4T(W+K) steps plus a ZFP block, clipped at the
domain boundary), bit for bit -- the reduced schedule is local.
The raw (uncompressed) run cannot be made on this box: its 309 GB store does
not fit in host memory (which is the paper's point).

  python tools/c3_run.py [--nz 1536] [--warmup 1] [--sweeps 2] [--samples 8]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402  (test infrastructure: the sampled parity check only)
from paper_2109_05410_b200 import oocz as Z  # noqa: E402
from paper_2109_05410_b200 import synth  # noqa: E402


def dense_chunk_gpu(nx, ny, nz, seed, z0, z1, torch):
    """synth.dense planes [z0, z1) computed on the GPU with the same fp64 operations."""
    i = np.arange(nx, dtype=np.float64)
    j = np.arange(ny, dtype=np.float64)
    k = np.arange(z0, z1, dtype=np.float64)
    out = torch.zeros((z1 - z0, ny, nx), dtype=torch.float64, device="cuda")
    for lam, ph, a in synth.dense_params(seed):
        sx = torch.from_numpy(np.sin(2 * np.pi * i / lam[0] + ph[0])).cuda()
        sy = torch.from_numpy(np.sin(2 * np.pi * j / lam[1] + ph[1])).cuda()
        asz = torch.from_numpy(a * np.sin(2 * np.pi * k / lam[2] + ph[2])).cuda()   # a * sz, as numpy
        out += asz[:, None, None] * (sy[:, None] * sx[None, :])[None, :, :]
    return out.to(torch.float32)


def dense_box(nx, ny, nz, seed, lo, hi):
    """synth.dense restricted to the box [lo, hi) (x, y, z): the same elementwise
    fp64 operations on sub-ranges of the index vectors, so the same values."""
    i = np.arange(lo[0], hi[0], dtype=np.float64)
    j = np.arange(lo[1], hi[1], dtype=np.float64)
    k = np.arange(lo[2], hi[2], dtype=np.float64)
    out = np.zeros((hi[2] - lo[2], hi[1] - lo[1], hi[0] - lo[0]), np.float64)
    for lam, ph, a in synth.dense_params(seed):
        sx = np.sin(2 * np.pi * i / lam[0] + ph[0])
        sy = np.sin(2 * np.pi * j / lam[1] + ph[1])
        sz = np.sin(2 * np.pi * k / lam[2] + ph[2])
        out += a * sz[:, None, None] * (sy[:, None] * sx[None, :])[None, :, :]
    return out.astype(np.float32)


def layered_box(nx, ny, nz, lo, hi):
    i = np.arange(lo[0], hi[0], dtype=np.float64)
    j = np.arange(lo[1], hi[1], dtype=np.float64)
    k = np.arange(lo[2], hi[2])
    vel = np.array([1500.0, 2500.0, 3500.0, 4500.0])[np.minimum((4 * k) // max(nz, 1), 3)]
    lat = 1.0 + 0.05 * np.sin(2 * np.pi * j / 97.0)[:, None] * np.sin(2 * np.pi * i / 89.0)[None, :]
    m = (vel[:, None, None] * lat[None, :, :] * 0.4 / 4500.0) ** 2
    return m.astype(np.float32)


def layered_chunk_gpu(nx, ny, nz, z0, z1, lat_gpu, torch):
    k = np.arange(z0, z1)
    vel = torch.from_numpy(np.array([1500.0, 2500.0, 3500.0, 4500.0])[np.minimum((4 * k) // max(nz, 1), 3)]).cuda()
    t = vel[:, None, None] * lat_gpu[None, :, :] * 0.4 / 4500.0
    return (t * t).to(torch.float32)


def main():
    import torch
    ap = argparse.ArgumentParser()
    ap.add_argument("--nx", type=int, default=4096)
    ap.add_argument("--nz", type=int, default=1536)
    ap.add_argument("--P", type=int, default=192)
    ap.add_argument("--T", type=int, default=4)
    ap.add_argument("--rate", type=int, default=16)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--sweeps", type=int, default=2)
    ap.add_argument("--samples", type=int, default=8)
    ap.add_argument("--chunk", type=int, default=16)
    ap.add_argument("--schedules", default="paper_faithful,serpentine")
    ap.add_argument("--no-parity", action="store_true", help="timing only (A/B variants)")
    args = ap.parse_args()
    nx = ny = args.nx
    nz, P, T, rate = args.nz, args.P, args.T, args.rate
    torch.cuda.set_device(0)
    res = {"config": {"grid": [nx, ny, nz], "P": P, "T": T, "rate": rate, "fields": 3,
                      "raw_bytes": 3 * nx * ny * nz * 4,
                      "compressed_store_bytes": 3 * Z.oocz_zfp_bytes(nx, ny, nz, rate)},
           "runs": {}}
    # 1) the GPU generator is bit-identical to synth's (two chunks, checked on the host)
    i = np.arange(nx, dtype=np.float64)
    j = np.arange(ny, dtype=np.float64)
    lat = 1.0 + 0.05 * np.sin(2 * np.pi * j / 97.0)[:, None] * np.sin(2 * np.pi * i / 89.0)[None, :]
    lat_gpu = torch.from_numpy(lat).cuda()
    for z0 in (0, nz - 4):
        g = dense_chunk_gpu(nx, ny, nz, 2, z0, z0 + 4, torch).cpu().numpy()
        assert np.array_equal(g.view(np.uint32), synth.dense(nx, ny, nz, seed=2, z0=z0, z1=z0 + 4).view(np.uint32))
        g = layered_chunk_gpu(nx, ny, nz, z0, z0 + 4, lat_gpu, torch).cpu().numpy()
        assert np.array_equal(g.view(np.uint32), synth.layered(nx, ny, nz, z0=z0, z1=z0 + 4).view(np.uint32))
        lo, hi = (nx - 40, 8, z0), (nx, 48, z0 + 4)                  # the box generators too
        assert np.array_equal(dense_box(nx, ny, nz, 2, lo, hi),
                              synth.dense(nx, ny, nz, seed=2, z0=z0, z1=z0 + 4)[:, 8:48, nx - 40:])
        assert np.array_equal(layered_box(nx, ny, nz, lo, hi), synth.layered(nx, ny, nz, z0=z0, z1=z0 + 4)[:, 8:48, nx - 40:])
    res["generator_check"] = ("GPU DENSE(2) / LAYERED chunks and the host sub-box generators == synth.dense / "
                              "synth.layered bit for bit (2 chunks)")
    rng = np.random.default_rng(5)
    pts = [(int(rng.integers(0, nx)), int(rng.integers(0, ny)), int(rng.integers(0, nz))) for _ in range(args.samples)]
    pts += [(3, 5, 1), (nx - 2, ny // 2, nz - 3)]          # next to the domain boundary
    nsteps = T * (args.warmup + args.sweeps)
    for spec in args.schedules.split(","):
        # "name[:P]": paper_faithful, serpentine, or serpentine_mres (serpentine sweeps + m
        # decoded once into HBM: 98 GiB at C3, so it needs a smaller P to fit)
        # "hbm[:P[:slots[:sets]]]": the whole compressed store in HBM (154.6 GB at
        # rate 16) beside one slab set -- the 309 GB state stepped without the host link
        parts = spec.split(":")                  # name[:P[:slots[:sets]]]
        sched = parts[0]
        Pk = int(parts[1]) if len(parts) > 1 else P
        slots = int(parts[2]) if len(parts) > 2 else 2
        hbm = sched == "hbm"
        sets = int(parts[3]) if len(parts) > 3 else (1 if hbm else 0)
        cfg = Z.oocz_default_config(nx, ny, nz, tb=T, block_planes=Pk, rate=[rate] * 3,
                                    store=Z.OOCZ_STORE_DEVICE if hbm else Z.OOCZ_STORE_HOST,
                                    serpentine=int(sched.startswith("serpentine")),
                                    m_resident=int(sched.endswith("mres")), slots=slots, slab_sets=sets)
        t0 = time.time()
        ctx = Z.oocz_create(cfg)
        t_create = time.time() - t0
        try:
            t0 = time.time()
            for z0 in range(0, nz, args.chunk):
                z1 = min(z0 + args.chunk, nz)
                d = dense_chunk_gpu(nx, ny, nz, 2, z0, z1, torch)
                Z.oocz_set_field_planes(ctx, Z.OOCZ_U, z0, d)
                Z.oocz_set_field_planes(ctx, Z.OOCZ_UPREV, z0, d)
                Z.oocz_set_field_planes(ctx, Z.OOCZ_M, z0, layered_chunk_gpu(nx, ny, nz, z0, z1, lat_gpu, torch))
                del d
            torch.cuda.synchronize()
            t_set = time.time() - t0
            Z.oocz_step(ctx, T * args.warmup)
            s0 = Z.oocz_get_stats(ctx)
            Z.oocz_step(ctx, T * args.sweeps)
            st = Z.oocz_get_stats(ctx)
            dev_s = st["last_step_device_ms"] / 1e3
            h2d = st["h2d_bytes"] - s0["h2d_bytes"]
            d2h = st["d2h_bytes"] - s0["d2h_bytes"]
            cups = nx * ny * nz * T * args.sweeps / dev_s
            run = {"P": Pk, "slots": slots, "slab_sets": sets, "store": "device" if hbm else "host",
                   "cell_updates_per_s": round(cups, 1), "s_per_sweep": round(dev_s / args.sweeps, 3),
                   "h2d_bytes_per_sweep": h2d // args.sweeps, "d2h_bytes_per_sweep": d2h // args.sweeps,
                   "h2d_GBps": round(h2d / dev_s / 1e9, 2), "d2h_GBps": round(d2h / dev_s / 1e9, 2),
                   "device_bytes": st["device_bytes_used"], "pinned_host_bytes": st["host_bytes_pinned"],
                   "create_s": round(t_create, 1), "set_fields_s": round(t_set, 1), "steps_total": nsteps}
            print(sched, json.dumps(run), flush=True)
            if args.no_parity:
                res["runs"][spec] = run
                continue
            # 2) sampled parity vs the oracle on sub-boxes
            # corruption from a cut edge moves 4 cells per step, plus up to 3 cells
            # (one ZFP block) at each of the W + K round trips
            R = 4 * nsteps + 4 * (args.warmup + args.sweeps) + 8
            ok = 0
            for (x, y, zz) in pts:
                zb = zz // 4 * 4
                g = Z.oocz_get_field_planes(ctx, Z.OOCZ_U, zb, np.empty((4, ny, nx), np.float32))
                got = g[zz - zb, y, x]
                lo = [max(0, (c - R) // 4 * 4) for c in (x, y, zz)]
                hi = [min(n, ((c + R) // 4 + 1) * 4) for c, n in zip((x, y, zz), (nx, ny, nz))]
                # sub-box of the inputs; where the box is cut inside the domain its edge
                # is an artificial zero boundary, R away from the point: outside the cone
                u = dense_box(nx, ny, nz, 2, lo, hi)
                m = layered_box(nx, ny, nz, lo, hi)
                ou, _ = oracle.run(u, u, m, T, (rate,) * 3, nsteps)
                want = ou[zz - lo[2], y - lo[1], x - lo[0]]
                same = np.float32(got).view(np.uint32) == np.float32(want).view(np.uint32)
                ok += int(same)
                if not same:
                    print("MISMATCH", (x, y, zz), got, want, flush=True)
            run["sampled_parity"] = {"points": len(pts), "bit_exact": ok, "steps": nsteps,
                                     "oracle": f"oracle.run on the sub-box within {R} cells of each point"}
            res["runs"][spec] = run
            print(sched, "parity", ok, "/", len(pts), flush=True)
        finally:
            Z.oocz_destroy(ctx)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
