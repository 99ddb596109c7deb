#!/usr/bin/env python3
"""Benchmark of the out-of-core compressed stencil stepper (arXiv 2109.05410).

One bench "step" = one sweep = T = 4 leapfrog steps over the whole grid through
the whole hot path (per z-block H2D/decode ->
4 cone-limited 25-point steps -> encode/D2H, region sharing, 3 streams).

Workload (BASELINE.json configs[1]): 512^3 fp32, DENSE(seed 1) wavefield,
u- = u, LAYERED m; P = 128 (4 z-blocks), T = 4, ZFP fixed rate 16 on all three
fields, and the same with compression off ("raw") for the paper's speedup
question.  Metric: cell-updates/s = nx*ny*nz*T*K / time of K sweeps.

  value : compressed store resident in HBM (inputs already on the device):
          decode -> stencil -> encode per block, device-timed (CUDA events on
          the library's own streams), max over ranks.
  e2e   : the paper's out-of-core path through the public C ABI with the
          store in pinned HOST memory: every sweep moves the whole compressed
          state H2D and the read-write fields D2H inside the timed region.

Multi-GPU (torchrun, N > 1): the grid is z-partitioned, one 512^3 slab per
rank (weak scaling), radius-4 halos exchanged in compressed form with NCCL.

--impl reference: the CPU oracle (oracle/, test infrastructure) timed on
the host cores on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "cell-updates/s out-of-core, ZFP vs raw, at 1/2/4/8 B200; max rel. error"
NX = NY = NZ = 512
T = 4
P = 128
RATE = 16


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            j = json.load(fh)
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ---------------------------------------------------------------- GPU arm
def make_fields(rank: int, S: int):
    from paper_2109_05410_b200 import synth
    z0 = rank * S
    u = synth.dense(NX, NY, NZ, seed=1, z0=z0 % NZ, z1=z0 % NZ + S) if S <= NZ else None
    m = synth.layered(NX, NY, NZ, z0=z0 % NZ, z1=z0 % NZ + S)
    return u, u, m


def run_mode(Z, store, rates, fields, rank, world, nccl_id, device, steps, warmup, dist, profile, m_resident=0,
             tb=T, precision=32, serpentine=0, slots=2, slab_sets=0, graphs=0):
    """Returns (device seconds for `steps` sweeps (max over ranks), stats, events, launches)."""
    import torch
    cfg = Z.oocz_default_config(NX, NY, NZ * world, tb=tb, block_planes=P, rate=list(rates), store=store,
                                m_resident=m_resident, precision=precision, serpentine=serpentine,
                                slots=slots, profile=profile, slab_sets=slab_sets, graphs=graphs)
    if callable(nccl_id):   # a fresh NCCL unique id per communicator (an id bootstraps one init only)
        nccl_id = nccl_id()
    ctx = Z.oocz_create(cfg, rank, world, nccl_id, device)
    try:
        for f, a in zip((Z.OOCZ_U, Z.OOCZ_UPREV, Z.OOCZ_M), fields):
            Z.oocz_set_field(ctx, f, a.astype(np.float64) if precision == 64 else a)
        Z.oocz_step(ctx, warmup * tb)
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        st0 = Z.oocz_get_stats(ctx)
        l0 = Z.oocz_kernel_launch_count()
        Z.oocz_step(ctx, steps * tb)
        launches = Z.oocz_kernel_launch_count() - l0
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        st = Z.oocz_get_stats(ctx)
        for k in ("sweeps", "h2d_bytes", "d2h_bytes", "halo_bytes"):   # the timed call only
            st[k] -= st0[k]
        dev_s = st["last_step_device_ms"] / 1e3
        if dist:
            from paper_2109_05410_b200 import dist as D
            dev_s = D.max_over_ranks(dist, dev_s, device="cuda")
        evs = Z.oocz_get_events(ctx) if profile else []
        # per-sweep bytes of the timed call only
        st_all = st
        return dev_s, st_all, evs, launches, ctx
    except Exception:
        Z.oocz_destroy(ctx)
        raise


def host_link_probe(nbytes: int = 512 << 20, reps: int = 5) -> dict:
    """Measured host-link peak (the out-of-core roofline's denominator):
    pinned cudaMemcpyAsync H2D alone, D2H alone, and both at once on two
    streams (the pipeline's situation), CUDA events, best of `reps`."""
    import torch
    h_in = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    h_out = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    d_a = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    d_b = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def run(h2d: bool, d2h: bool) -> float:
        best = 0.0
        for _ in range(reps):
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e0.record(s1)
            s2.wait_event(e0)
            if h2d:
                with torch.cuda.stream(s1):
                    d_a.copy_(h_in, non_blocking=True)
            if d2h:
                with torch.cuda.stream(s2):
                    h_out.copy_(d_b, non_blocking=True)
            e1, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e1.record(s1)
            e2.record(s2)
            torch.cuda.synchronize()
            ms = max(e0.elapsed_time(e1), e0.elapsed_time(e2))
            best = max(best, nbytes / (ms / 1e3) / 1e9)
        return best

    return {"h2d_GBps": round(run(True, False), 2), "d2h_GBps": round(run(False, True), 2),
            "concurrent_per_direction_GBps": round(run(True, True), 2), "bytes": nbytes}


def lanes_summary(evs) -> dict:
    """Per-lane busy time over the profiled step (SPEC.md:352 'per-lane idle')."""
    names = {0: "h2d", 1: "compute", 2: "d2h", 3: "comm", 4: "decode", 5: "encode"}
    if not evs:
        return {}
    t0 = min(e["start_ms"] for e in evs)
    t1 = max(e["end_ms"] for e in evs)
    out = {}
    for lane in sorted({e["lane"] for e in evs}):
        busy = sum(e["end_ms"] - e["start_ms"] for e in evs if e["lane"] == lane)
        out[names.get(lane, str(lane))] = {"busy_ms": round(busy, 3), "busy_frac": round(busy / (t1 - t0), 3)}
    out["span_ms"] = round(t1 - t0, 3)
    return out


def isolated_kernels(Z, fields, peak_gbs, reps: int = 10) -> dict:
    """Each hot kernel alone on one block's slab (P + 2h planes of the C2 data),
    CUDA events on the launching stream, L2 flushed between launches; achieved =
    algorithmic bytes / median duration."""
    import torch
    planes = P + 8 * T
    u = torch.from_numpy(np.ascontiguousarray(fields[0][:planes])).cuda()
    m = torch.from_numpy(np.ascontiguousarray(fields[2][:planes])).cuda()
    up = u.clone()
    out = torch.empty_like(u)
    words = torch.empty(Z.oocz_zfp_bytes(NX, NY, planes, RATE) // 8, dtype=torch.int64, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream()

    def med(fn):
        ts = []
        for _ in range(reps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            fn()
            b.record(s)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) / 1e3)
        return sorted(ts)[len(ts) // 2]

    cells = NX * NY * planes
    cbytes = cells // 64 * 8 * RATE
    upd = NX * NY * (planes - 8)
    res = {}
    for name, fn, nbytes in (
            ("zfp_encode_kernel", lambda: Z.oocz_zfp_encode(u, NX, NY, planes, RATE, words, s), 4 * cells + cbytes),
            ("zfp_decode_kernel", lambda: Z.oocz_zfp_decode(words, NX, NY, planes, RATE, out, s), 4 * cells + cbytes),
            ("stencil25_kernel", lambda: Z.oocz_stencil_step_planes(u, up, m, NX, NY, planes, Z.default_coeffs(),
                                                                    4, planes - 4, 0, planes, s), 16 * upd)):
        t = med(fn)
        res[name] = {"ms": round(t * 1e3, 4), "achieved_GBps": round(nbytes / t / 1e9, 1),
                     "frac": round(nbytes / t / 1e9 / peak_gbs, 4), "algorithmic_bytes": int(nbytes)}
    # fp64 twins (the paper's precision) at its 2:1 rate 32/64
    u64, m64 = u.double(), m.double()
    up64, out64 = u64.clone(), torch.empty_like(u64)
    r64 = 32
    words64 = torch.empty(Z.oocz_zfp_bytes(NX, NY, planes, r64) // 8, dtype=torch.int64, device="cuda")
    cb64 = cells // 64 * 8 * r64
    for name, fn, nbytes in (
            ("zfp_encode64_kernel", lambda: Z.oocz_zfp_encode_f64(u64, NX, NY, planes, r64, words64, s),
             8 * cells + cb64),
            ("zfp_decode64_kernel", lambda: Z.oocz_zfp_decode_f64(words64, NX, NY, planes, r64, out64, s),
             8 * cells + cb64),
            ("stencil25_kernel<double>", lambda: Z.oocz_stencil_step_planes_f64(
                u64, up64, m64, NX, NY, planes, Z.default_coeffs64(), 4, planes - 4, 0, planes, s), 32 * upd)):
        t = med(fn)
        res[name] = {"ms": round(t * 1e3, 4), "achieved_GBps": round(nbytes / t / 1e9, 1),
                     "frac": round(nbytes / t / 1e9 / peak_gbs, 4), "algorithmic_bytes": int(nbytes)}
    return res


def rel_errors(a: np.ndarray, b: np.ndarray, per_plane: int = 100, seed: int = 7) -> dict:
    """Compressed run `a` vs the uncompressed run `b` after the same steps
    (R18/R19): normwise max|a-b|/max|b| over the whole
    field, and the paper's mean point-wise |a-b|/|b| over `per_plane` seeded
    points per plane (|b| < 1e-30 skipped)."""
    from paper_2109_05410_b200 import synth
    a64, b64 = a.astype(np.float64), b.astype(np.float64)
    normwise = float(np.abs(a64 - b64).max() / max(np.abs(b64).max(), 1e-300))
    nz, ny, nx = b.shape
    r = synth.uniforms(seed, 2 * per_plane * nz).reshape(nz, per_plane, 2)
    ys = (r[..., 0] * ny).astype(np.int64)
    xs = (r[..., 1] * nx).astype(np.int64)
    zs = np.repeat(np.arange(nz), per_plane).reshape(nz, per_plane)
    av, bv = a64[zs, ys, xs], b64[zs, ys, xs]
    keep = np.abs(bv) >= 1e-30
    mean_pw = float(np.mean(np.abs(av - bv)[keep] / np.abs(bv)[keep])) if keep.any() else 0.0
    sig = keep & (np.abs(bv) >= 1e-6 * np.abs(b64).max())     # points the wave has reached
    mean_sig = float(np.mean(np.abs(av - bv)[sig] / np.abs(bv)[sig])) if sig.any() else 0.0
    return {"normwise_max": normwise, "mean_pointwise": mean_pw, "points": int(keep.sum()),
            "skipped": int((~keep).sum()), "mean_pointwise_significant": mean_sig,
            "significant_points": int(sig.sum()), "vs": "same build, compression off (raw)"}


def roofline(evs, peak_gbs, peak_src):
    """Dominant kernel of the timed region from the per-launch CUDA events."""
    from paper_2109_05410_b200.oocz import STAGES
    per = {}
    for e in evs:
        name = STAGES[e["stage"]]
        if name not in ("stencil", "decode", "encode"):
            continue
        d = per.setdefault(name, [0.0, 0, 0])
        d[0] += e["end_ms"] - e["start_ms"]
        d[1] += e["bytes"]
        d[2] += 1
    if not per:
        return None, {}
    dom = max(per, key=lambda k: per[k][0])
    ms, nbytes, n = per[dom]
    achieved = nbytes / (ms / 1e3) / 1e9
    table = {k: {"ms": round(v[0], 4), "launches": v[2], "GB/s": round(v[1] / (v[0] / 1e3) / 1e9, 1)}
             for k, v in per.items()}
    kern = {"stencil": "stencil25_kernel", "decode": "zfp_decode_kernel", "encode": "zfp_encode_kernel"}[dom]
    traffic, tsrc = None, None
    try:   # DRAM bytes per launch from a committed ncu capture of the same in-step launches
        with open(os.path.join(ROOT, "profiles", TRAFFIC_JSON)) as fh:
            tj = json.load(fh)
        if dom == "stencil":
            traffic = int(tj["traffic_over_algorithmic"] * nbytes / n)
            tsrc = (f"profiles/{TRAFFIC_JSON}: ncu dram read+write / algorithmic = "
                    f"{tj['traffic_over_algorithmic']} on the same launches, x this run's algorithmic bytes per launch")
    except Exception:
        pass
    return {"bound": "hbm", "kernel": kern, "achieved": round(achieved, 1), "peak": peak_gbs,
            "peak_source": peak_src, "unit": "GB/s", "frac": round(achieved / peak_gbs, 4),
            "traffic": traffic, "traffic_source": tsrc, "avg_launch_ms": round(ms / n, 4),
            "algorithmic_bytes_per_launch": int(nbytes / n)}, table


TRAFFIC_JSON = "r01_stencil_instep_traffic.json"
ALU_PEAK = 148 * 4 * 0.5 * 1.965   # G warp-instructions/s: ALU pipe, rt 2 cycles per SMSP (B300_MICROARCH)


def codec_alu_roofline(table) -> dict | None:
    """The codec kernels are bound by the integer ALU pipe (IADD3/LOP3/SHF/PRMT,
    DESIGN.md "Roofline"), not by HBM: their fraction is the ALU pipe's share of
    its peak issue rate (148 SMs x 4 sub-partitions x one warp-instruction per
    2 cycles at 1965 MHz = 581.6 G warp-instructions/s), measured by ncu
    (sm__inst_executed_pipe_alu) on the committed capture of the same kernels."""
    try:
        with open(os.path.join(ROOT, "profiles", "r01_ncu_kernels.json")) as fh:
            kj = json.load(fh)
    except Exception:
        return None
    out = {}
    for name, stage in (("zfp_decode_kernel", "decode"), ("zfp_encode_kernel", "encode")):
        ks = [k for k in kj["kernels"] if k["kernel"].endswith(name)]
        if not ks:
            continue
        k = ks[0]
        frac = k["sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"] / 100.0
        out[name] = {"bound": "alu", "achieved": round(frac * ALU_PEAK, 1), "peak": round(ALU_PEAK, 1),
                     "unit": "G ALU-pipe warp-instructions/s", "frac": round(frac, 4),
                     "issue_active": round(k["smsp__issue_active.avg.pct_of_peak_sustained_active"] / 100, 4),
                     "isolated_us": k["gpu__time_duration.sum"],
                     "in_step_avg_ms": round(table[stage]["ms"] / table[stage]["launches"], 4) if stage in table else None,
                     "source": "profiles/r01_ncu_kernels.json (ncu --set full, one C2 slab, rate 16)"}
    return out or None


def gpu_arm(args):
    import torch
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as td
        td.init_process_group("nccl", device_id=torch.device("cuda", local))
        dist = td
    from paper_2109_05410_b200 import oocz as Z
    from paper_2109_05410_b200 import dist as D
    nccl_id = (lambda: D.share_nccl_id(dist, rank, Z.oocz_get_nccl_id, device="cuda")) if world > 1 else None
    fields = make_fields(rank, NZ)
    cells = NX * NY * NZ * world * T * args.steps
    peak_gbs, peak_src = peaks()
    link = host_link_probe()
    out = {}
    with ClockSampler(local) as clk:
        # (label, store, rates, options).  The headline runs the library's fastest
        # orchestration of the SAME computation (bit-identical results, tests):
        # serpentine sweeps + m resident in HBM (readings R22/R23);
        # "pf_*" are the paper-faithful schedule (ascending sweeps, m streamed).
        # Each path runs its fastest schedule of the same computation: with the store
        # in HBM m resident (serpentine sweeps save host-link bytes only, and the
        # block at each turn serialises decode after its own encode); out of core
        # serpentine + m resident + 3 staging slots.
        OD = dict(m_resident=1)
        OH = dict(serpentine=1, m_resident=1, slots=3)
        PF = dict(serpentine=0, m_resident=0)
        modes = [("zfp_dev", 1, (RATE,) * 3, OD), ("zfp_host", 0, (RATE,) * 3, OH),
                 ("raw_dev", 1, (0, 0, 0), OD), ("raw_host", 0, (0, 0, 0), OH)]
        # the single-GPU analyses (other rates, schedules, paper modes, fp64, T) run at
        # N = 1; a multi-GPU run measures the headline paths only (each extra mode is
        # another NCCL communicator and pinned store per rank)
        if not args.quick and world == 1:   # configs[1]: rates 8/16/24
            modes += [(f"r{r}_{k}", st, (r,) * 3, o) for r in (8, 24) for k, st, o in (("dev", 1, OD), ("host", 0, OH))]
            # the paper-faithful schedule, and each orchestration alone
            modes += [("pf_zfp_dev", 1, (RATE,) * 3, PF), ("pf_zfp_host", 0, (RATE,) * 3, PF),
                      ("pf_raw_dev", 1, (0, 0, 0), PF), ("pf_raw_host", 0, (0, 0, 0), PF),
                      ("mres_host", 0, (RATE,) * 3, dict(m_resident=1)),
                      ("serp_dev", 1, (RATE,) * 3, dict(serpentine=1)), ("serp_host", 0, (RATE,) * 3, dict(serpentine=1)),
                      ("sm_dev", 1, (RATE,) * 3, dict(serpentine=1, m_resident=1)),
                      # two staging slots: the block after each turn re-reads its own rows
                      ("sm2_host", 0, (RATE,) * 3, dict(serpentine=1, m_resident=1, slots=2))]
            # the paper's codes 2-4 as fp32 rate vectors, out of core,
            # paper-faithful schedule: one read-write field (u-, reading R7) at 16/32, the
            # read-only m at 16/32, one read-write field + m at 12/32 (the paper's 24/64)
            modes += [("pm2_host", 0, (0, 16, 0), PF), ("pm3_host", 0, (0, 0, 16), PF),
                      ("pm4_host", 0, (0, 12, 12), PF)]
            # temporal-blocking depth: T = 8 and the paper's T = 12
            # (PAPER.md:217), same P = 128: host bytes per step fall as 1/T, redundant
            # stencil work grows as 4(T-1)/P
            modes += [(f"t{t}_{k}", st, (RATE,) * 3, dict(o, tb=t)) for t in (8, 12) for k, st, o in (("dev", 1, OD), ("host", 0, OH))]
            # the paper's own precision (fp64) and rates 32/64, 24/64
            # (PAPER.md:213-215): codes 1-4 out of core (paper-faithful schedule), plus all
            # fields at 32/64 (paper-faithful and orchestrated)
            F = dict(PF, precision=64)
            modes += [("f64raw_host", 0, (0, 0, 0), F), ("f64pm2_host", 0, (0, 32, 0), F),
                      ("f64pm3_host", 0, (0, 0, 32), F), ("f64pm4_host", 0, (0, 24, 24), F),
                      ("f64all_host", 0, (32, 32, 32), F), ("f64all_dev", 1, (32, 32, 32), F),
                      ("f64raw_dev", 1, (0, 0, 0), F),
                      ("f64allo_host", 0, (32, 32, 32), dict(OH, precision=64)),
                      ("f64allo_dev", 1, (32, 32, 32), dict(OD, precision=64))]
        for label, store, rates, opt in modes:
            tb = opt.get("tb", T)
            prec = opt.get("precision", 32)
            dev_s, st, evs, launches, ctx = run_mode(Z, store, rates, fields, rank, world, nccl_id, local,
                                                     args.steps, args.warmup, dist,
                                                     profile=int(label in ("zfp_dev", "zfp_host")),
                                                     m_resident=opt.get("m_resident", 0), tb=tb,
                                                     precision=prec, serpentine=opt.get("serpentine", 0),
                                                     slots=opt.get("slots", 2),
                                                     slab_sets=opt.get("slab_sets", 0))
            sweeps_total = st["sweeps"]
            cells_mode = cells // T * tb
            out[label] = {"s": dev_s, "cups": cells_mode / dev_s, "launches": launches, "evs": evs,
                          "h2d_per_sweep": st["h2d_bytes"] / max(sweeps_total, 1),
                          "d2h_per_sweep": st["d2h_bytes"] / max(sweeps_total, 1),
                          "halo_per_sweep": st["halo_bytes"] / max(sweeps_total, 1)}
            if store == 1 or "pm" in label or label.startswith("f64") or label.endswith("raw_host"):
                # final u^t, for the compressed-vs-raw error (same step count)
                out[label]["u"] = Z.oocz_get_field(ctx, Z.OOCZ_U, np.empty((NZ, NY, NX),
                                                                           np.float64 if prec == 64 else np.float32))
            Z.oocz_destroy(ctx)
    clocks = clk.summary()
    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    roof, table = roofline(out["zfp_dev"]["evs"], peak_gbs, peak_src)
    err = rel_errors(out["zfp_dev"]["u"], out["raw_dev"]["u"])
    err["steps"] = (args.warmup + args.steps) * T
    paper_modes = None
    if "pm2_host" in out:
        ref = out["pf_raw_host"]
        paper_modes = {"what": "PAPER.md:212-215 codes as rate vectors (u, u-, m); out of core; "
                               "speedup vs code 1 (the paper: 1.16x / 1.18x / 1.20x, fp64, V100-PCIe)",
                       "1_original": {"rates": [0, 0, 0], "e2e": round(ref["cups"], 1)}}
        for key, lab, rates in (("2_rw_16", "pm2_host", [0, 16, 0]), ("3_ro_16", "pm3_host", [0, 0, 16]),
                                ("4_rw_ro_12", "pm4_host", [0, 12, 12])):
            er = rel_errors(out[lab]["u"], ref["u"])
            paper_modes[key] = {"rates": rates, "e2e": round(out[lab]["cups"], 1),
                                "speedup": round(out[lab]["cups"] / ref["cups"], 3),
                                "normwise_max_rel_error": er["normwise_max"],
                                "mean_pointwise_rel_error": er["mean_pointwise"]}
    paper_fp64 = None
    if "f64raw_host" in out:
        ref = out["f64raw_host"]
        paper_fp64 = {"what": "the paper's precision and rates (fp64; PAPER.md:208, :212-215): codes 1-4 out of core "
                              "and every field at 32/64; speedup vs code 1 (the paper: 1.16x / 1.18x / 1.20x, "
                              "V100-PCIe)",
                      "1_original": {"rates": [0, 0, 0], "e2e": round(ref["cups"], 1),
                                     "value": round(out["f64raw_dev"]["cups"], 1)}}
        for key, lab, rates in (("2_rw_32", "f64pm2_host", [0, 32, 0]), ("3_ro_32", "f64pm3_host", [0, 0, 32]),
                                ("4_rw_ro_24", "f64pm4_host", [0, 24, 24]), ("all_32", "f64all_host", [32, 32, 32])):
            er = rel_errors(out[lab]["u"], ref["u"])
            paper_fp64[key] = {"rates": rates, "e2e": round(out[lab]["cups"], 1),
                               "speedup": round(out[lab]["cups"] / ref["cups"], 3),
                               "e2e_h2d_bytes_per_step": int(out[lab]["h2d_per_sweep"]),
                               "normwise_max_rel_error": er["normwise_max"],
                               "mean_pointwise_rel_error": er["mean_pointwise"]}
        paper_fp64["all_32"]["value"] = round(out["f64all_dev"]["cups"], 1)
        paper_fp64["all_32_orchestrated"] = {"rates": [32, 32, 32], "e2e": round(out["f64allo_host"]["cups"], 1),
                                             "value": round(out["f64allo_dev"]["cups"], 1),
                                             "speedup": round(out["f64allo_host"]["cups"] / ref["cups"], 3),
                                             "schedule": "value: m resident; e2e: serpentine + m resident, 3 slots"}
    orch = None
    if "mres_host" in out:
        orch = {"what": "SURVEY 8(f) row 2, beyond the paper, same bits: the paper-faithful schedule (ascending "
                        "sweeps, m streamed), m decoded once and kept in HBM (m_resident=1, R23), serpentine "
                        "sweeps (serpentine=1, R22), both (2 staging slots); the headline value runs m_resident, "
                        "the headline e2e serpentine + m_resident with 3 staging slots"}
        for key, dlab, hlab in (("paper_faithful", "pf_zfp_dev", "pf_zfp_host"),
                                ("m_resident", "zfp_dev", "mres_host"), ("serpentine", "serp_dev", "serp_host"),
                                ("serpentine+m_resident", "sm_dev", "sm2_host")):
            dv, hs = out[dlab], out[hlab]
            orch[key] = {"value": round(dv["cups"], 1), "e2e": round(hs["cups"], 1),
                         "e2e_h2d_bytes_per_step": int(hs["h2d_per_sweep"]),
                         "e2e_d2h_bytes_per_step": int(hs["d2h_per_sweep"]),
                         "e2e_host_link_GBps": round(hs["h2d_per_sweep"] / (hs["s"] / args.steps) / 1e9, 2)}
        if "zfp_host" in out:
            hs = out["zfp_host"]
            orch["serpentine+m_resident, 3 staging slots"] = {
                "e2e": round(hs["cups"], 1), "e2e_h2d_bytes_per_step": int(hs["h2d_per_sweep"]),
                "e2e_d2h_bytes_per_step": int(hs["d2h_per_sweep"]),
                "e2e_d2h_GBps": round(hs["d2h_per_sweep"] / (hs["s"] / args.steps) / 1e9, 2)}
    per_rate = {}
    for r in (8, 24):
        if f"r{r}_dev" in out:
            er = rel_errors(out[f"r{r}_dev"]["u"], out["raw_dev"]["u"])
            per_rate[str(r)] = {"value": round(out[f"r{r}_dev"]["cups"], 1),
                                "e2e": round(out[f"r{r}_host"]["cups"], 1),
                                "e2e_h2d_bytes_per_step": int(out[f"r{r}_host"]["h2d_per_sweep"]),
                                "normwise_max_rel_error": er["normwise_max"],
                                "mean_pointwise_rel_error": er["mean_pointwise"]}
    iso = isolated_kernels(Z, fields, peak_gbs)
    v, e = out["zfp_dev"], out["zfp_host"]
    line = {
        "metric": METRIC,
        "value": round(v["cups"], 1),
        "unit": "cell-updates/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(v["s"] * 1e3 / args.steps, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic (DENSE seed 1 wavefield, u- = u, LAYERED m; SURVEY 8(d))",
        "config": {"workload": f"C2: {NX}^3 fp32 per GPU, 25-point leapfrog, P={P} ({NZ // P} z-blocks), "
                               f"T={T}, ZFP rate {RATE} on u, u-, m; compressed store resident in HBM; "
                               f"m decoded once (same bits as the paper's schedule)",
                   "schedule": "value: m_resident=1; e2e: serpentine=1, m_resident=1, slots=3 (each path's "
                               "fastest schedule, all bit-identical; the paper-faithful schedule and each "
                               "orchestration alone: orchestrated.*)",
                   "grid": [NX, NY, NZ * world], "tb": T, "block_planes": P, "rate": RATE,
                   "step": "one sweep = T leapfrog steps over the whole grid",
                   "l2": "inputs larger than L2 (compressed store 768 MiB + 480 MiB slab per GPU)",
                   "parallelism": f"z-slabs x{world}, NCCL compressed halos" if world > 1 else "single GPU"},
        "e2e": {"value": round(e["cups"], 1), "unit": "cell-updates/s",
                "h2d_bytes_per_step": int(e["h2d_per_sweep"]), "d2h_bytes_per_step": int(e["d2h_per_sweep"]),
                "path": "oocz_step with the store in pinned host memory (the paper's out-of-core path)",
                "host_link_GBps": {"h2d": round(e["h2d_per_sweep"] / (e["s"] / args.steps) / 1e9, 2),
                                   "d2h": round(e["d2h_per_sweep"] / (e["s"] / args.steps) / 1e9, 2)},
                # the out-of-core roofline: bytes the method must move per sweep in the
                # busier direction (region sharing: every stored byte once H2D, the
                # read-write ones once D2H; less with serpentine / m resident) over the
                # measured concurrent pinned bandwidth per direction
                "roofline": {"bound": "host-link",
                             "achieved": round(max(e["h2d_per_sweep"], e["d2h_per_sweep"]) /
                                               (e["s"] / args.steps) / 1e9, 2),
                             "peak": link["concurrent_per_direction_GBps"], "unit": "GB/s",
                             "frac": round(max(e["h2d_per_sweep"], e["d2h_per_sweep"]) / (e["s"] / args.steps) /
                                           1e9 / link["concurrent_per_direction_GBps"], 4),
                             "peak_source": "measured in this run (bench.host_link_probe)"},
                "host_link_probe": link,
                "lanes": lanes_summary(e["evs"])},
        "raw": {"value": round(out["raw_dev"]["cups"], 1), "e2e": round(out["raw_host"]["cups"], 1),
                "e2e_h2d_bytes_per_step": int(out["raw_host"]["h2d_per_sweep"]),
                "schedule": "the headline's (value: m resident; e2e: serpentine + m resident, 3 slots)"},
        "speedup_zfp_vs_raw": {"value": round(v["cups"] / out["raw_dev"]["cups"], 3),
                               "e2e": round(e["cups"] / out["raw_host"]["cups"], 3),
                               "paper_context": "1.20x (fp64, V100-PCIe, PAPER.md:227)",
                               **({"paper_faithful_e2e": round(out["pf_zfp_host"]["cups"] / out["pf_raw_host"]["cups"], 3)}
                                  if "pf_raw_host" in out else {})},
        "max_rel_error": err,
        "gpu_launches": int(v["launches"]),
        "roofline": roof,
        "roofline_codec": codec_alu_roofline(table),
        "kernels_in_step": table,
        "lanes": lanes_summary(v["evs"]),
        "roofline_isolated": iso,
        "other_rates": per_rate,
        "orchestrated": orch,
        "paper_modes": paper_modes,
        "paper_precision_fp64": paper_fp64,
        "temporal_blocking": {f"T={t}": {"value": round(out[f"t{t}_dev"]["cups"], 1),
                                         "e2e": round(out[f"t{t}_host"]["cups"], 1),
                                         "e2e_h2d_bytes_per_step": int(out[f"t{t}_host"]["h2d_per_sweep"]),
                                         "step": f"one sweep = {t} leapfrog steps"}
                              for t in (8, 12) if f"t{t}_dev" in out} or None,
        "clocks": clocks,
    }
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(seconds=args.cpu_seconds)
    print(json.dumps(line))
    if dist:
        dist.destroy_process_group()


# ---------------------------------------------------------------- CPU oracle arm
def _oracle_sweep_sample(planes: int):
    """One sweep (T steps + round trips) of the oracle on a 512 x 512 x `planes`
    sample of the workload; returns (cells*T, seconds)."""
    import oracle
    from paper_2109_05410_b200 import synth
    u = synth.dense(NX, NY, NZ, seed=1, z0=0, z1=planes)
    m = synth.layered(NX, NY, NZ, z0=0, z1=planes)
    t0 = time.perf_counter()
    oracle.advance(u, u, m, T, (RATE,) * 3, T)
    dt = time.perf_counter() - t0
    return NX * NY * planes * T, dt


def cpu_baseline(seconds: float = 15.0):
    """The oracle, as it stands, on the host cores: whole sweeps of the C2 grid
    (or a slab of it) until about `seconds` of CPU work have been timed."""
    import oracle
    oracle.build()
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    n, dt = _oracle_sweep_sample(64)                  # calibrate
    planes = int(max(16, min(NZ, (seconds * n / dt) / (NX * NY * T))) // 4 * 4)
    tot_n, tot_s, sweeps = 0, 0.0, 0
    while tot_s < seconds and sweeps < 8:
        n, dt = _oracle_sweep_sample(planes)
        tot_n += n
        tot_s += dt
        sweeps += 1
    return {"value": round(tot_n / tot_s, 1), "unit": "cell-updates/s", "cores": cores, "kind": "oracle",
            "sample": f"{sweeps} sweep(s) (T={T} steps + rate-{RATE} round trips each) of a {NX}x{NY}x{planes} "
                      f"slab of the C2 workload, {tot_s:.1f} s of oracle time"}


def reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    oracle.build()
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    planes = 32
    for _ in range(args.warmup):
        _oracle_sweep_sample(planes)
    tot_n, tot_s = 0, 0.0
    for _ in range(args.steps):
        n, dt = _oracle_sweep_sample(planes)
        tot_n += n
        tot_s += dt
    v = tot_n / tot_s
    sample = (f"each step: one sweep (T={T} steps + rate-{RATE} round trips) of a {NX}x{NY}x{planes} "
              f"slab of the C2 workload")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(v, 1), "unit": "cell-updates/s",
        "n_gpus": int(os.environ.get("WORLD_SIZE", "1")), "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(tot_s * 1e3 / args.steps, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"C2 sample: {NX}x{NY}x{planes} of the {NX}^3 grid, T={T}, rate {RATE}"},
        "cpu_baseline": {"value": round(v, 1), "unit": "cell-updates/s", "cores": cores, "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": round(v, 1), "unit": "cell-updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--quick", action="store_true", help="rate 16 and raw only")
    args = ap.parse_args()
    if args.warmup < 3:
        print("warning: --warmup < 3 is below the timing rules", file=sys.stderr)
    if args.impl == "reference":
        reference_arm(args)
    else:
        gpu_arm(args)


if __name__ == "__main__":
    main()
