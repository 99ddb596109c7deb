#!/usr/bin/env python3
"""Benchmark of the out-of-core compressed stencil stepper (arXiv 2109.05410).

One bench "step" = one sweep = T = 4 leapfrog steps over the whole grid
through the whole hot path (per z-block H2D / decode
-> 4 temporally blocked 25-point steps -> encode / D2H, region sharing,
separate copy / codec / stencil streams).

Headline workload (BASELINE.json configs[2]): a 4096 x 4096 x
1536 fp32 wavefield, previous wavefield and velocity model -- 309 GB of state,
more than the GPU's HBM and the host's RAM -- DENSE(seed 2) u, u- = u, LAYERED
m, streamed OUT OF CORE on one B200 at ZFP fixed rate 16 on all three fields
(a 154.6 GB pinned compressed store), T = 4.  Inputs are generated on the GPU
in plane chunks (synth.dense_torch / layered_torch, bit-identical to synth)
and compressed with oocz_set_field_planes; no full-size array ever exists.

  value : cell-updates/s = nx*ny*nz*T*K / device time of K sweeps, the store
          in pinned HOST memory: every sweep moves the compressed state over
          the host link (PCIe) inside the timed region.  Device-timed with CUDA
          events on the library's own streams (first enqueue -> join), max over
          ranks.  Schedule: the library's fastest orchestration of the same
          computation (serpentine sweeps + m decoded once into HBM + 3 staging
          slots, R22/R23; bit-identical results, tests).
  e2e   : the same K sweeps timed by the host wall clock around oocz_step
          (the public C ABI call), max over ranks.
  c3_paper_faithful : the paper's schedule (ascending sweeps, m streamed, P=192).
  zfp_vs_raw : the paper's question at the largest C3-shaped grid whose RAW
          store fits this host (4096 x 4096 x 768: 154.6 GB raw = the C3 rate-16
          store), both schedules, plus the error of the compressed run.
  c3_hbm_resident : the compressed C3 store held in HBM instead (no host link).
  c2 : the 512^3 configuration (configs[1]) -- HBM-resident and out-of-core,
          rates 8/16/24, the paper's codes 2-4 in fp32 and fp64, T = 8 / 12.

Multi-GPU (torchrun, N > 1; configs[3]): the same C3 grid
z-partitioned over N ranks (strong scaling), each rank streaming its own slab
out of core from its own pinned store, radius-4 halos exchanged in compressed
form with NCCL.

--impl reference: the CPU oracle (oracle/, test infrastructure) timed on the
host cores on a bounded sample of the same workload.
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
T = 4
RATE = 16
# C3 (configs[2])
C3N, C3Z, C3SEED = 4096, 1536, 2
# C2 (configs[1])
NX = NY = NZ = 512
P = 128


_T0 = time.perf_counter()


def log(msg: str) -> None:
    """Progress on stderr (the JSON line is the only stdout)."""
    print(f"[bench {time.perf_counter() - _T0:7.1f}s] {msg}", file=sys.stderr, flush=True)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            j = json.load(fh)
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed regions."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap,utilization.gpu")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.active = False
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out and self.active:
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
                "reasons": reasons, "samples": len(self.samples),
                "note": "sampled only while timed sweeps run (out-of-core sweeps leave the SMs partly idle)"}


def host_info() -> dict:
    """lscpu model, sockets, physical cores, and host RAM (for the oracle and the store)."""
    info = {"logical_cpus": os.cpu_count()}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        kv = {ln.split(":", 1)[0].strip(): ln.split(":", 1)[1].strip() for ln in out.splitlines() if ":" in ln}
        info["model"] = kv.get("Model name")
        sockets = int(kv.get("Socket(s)", "1") or 1)
        cps = int(kv.get("Core(s) per socket", "0") or 0)
        info["sockets"] = sockets
        info["physical_cores"] = sockets * cps if cps else None
        info["threads_per_core"] = int(kv.get("Thread(s) per core", "1") or 1)
        info["hypervisor"] = kv.get("Hypervisor vendor")
    except Exception:
        pass
    try:
        with open("/proc/meminfo") as fh:
            mi = {ln.split(":")[0]: int(ln.split()[1]) * 1024 for ln in fh}
        info["mem_total_bytes"] = mi.get("MemTotal")
        info["mem_available_bytes"] = mi.get("MemAvailable")
    except Exception:
        pass
    return info


def host_link_probe(nbytes: int = 1 << 30, reps: int = 6) -> dict:
    """Measured host-link peak (the out-of-core roofline's denominator):
    cudaMemcpyAsync H2D alone, D2H alone, and both at once on two streams (the
    pipeline's situation; each direction's rate from its own stream's elapsed
    time), CUDA events, best of `reps`.  The host buffers come from the same
    allocator as the store (oocz_host_alloc: THP pages registered with
    cudaHostRegister), so probe and pipeline copy the same kind of memory."""
    import torch
    from paper_2109_05410_b200 import oocz as Z
    try:
        from cuda.bindings import runtime as rt
    except ImportError:                    # older cuda-python layout
        from cuda import cudart as rt
    h_in, h_out = Z.oocz_host_alloc(nbytes), Z.oocz_host_alloc(nbytes)
    d_a = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    d_b = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    H2D, D2H = rt.cudaMemcpyKind.cudaMemcpyHostToDevice, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost

    def run(h2d: bool, d2h: bool):
        best = [0.0, 0.0]
        for _ in range(reps):
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e0.record(s1)
            s2.wait_event(e0)
            if h2d:
                rt.cudaMemcpyAsync(d_a.data_ptr(), h_in, nbytes, H2D, s1.cuda_stream)
            if d2h:
                rt.cudaMemcpyAsync(h_out, d_b.data_ptr(), nbytes, D2H, s2.cuda_stream)
            e1, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e1.record(s1)
            e2.record(s2)
            torch.cuda.synchronize()
            for i, e in enumerate((e1, e2)):
                best[i] = max(best[i], nbytes / (e0.elapsed_time(e) / 1e3) / 1e9)
        return best

    try:
        h2d_alone = run(True, False)[0]
        d2h_alone = run(False, True)[1]
        both = run(True, True)
    finally:
        Z.oocz_host_free(h_in)
        Z.oocz_host_free(h_out)
    return {"h2d_GBps": round(h2d_alone, 2), "d2h_GBps": round(d2h_alone, 2),
            "concurrent_h2d_GBps": round(both[0], 2), "concurrent_d2h_GBps": round(both[1], 2),
            "concurrent_per_direction_GBps": round(min(both), 2), "bytes": nbytes,
            "host_memory": "oocz_host_alloc (THP pages + cudaHostRegister), as the store"}


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


# DRAM bytes / algorithmic bytes per launch of each hot kernel, from the committed
# ncu --set full capture of the C3-wide launch shape (tools/ncu_r02.sh)
TRAFFIC_JSON = "r02g_stencil_c3_traffic.json"
TRAFFIC_KEY = {"stencil": "traffic_over_algorithmic", "decode": "zfp_decode_kernel", "encode": "zfp_encode_kernel"}
ALU_PEAK = 148 * 4 * 0.5 * 1.965   # G warp-instructions/s: ALU pipe, rt 2 cycles per SMSP (B300_MICROARCH)


def kernel_table(evs) -> dict:
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
    return per


def roofline(evs, peak_gbs, peak_src, force=None):
    """Dominant kernel of the timed region from its per-launch CUDA events
    (recorded on the stream each kernel is launched on): achieved =
    algorithmic bytes of all its launches / their summed duration."""
    per = kernel_table(evs)
    if not per:
        return None, {}
    dom = force if force in per else max(per, key=lambda k: per[k][0])
    ms, nbytes, n = per[dom]
    achieved = nbytes / (ms / 1e3) / 1e9
    table = {k: {"ms": round(v[0], 4), "launches": v[2], "GB/s": round(v[1] / (v[0] / 1e3) / 1e9, 1),
                 "avg_launch_ms": round(v[0] / v[2], 4)}
             for k, v in per.items()}
    if dom != "stencil" and not force:
        alu = _alu_roofline(dom, per[dom])
        if alu:
            return alu, table
    kern = {"stencil": "stencil25_kernel", "decode": "zfp_decode_kernel", "encode": "zfp_encode_kernel"}[dom]
    traffic, tsrc = None, None
    try:   # DRAM bytes per launch from a committed ncu capture of the same kind of launch
        with open(os.path.join(ROOT, "profiles", TRAFFIC_JSON)) as fh:
            ratio = float(json.load(fh)[TRAFFIC_KEY[dom]])
        traffic = int(ratio * nbytes / n)
        tsrc = (f"profiles/{TRAFFIC_JSON}: ncu dram read+write / algorithmic = {ratio} on a C3-wide "
                f"launch, x this run's algorithmic bytes per launch")
    except Exception:
        pass
    return {"bound": "hbm", "kernel": kern, "achieved": round(achieved, 1), "peak": peak_gbs,
            "peak_source": peak_src, "unit": "GB/s", "frac": round(achieved / peak_gbs, 4),
            "traffic": traffic, "traffic_source": tsrc, "avg_launch_ms": round(ms / n, 4),
            "launches": n, "algorithmic_bytes_per_launch": int(nbytes / n),
            "algorithmic_bytes": "stencil: 16 B per updated cell (read u, u-, m; write u+); decode / encode: "
                                 "compressed bytes + 4 B per value (DESIGN.md section 6)"}, table


def _alu_roofline(stage: str, rec) -> dict | None:
    """The dominant kernel is a codec kernel (with m decoded per block the decode
    leads the device time): it is bound by the integer ALU pipe, so its roofline is
    ALU-pipe warp-instructions per second.  Instructions per value come from the
    committed ncu capture of the C3-wide launch (profiles/r02g_ncu_kernels.json:
    ALU-pipe share x peak x duration / values); values per in-step launch from the
    launch's algorithmic bytes (compressed + 4 B per value at rate 16: 6 B/value)."""
    name = {"decode": "zfp_decode_kernel", "encode": "zfp_encode_kernel"}[stage]
    try:
        with open(os.path.join(ROOT, "profiles", "r02g_ncu_kernels.json")) as fh:
            ks = [k for k in json.load(fh)["c3_slab"]["kernels"] if k["kernel"].endswith(name)]
    except Exception:
        return None
    if not ks:
        return None
    k = ks[0]
    values = C3N * C3N * 96
    alu_per_value = k["alu_pipe_pct"] / 100.0 * ALU_PEAK * 1e9 * k["us"] * 1e-6 / values
    ms, nbytes, n = rec
    per_launch_values = nbytes / n / (4 + RATE / 8)
    achieved = alu_per_value * per_launch_values / (ms / n / 1e3) / 1e9
    return {"bound": "alu", "kernel": name, "achieved": round(achieved, 1), "peak": round(ALU_PEAK, 1),
            "peak_source": "148 SMs x 4 sub-partitions x one ALU-pipe warp-instruction per 2 cycles x 1.965 GHz "
                           "(B300_MICROARCH pipe rates; DESIGN.md section 6)",
            "unit": "G ALU-pipe warp-instructions/s", "frac": round(achieved / ALU_PEAK, 4),
            "traffic": None, "avg_launch_ms": round(ms / n, 4), "launches": n,
            "alu_instructions_per_value": round(alu_per_value * 32, 2),
            "what": "the dominant kernel of the step (most device time) is the decoder, bound by the integer "
                    "ALU pipe: ALU-pipe warp-instructions per value from ncu on the C3-wide launch "
                    "(profiles/r02g_ncu_kernels.json) x values per in-step launch / the in-step launch time "
                    "(CUDA events on the decode stream); the HBM-bound stencil's roofline is roofline_stencil"}


def codec_alu_roofline(table) -> dict | None:
    """The codec kernels are bound by the integer ALU pipe,
    not by HBM: their fraction is the ALU pipe's share of its peak issue rate
    (148 SMs x 4 sub-partitions x one warp-instruction per 2 cycles at 1965 MHz),
    measured by ncu (sm__inst_executed_pipe_alu) on the committed capture of the
    C3-wide launch shape (profiles/r02g_ncu_kernels.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02g_ncu_kernels.json")) as fh:
            kj = json.load(fh)["c3_slab"]
    except Exception:
        return None
    out = {}
    for name, stage in (("zfp_decode_kernel", "decode"), ("zfp_encode_kernel", "encode")):
        ks = [k for k in kj["kernels"] if k["kernel"].endswith(name)]
        if not ks:
            continue
        k = ks[0]
        frac = k["alu_pipe_pct"] / 100.0
        out[name] = {"bound": "alu", "achieved": round(frac * ALU_PEAK, 1), "peak": round(ALU_PEAK, 1),
                     "unit": "G ALU-pipe warp-instructions/s", "frac": round(frac, 4),
                     "issue_active": round(k["issue_active_pct"] / 100, 4), "isolated_us": k["us"],
                     "in_step_avg_ms": table[stage]["avg_launch_ms"] if stage in table else None,
                     "source": "profiles/r02g_ncu_kernels.json (ncu --set full, 4096^2 x 96-plane C3 slab, rate 16, round-2 codec)"}
    return out or None


def rel_errors(a: np.ndarray, b: np.ndarray, per_plane: int = 100, seed: int = 7) -> dict:
    """Compressed run `a` vs the uncompressed run `b` after the same steps
    (R18/R19): normwise max|a-b|/max|b| over the given
    planes, the paper's mean point-wise |a-b|/|b| over `per_plane` seeded points
    per plane (|b| < 1e-30 skipped), and the same over the points the wave has
    reached (|b| >= 1e-6 max|b|)."""
    from paper_2109_05410_b200 import synth
    a64, b64 = a.astype(np.float64), b.astype(np.float64)
    normwise = float(np.abs(a64 - b64).max() / max(np.abs(b64).max(), 1e-300))
    l2 = float(np.sqrt(np.sum((a64 - b64) ** 2)) / max(np.sqrt(np.sum(b64 ** 2)), 1e-300))
    nz, ny, nx = b.shape
    r = synth.uniforms(seed, 2 * per_plane * nz).reshape(nz, per_plane, 2)
    ys = (r[..., 0] * ny).astype(np.int64)
    xs = (r[..., 1] * nx).astype(np.int64)
    zs = np.repeat(np.arange(nz), per_plane).reshape(nz, per_plane)
    av, bv = a64[zs, ys, xs], b64[zs, ys, xs]
    keep = np.abs(bv) >= 1e-30
    mean_pw = float(np.mean(np.abs(av - bv)[keep] / np.abs(bv)[keep])) if keep.any() else 0.0
    sig = keep & (np.abs(bv) >= 1e-6 * np.abs(b64).max())
    mean_sig = float(np.mean(np.abs(av - bv)[sig] / np.abs(bv)[sig])) if sig.any() else 0.0
    return {"normwise_max": normwise, "l2": l2, "mean_pointwise": mean_pw, "points": int(keep.sum()),
            "skipped": int((~keep).sum()), "mean_pointwise_significant": mean_sig,
            "significant_points": int(sig.sum()), "vs": "same build, compression off (raw)"}


# ---------------------------------------------------------------- C3 / C4: out of core at scale
def set_fields_gpu(Z, ctx, nx, ny, nz, z_lo, S, seed, chunk=16):
    """Set this rank's slab [z_lo, z_lo + S) of DENSE(seed) (u and u-) and LAYERED
    (m), generated on the GPU chunk by chunk; returns seconds."""
    import torch
    from paper_2109_05410_b200 import synth
    t0 = time.perf_counter()
    for z0 in range(0, S, chunk):
        z1 = min(z0 + chunk, S)
        d = synth.dense_torch(nx, ny, nz, seed, z_lo + z0, z_lo + z1)
        Z.oocz_set_field_planes(ctx, Z.OOCZ_U, z0, d)
        Z.oocz_set_field_planes(ctx, Z.OOCZ_UPREV, z0, d)
        del d
        Z.oocz_set_field_planes(ctx, Z.OOCZ_M, z0, synth.layered_torch(nx, ny, nz, z_lo + z0, z_lo + z1))
    torch.cuda.synchronize()
    return time.perf_counter() - t0


def pick_P(S: int, prefer: int) -> int:
    for p in (prefer, 96, 64, 48, 32):
        if p <= S and S % p == 0 and p >= 8 * T:
            return p
    return S


def run_c3(Z, label, nx, ny, nz, rates, opt, arena, rank, world, nccl_id, device, steps, warmup, dist,
           profile=0, sample_planes=None):
    """One out-of-core (or HBM-resident) run on the C3-shaped grid: create (with
    the shared pinned arena), set fields on the GPU, W warm-up sweeps, K timed
    sweeps; device time (library events) and host wall time of the timed call,
    max over ranks."""
    import torch
    S = nz // world
    store = opt.get("store", 0)
    tb = opt.get("tb", T)
    def make_cfg(k=0, budget=0):
        return Z.oocz_default_config(nx, ny, nz, tb=tb, block_planes=opt["P"], rate=list(rates), store=store,
                                     m_resident=opt.get("m_resident", 0), serpentine=opt.get("serpentine", 0),
                                     slots=opt.get("slots", 2), slab_sets=opt.get("slab_sets", 0), profile=profile,
                                     cone=opt.get("cone", 0), resident_blocks=k, device_bytes=budget,
                                     m_hbm=opt.get("m_hbm", 0))
    cfg = make_cfg()
    if callable(nccl_id):
        nccl_id = nccl_id()
    torch.cuda.empty_cache()             # the generator's chunks: HBM for the context (C3 fills it)
    log(f"{label}: grid {nx}x{ny}x{nz} rates {list(rates)} {opt} W={warmup} K={steps}")
    t0 = time.perf_counter()
    resident = 0
    if opt.get("resident_blocks") == "max":
        # resident_blocks = -1: the library keeps as many z-blocks' compressed rows in
        # HBM as the budget allows (8 GiB left for the field generator); the rest must
        # fit the pinned arena
        budget = torch.cuda.mem_get_info(device)[0] - (8 << 30)
        ctx = Z.oocz_create_ex(make_cfg(-1, budget), rank, world, nccl_id, device, arena[0], arena[1])
        cfg = Z.oocz_get_config(ctx)
        resident = cfg.resident_blocks
    elif store == 0:
        ctx = Z.oocz_create_ex(cfg, rank, world, nccl_id, device, arena[0], arena[1])
    else:
        ctx = Z.oocz_create(cfg, rank, world, nccl_id, device)
    t_create = time.perf_counter() - t0
    try:
        # a compressed store in HBM leaves little room for the generator's fp64 chunks
        t_set = set_fields_gpu(Z, ctx, nx, ny, nz, rank * S, S, C3SEED, chunk=opt.get("gen_chunk", 16 if store == 0 else 4))
        Z.oocz_step(ctx, warmup * tb)
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        st0 = Z.oocz_get_stats(ctx)
        l0 = Z.oocz_kernel_launch_count()
        h0 = time.perf_counter()
        Z.oocz_step(ctx, steps * tb)         # returns when every stream is done
        host_s = time.perf_counter() - h0
        launches = Z.oocz_kernel_launch_count() - l0
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        st = Z.oocz_get_stats(ctx)
        dev_s = st["last_step_device_ms"] / 1e3
        if dist:
            from paper_2109_05410_b200 import dist as D
            dev_s = D.max_over_ranks(dist, dev_s, device="cuda")
            host_s = D.max_over_ranks(dist, host_s, device="cuda")
        sweeps = st["sweeps"] - st0["sweeps"]
        h2d = (st["h2d_bytes"] - st0["h2d_bytes"]) / max(sweeps, 1)
        d2h = (st["d2h_bytes"] - st0["d2h_bytes"]) / max(sweeps, 1)
        cells = nx * ny * nz * tb * steps
        res = {"label": label, "tb": tb, "grid": [nx, ny, nz], "rates": list(rates), "P": opt["P"], "D": S // opt["P"],
               "schedule": {k: v for k, v in opt.items() if k != "P"},
               "cups": cells / dev_s, "e2e_cups": cells / host_s, "device_s": dev_s, "host_s": host_s,
               "sweeps": steps, "warmup": warmup, "launches": launches,
               "h2d_per_sweep": h2d, "d2h_per_sweep": d2h, "halo_per_sweep": (st["halo_bytes"] - st0["halo_bytes"]) / max(sweeps, 1),
               "h2d_GBps": h2d * steps / dev_s / 1e9, "d2h_GBps": d2h * steps / dev_s / 1e9,
               "device_bytes": st["device_bytes_used"], "host_store_bytes": Z.oocz_host_store_bytes(cfg, world) if store == 0 else 0,
               "resident_blocks": resident, "create_s": round(t_create, 2), "set_fields_s": round(t_set, 2),
               "evs": Z.oocz_get_events(ctx) if profile else []}
        if sample_planes is not None:    # planes of u for the compressed-vs-raw error
            res["u_planes"] = np.concatenate([Z.oocz_get_field_planes(ctx, Z.OOCZ_U, z0, np.empty((4, ny, nx), np.float32))
                                              for z0 in sample_planes])
        log(f"{label}: {res['cups'] / 1e9:.1f} G cell-updates/s (host {res['e2e_cups'] / 1e9:.1f} G), "
            f"create {t_create:.1f} s, set {t_set:.1f} s")
        return res
    finally:
        Z.oocz_destroy(ctx)


def c3_arm(args, Z, rank, world, local, dist, nccl_id, peak_gbs, peak_src, link, clk, info):
    import torch
    nx = ny = C3N
    nz = C3Z
    S = nz // world
    # the pinned host store is allocated ONCE (pinning runs at ~2 GB/s) and reused by every
    # out-of-core run below: the largest is the rate-16 C3 store (= the raw 4096^2 x 768 one)
    cfg16 = Z.oocz_default_config(nx, ny, nz, tb=T, block_planes=pick_P(S, 64), rate=[RATE] * 3)
    need = Z.oocz_host_store_bytes(cfg16, world)
    raw_nz = nz // 2                                     # raw 4 B/value = 2 x rate 16
    t0 = time.perf_counter()
    log(f"pinning a {need / 1e9:.1f} GB host arena")
    arena_p = Z.oocz_host_alloc(need)
    arena = (arena_p, need)
    t_arena = time.perf_counter() - t0
    out = {"arena": {"bytes": need, "alloc_s": round(t_arena, 1)}}
    try:
        # m's compressed stream in HBM (m_hbm, decoded per block) instead of a decoded m, one
        # slab set (the device work, decode -> stencil -> encode in series, still fits in
        # the link time), and the HBM that frees as 20 output staging slots: 10 kept blocks
        # per serpentine turn.  They fill HBM to ~182 GB, so the field
        # generator works in 4-plane chunks; a box with less free HBM falls back to 16 slots
        # and two slab sets, then 12, then 4 with m decoded in HBM
        HS = dict(P=pick_P(S, 64), serpentine=1, m_hbm=1, slots=20, slab_sets=1, gen_chunk=4)
        PF = dict(P=pick_P(S, 192), serpentine=0, m_resident=0, slots=2, cone=1)
        clk.active = True
        fallbacks = []
        for hs in (HS, dict(HS, slots=16, slab_sets=0), dict(HS, slots=12, slab_sets=0),
                   dict(P=HS["P"], serpentine=1, m_resident=1, slots=4)):
            try:
                out["headline"] = run_c3(Z, "c3_zfp_host", nx, ny, nz, (RATE,) * 3, hs, arena, rank, world,
                                         nccl_id, local, args.steps, args.warmup, dist, profile=1)
                HS = hs
                break
            except Exception as e:
                if world > 1 or hs.get("slots") == 4:
                    raise
                log(f"c3_zfp_host {hs} failed ({type(e).__name__}: {str(e)[:120]}); next schedule")
                fallbacks.append(f"{hs}: {type(e).__name__}: {str(e)[:120]}")
                torch.cuda.empty_cache()
        if fallbacks:
            out["headline"]["fallback"] = fallbacks
        clk.active = False
        if world == 1 and not args.quick:
            sw, wu = args.sec_steps, 1
            clk.active = True
            out["pf"] = run_c3(Z, "c3_zfp_host_pf", nx, ny, nz, (RATE,) * 3, PF, arena, rank, world, nccl_id, local,
                               sw, wu, dist)
            # the paper's own temporal depth T = 12 on the same grid: a third of
            # the host bytes per step (P = 96: the slabs of h = 48 planes fit beside the staging)
            out["t12"] = run_c3(Z, "c3_zfp_host_t12", nx, ny, nz, (RATE,) * 3, dict(P=96, serpentine=1, slots=2, tb=12),
                                arena, rank, world, nccl_id, local, sw, wu, dist)
            # ZFP vs raw on the largest C3-shaped grid whose raw store fits this host
            planes = [0, raw_nz // 4, raw_nz // 2, 3 * raw_nz // 4 - 4, raw_nz - 4]
            HSr = dict(P=pick_P(raw_nz, 64), serpentine=1, m_resident=1, slots=4)   # (raw slots are twice the size)
            PFr = dict(PF, P=pick_P(raw_nz, 96))
            for key, rates, opt in (("half_zfp_hs", (RATE,) * 3, HSr), ("half_raw_hs", (0, 0, 0), HSr),
                                    ("half_zfp_pf", (RATE,) * 3, PFr), ("half_raw_pf", (0, 0, 0), PFr)):
                out[key] = run_c3(Z, key, nx, ny, raw_nz, rates, opt, arena, rank, world, nccl_id, local, sw, wu,
                                  dist, sample_planes=planes)
            # rate 24 on the full C3 grid: a 231.9 GB compressed store, more than this host's
            # RAM (and the arena); the rows of the first K z-blocks stay in HBM
            # (resident_blocks, the largest K that fits), the rest stream as usual
            try:
                out["r24_resident"] = run_c3(Z, "c3_r24_resident", nx, ny, nz, (24,) * 3,
                                             dict(P=pick_P(S, 64), serpentine=1, slots=2, resident_blocks="max"),
                                             arena, rank, world, nccl_id, local, sw, wu, dist)
            except Exception as e:       # a secondary number: report, do not lose the headline
                out["r24_resident"] = {"error": f"{type(e).__name__}: {e}"[:300]}
            clk.active = False
    finally:
        Z.oocz_host_free(arena_p)
    if not args.quick:
        # the compressed C3 store held in HBM (154.6 GB, or its 1/world share per GPU)
        # beside one slab set (two when z-split: the share leaves room): no host link.
        # With world >= 2 the per-GPU share fits HBM, so the out-of-core headline is a
        # forced mode there and this is the in-HBM number beside it.
        clk.active = True
        try:
            out["hbm"] = run_c3(Z, "c3_zfp_dev", nx, ny, nz, (RATE,) * 3,
                                dict(P=96, store=1, slab_sets=1 if world == 1 else 2), None,
                                rank, world, nccl_id, local, args.sec_steps, 1, dist)
        except Exception as e:            # a secondary number: report, do not lose the headline
            out["hbm_error"] = f"{type(e).__name__}: {e}"[:300]
        clk.active = False
    torch.cuda.empty_cache()
    return out


def paper_problem(Z, device, sweeps: int = 2, warmup: int = 1) -> dict:
    """The paper's own experiment on this GPU: PAPER.md:182-192 (Table I: 1152^3
    points, fp64), :208-217 (T = 12, 8 divisions), :212-215 (codes 1-4), the
    paper's schedule (ascending sweeps, m streamed, the trapezoid cone) out of
    core from pinned host memory; speedup of each code vs code 1 and its error,
    next to the paper's 1.16x / 1.18x / 1.20x on V100-PCIe.
    Inputs DENSE(1) + LAYERED in fp64, generated on the GPU."""
    import torch
    from paper_2109_05410_b200 import synth
    n, tb, P = 1152, 12, 144
    sample = [0, n // 4, n // 2, 3 * n // 4 - 4, n - 4]
    out = {"what": "the paper's problem (1152^3 fp64, T = 12, P = 144: 8 z-blocks, its codes 1-4, its schedule), "
                   "out of core; speedup vs code 1 (the paper: 1.16x / 1.18x / 1.20x, V100-PCIe, PAPER.md:227)",
           "sweeps": sweeps, "warmup": warmup}
    ref = None
    for key, rates in (("1_original", (0, 0, 0)), ("2_rw_32", (0, 32, 0)), ("3_ro_32", (0, 0, 32)),
                       ("4_rw_ro_24", (0, 24, 24))):
        cfg = Z.oocz_default_config(n, n, n, tb=tb, block_planes=P, rate=list(rates), store=0, precision=64,
                                    serpentine=0, m_resident=0, slots=2, cone=1)
        log(f"paper problem {key}")
        ctx = Z.oocz_create(cfg, 0, 1, None, device)
        try:
            for z0 in range(0, n, 16):
                d = synth.dense_torch(n, n, n, 1, z0, z0 + 16, fp64=True)
                Z.oocz_set_field_planes(ctx, Z.OOCZ_U, z0, d)
                Z.oocz_set_field_planes(ctx, Z.OOCZ_UPREV, z0, d)
                del d
                Z.oocz_set_field_planes(ctx, Z.OOCZ_M, z0, synth.layered_torch(n, n, n, z0, z0 + 16, fp64=True))
            Z.oocz_step(ctx, tb * warmup)
            torch.cuda.synchronize()
            s0 = Z.oocz_get_stats(ctx)
            h0 = time.perf_counter()
            Z.oocz_step(ctx, tb * sweeps)
            host_s = time.perf_counter() - h0
            st = Z.oocz_get_stats(ctx)
            dev_s = st["last_step_device_ms"] / 1e3
            cells = n ** 3 * tb * sweeps
            u = np.concatenate([Z.oocz_get_field_planes(ctx, Z.OOCZ_U, z0, np.empty((4, n, n), np.float64))
                                for z0 in sample])
            row = {"rates": list(rates), "value": round(cells / dev_s, 1), "e2e": round(cells / host_s, 1),
                   "h2d_bytes_per_sweep": (st["h2d_bytes"] - s0["h2d_bytes"]) // sweeps,
                   "d2h_bytes_per_sweep": (st["d2h_bytes"] - s0["d2h_bytes"]) // sweeps}
        finally:
            Z.oocz_destroy(ctx)
        if ref is None:
            ref = (row, u)
        else:
            err = rel_errors(u, ref[1])
            row["speedup"] = round(row["value"] / ref[0]["value"], 3)
            row["normwise_max_rel_error"] = err["normwise_max"]
            row["mean_pointwise_rel_error"] = err["mean_pointwise_significant"]
        out[key] = row
    return out


def Z_ROWS(grid, rate, esz=4):
    """bytes of one field's fixed-rate stream on grid (nx, ny, nz): 8 * rate per 4^3 block"""
    nx, ny, nz = grid
    return (nx // 4) * (ny // 4) * (nz // 4) * 8 * rate if rate else nx * ny * nz * esz


def c3_report(c3, args, world, link, peak_gbs, peak_src, info):
    h = c3["headline"]
    roof, table = roofline(h["evs"], peak_gbs, peak_src)
    # the binding direction: the one whose bytes per sweep take longest at its own
    # measured rate with both directions busy (the roof is that time per sweep)
    t_dir = {d: h[f"{d}_per_sweep"] / (link[f"concurrent_{d}_GBps"] * 1e9) for d in ("h2d", "d2h")}
    bound_dir = max(t_dir, key=t_dir.get)
    busier = h[f"{bound_dir}_per_sweep"]
    link_peak = link[f"concurrent_{bound_dir}_GBps"]
    rep = {
        "value": round(h["cups"], 1),
        "ms_per_step": round(h["device_s"] * 1e3 / args.steps, 3),
        "e2e": {"value": round(h["e2e_cups"], 1), "unit": "cell-updates/s",
                "h2d_bytes_per_step": int(h["h2d_per_sweep"]), "d2h_bytes_per_step": int(h["d2h_per_sweep"]),
                "path": "host wall clock around oocz_step (the public C ABI) over the K timed sweeps; the "
                        "compressed store is in pinned host memory, so each sweep's H2D of the state and D2H "
                        "of the updated read-write fields are inside the call",
                "ms_per_step": round(h["host_s"] * 1e3 / args.steps, 3)},
        "roofline": roof,
        "roofline_stencil": roofline(h["evs"], peak_gbs, peak_src, force="stencil")[0],
        "roofline_host_link": {
            "bound": "host-link", "direction": bound_dir,
            "achieved": round(busier * args.steps / h["device_s"] / 1e9, 2),
            "peak": link_peak, "unit": "GB/s",
            "frac": round(busier * args.steps / h["device_s"] / 1e9 / link_peak, 4),
            "h2d_GBps": round(h["h2d_GBps"], 2), "d2h_GBps": round(h["d2h_GBps"], 2),
            "peak_source": "measured in this run: pinned H2D and D2H at once on two streams (host_link_probe)",
            "what": "the out-of-core roofline (SURVEY 8(d)): of H2D and D2H, the direction whose bytes per "
                    "sweep take longest at its measured rate with both directions busy binds; achieved = its "
                    "bytes per sweep / sweep time, peak = its measured rate",
            "host_link_probe": link},
        "kernels_in_step": table,
        "codec_alu_roofline": codec_alu_roofline(table),
        "lanes": lanes_summary(h["evs"]),
        "gpu_launches": int(h["launches"]),
        "headline_run": {k: (round(v, 4) if isinstance(v, float) else v) for k, v in h.items()
                         if k not in ("evs", "u_planes")},
    }
    if "pf" in c3:
        pf = c3["pf"]
        rep["c3_paper_faithful"] = {
            "value": round(pf["cups"], 1), "e2e": round(pf["e2e_cups"], 1), "P": pf["P"], "D": pf["D"],
            "h2d_bytes_per_step": int(pf["h2d_per_sweep"]), "d2h_bytes_per_step": int(pf["d2h_per_sweep"]),
            "h2d_GBps": round(pf["h2d_GBps"], 2), "d2h_GBps": round(pf["d2h_GBps"], 2),
            "sweeps": pf["sweeps"],
            "schedule": "the paper's: ascending sweeps, m streamed and decoded every sweep, the trapezoid cone "
                        "(cone = 1), 2 staging slots",
            "headline_over_paper_faithful": round(h["cups"] / pf["cups"], 3)}
    if "t12" in c3:
        t = c3["t12"]
        rep["c3_paper_T12"] = {"value": round(t["cups"], 1), "e2e": round(t["e2e_cups"], 1), "tb": 12, "P": t["P"],
                               "D": t["D"], "h2d_bytes_per_step": int(t["h2d_per_sweep"]),
                               "d2h_bytes_per_step": int(t["d2h_per_sweep"]),
                               "h2d_GBps": round(t["h2d_GBps"], 2), "d2h_GBps": round(t["d2h_GBps"], 2),
                               "schedule": "serpentine, m streamed, 2 slots; one step = one sweep of 12 leapfrog steps",
                               "what": "the paper's temporal blocking depth (PAPER.md:217, T = 12) on the C3 grid: "
                                       "a third of the host bytes per cell-update of T = 4"}
    if "half_raw_pf" in c3:
        zr = {"grid": c3["half_raw_pf"]["grid"],
              "why": "the full C3 raw store (3 x 103.1 GB = 309.2 GB) cannot exist on this host "
                     f"(RAM {info.get('mem_total_bytes', 0) / 1e9:.1f} GB); 4096 x 4096 x 768 is the largest C3-shaped "
                     "grid whose raw store (154.6 GB) fits, the same bytes as the C3 rate-16 store",
              "c3_raw_store_bytes": 3 * C3N * C3N * C3Z * 4, "host_mem_bytes": info.get("mem_total_bytes")}
        for sched, zk, rk in (("headline_schedule", "half_zfp_hs", "half_raw_hs"),
                              ("paper_faithful", "half_zfp_pf", "half_raw_pf")):
            z, r = c3[zk], c3[rk]
            err = rel_errors(z["u_planes"], r["u_planes"])
            err["planes"] = "u after the same steps, 5 block-rows spread over z (100 seeded points per plane)"
            zr[sched] = {"zfp": round(z["cups"], 1), "raw": round(r["cups"], 1),
                         "speedup": round(z["cups"] / r["cups"], 3),
                         "zfp_e2e": round(z["e2e_cups"], 1), "raw_e2e": round(r["e2e_cups"], 1),
                         "zfp_h2d_bytes_per_step": int(z["h2d_per_sweep"]),
                         "raw_h2d_bytes_per_step": int(r["h2d_per_sweep"]),
                         "zfp_h2d_GBps": round(z["h2d_GBps"], 2), "raw_h2d_GBps": round(r["h2d_GBps"], 2),
                         "P": z["P"], "steps": (z["sweeps"] + z["warmup"]) * T, "max_rel_error": err}
        zr["paper_context"] = "1.20x (fp64, mode 4, V100-PCIe 3.0, PAPER.md:227)"
        rep["zfp_vs_raw"] = zr
    if "r24_resident" in c3:
        r = c3["r24_resident"]
        if "error" in r:
            rep["c3_rate24_resident_blocks"] = r
        else:
            store = 3 * Z_ROWS(r["grid"], 24)
            rep["c3_rate24_resident_blocks"] = {
                "value": round(r["cups"], 1), "e2e": round(r["e2e_cups"], 1), "rates": r["rates"], "P": r["P"],
                "D": r["D"], "resident_blocks": r["resident_blocks"], "compressed_store_bytes": store,
                "host_store_bytes": r["host_store_bytes"], "host_mem_bytes": info.get("mem_total_bytes"),
                "h2d_bytes_per_step": int(r["h2d_per_sweep"]), "d2h_bytes_per_step": int(r["d2h_per_sweep"]),
                "h2d_GBps": round(r["h2d_GBps"], 2), "d2h_GBps": round(r["d2h_GBps"], 2), "sweeps": r["sweeps"],
                "what": "C3 at rate 24 on all three fields: the compressed store exceeds this host's RAM, so it "
                        "runs only with the rows of the first resident_blocks z-blocks kept in HBM "
                        "(cfg.resident_blocks = -1: the largest split that fits) and the rest streamed; serpentine, "
                        "m streamed, 2 slots"}
    if "hbm_error" in c3:
        rep["c3_hbm_resident"] = {"error": c3["hbm_error"]}
    if "hbm" in c3:
        d = c3["hbm"]
        rep["c3_hbm_resident"] = {"value": round(d["cups"], 1), "P": d["P"],
                                  "slab_sets": d["schedule"].get("slab_sets"),
                                  "device_bytes": d["device_bytes"], "sweeps": d["sweeps"],
                                  "what": "the same C3 problem with the 154.6 GB compressed store held in HBM "
                                          "(store = device; per GPU its 1/n_gpus share when z-split): decode -> "
                                          "stencil -> encode per block, no host link" +
                                          ("; the share fits HBM, so the out-of-core headline is a forced mode "
                                           "at this GPU count (SURVEY 8(d) C4)" if world > 1 else "")}
    return rep


# ---------------------------------------------------------------- C2 (configs[1]): 512^3
def make_fields_c2():
    from paper_2109_05410_b200 import synth
    u = synth.dense(NX, NY, NZ, seed=1)
    m = synth.layered(NX, NY, NZ)
    return u, u, m


def run_mode_c2(Z, store, rates, fields, device, steps, warmup, profile, m_resident=0, tb=T, precision=32,
                serpentine=0, slots=2, slab_sets=0, cone=0, block_planes=P, graphs=0):
    """Returns (device seconds for `steps` sweeps, stats, events, launches, ctx)."""
    import torch
    cfg = Z.oocz_default_config(NX, NY, NZ, tb=tb, block_planes=block_planes, rate=list(rates), store=store,
                                m_resident=m_resident, precision=precision, serpentine=serpentine,
                                slots=slots, profile=profile, slab_sets=slab_sets, cone=cone, graphs=graphs)
    ctx = Z.oocz_create(cfg, 0, 1, None, device)
    try:
        for f, a in zip((Z.OOCZ_U, Z.OOCZ_UPREV, Z.OOCZ_M), fields):
            Z.oocz_set_field(ctx, f, a.astype(np.float64) if precision == 64 else a)
        Z.oocz_step(ctx, warmup * tb)
        torch.cuda.synchronize()
        st0 = Z.oocz_get_stats(ctx)
        l0 = Z.oocz_kernel_launch_count()
        Z.oocz_step(ctx, steps * tb)
        launches = Z.oocz_kernel_launch_count() - l0
        st = Z.oocz_get_stats(ctx)
        for k in ("sweeps", "h2d_bytes", "d2h_bytes", "halo_bytes"):
            st[k] -= st0[k]
        evs = Z.oocz_get_events(ctx) if profile else []
        return st["last_step_device_ms"] / 1e3, st, evs, launches, ctx
    except Exception:
        Z.oocz_destroy(ctx)
        raise


def in_core_c2(Z, fields, steps, warmup, ref_u, peak_gbs) -> dict:
    """C2 in core (BASELINE configs[1] "in-core vs compressed-transit"): raw u, u-, m
    resident in HBM, stepped by the stateless leapfrog entry point (one stencil
    launch per step over all 512 planes: no z-blocks, no codec, no copies).  The
    same (warmup + steps) x T steps as the engine's raw run, whose u it must equal
    bit for bit (the block schedule computes the in-core leapfrog)."""
    import torch
    u = torch.from_numpy(np.ascontiguousarray(fields[0])).cuda()
    up = torch.from_numpy(np.ascontiguousarray(fields[1])).cuda()
    m = torch.from_numpy(np.ascontiguousarray(fields[2])).cuda()
    s = torch.cuda.current_stream()
    c = Z.default_coeffs()
    Z.oocz_stencil_steps(u, up, m, NX, NY, NZ, c, warmup * T, s)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    l0 = Z.oocz_kernel_launch_count()
    a.record(s)
    Z.oocz_stencil_steps(u, up, m, NX, NY, NZ, c, steps * T, s)
    b.record(s)
    torch.cuda.synchronize()
    t = a.elapsed_time(b) / 1e3
    upd = NX * NY * NZ * steps * T
    got = u.cpu().numpy()
    return {"value": round(upd / t, 1), "steps": steps * T, "launches": Z.oocz_kernel_launch_count() - l0,
            "achieved_GBps": round(16 * upd / t / 1e9, 1), "hbm_frac": round(16 * upd / t / 1e9 / peak_gbs, 4),
            "bit_identical_to_engine_raw": bool(np.array_equal(got.view(np.uint32), ref_u.view(np.uint32))),
            "what": "raw fields in HBM stepped by oocz_stencil_steps (16 B per cell-update); the compressed "
                    "paths' value_hbm_resident is set against this; hbm_frac is against the 1:1 copy peak, "
                    "which the stencil's 3:1 read:write mix can exceed"}


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


def c2_arm(args, Z, device, peak_gbs, peak_src, link, clk):
    fields = make_fields_c2()
    steps, warmup = args.c2_steps, 3
    cells = NX * NY * NZ * T * steps
    OD = dict(m_resident=1)
    OH = dict(serpentine=1, m_resident=1, slots=4)   # (4 slots: 67 vs 64 G, profiles/r02_c2_slots.txt)
    PF = dict(serpentine=0, m_resident=0, cone=1)
    modes = [("zfp_dev", 1, (RATE,) * 3, OD), ("zfp_host", 0, (RATE,) * 3, OH),
             ("raw_dev", 1, (0, 0, 0), OD), ("raw_host", 0, (0, 0, 0), OH)]
    if not args.quick:
        modes += [(f"r{r}_{k}", st, (r,) * 3, o) for r in (8, 24) for k, st, o in (("dev", 1, OD), ("host", 0, OH))]
        modes += [("pf_zfp_dev", 1, (RATE,) * 3, PF), ("pf_zfp_host", 0, (RATE,) * 3, PF),
                  ("pf_raw_dev", 1, (0, 0, 0), PF), ("pf_raw_host", 0, (0, 0, 0), PF)]
        # the paper's codes 2-4 as fp32 rate vectors, out of core,
        # paper-faithful schedule: one read-write field (u-, reading R7/R25) at 16/32,
        # the read-only m at 16/32, one read-write field + m at 12/32 (the paper's 24/64)
        modes += [("pm2_host", 0, (0, 16, 0), PF), ("pm3_host", 0, (0, 0, 16), PF),
                  ("pm4_host", 0, (0, 12, 12), PF)]
        modes += [(f"t{t}_{k}", st, (RATE,) * 3, dict(o, tb=t)) for t in (8, 12)
                  for k, st, o in (("dev", 1, OD), ("host", 0, OH))]
        F = dict(PF, precision=64)
        modes += [("f64raw_host", 0, (0, 0, 0), F), ("f64pm2_host", 0, (0, 32, 0), F),
                  ("f64pm3_host", 0, (0, 0, 32), F), ("f64pm4_host", 0, (0, 24, 24), F),
                  ("f64all_host", 0, (32, 32, 32), F), ("f64all_dev", 1, (32, 32, 32), F),
                  ("f64raw_dev", 1, (0, 0, 0), F),
                  ("f64allo_host", 0, (32, 32, 32), dict(OH, precision=64)),
                  ("f64allo_dev", 1, (32, 32, 32), dict(OD, precision=64))]
    out = {}
    for label, store, rates, opt in modes:
        log(f"c2 {label}")
        tb = opt.get("tb", T)
        prec = opt.get("precision", 32)
        clk.active = True
        dev_s, st, evs, launches, ctx = run_mode_c2(Z, store, rates, fields, device, steps, warmup,
                                                    profile=int(label == "zfp_dev"),
                                                    m_resident=opt.get("m_resident", 0), tb=tb, precision=prec,
                                                    serpentine=opt.get("serpentine", 0), slots=opt.get("slots", 2),
                                                    slab_sets=opt.get("slab_sets", 0), cone=opt.get("cone", 0))
        clk.active = False
        sw = max(st["sweeps"], 1)
        out[label] = {"s": dev_s, "cups": cells // T * tb / dev_s, "launches": launches, "evs": evs,
                      "h2d_per_sweep": st["h2d_bytes"] / sw, "d2h_per_sweep": st["d2h_bytes"] / sw}
        if store == 1 or "pm" in label or label.startswith("f64") or label.endswith("raw_host"):
            out[label]["u"] = Z.oocz_get_field(ctx, Z.OOCZ_U, np.empty((NZ, NY, NX),
                                                                       np.float64 if prec == 64 else np.float32))
        Z.oocz_destroy(ctx)
    roof, table = roofline(out["zfp_dev"]["evs"], peak_gbs, peak_src)
    err = rel_errors(out["zfp_dev"]["u"], out["raw_dev"]["u"])
    err["steps"] = (warmup + steps) * T
    v, e = out["zfp_dev"], out["zfp_host"]
    rep = {"workload": f"C2: {NX}^3 fp32, DENSE(1) + LAYERED, P={P} ({NZ // P} z-blocks), T={T}",
           "steps": steps, "warmup": warmup,
           "value_hbm_resident": round(v["cups"], 1),
           "e2e_out_of_core": round(e["cups"], 1),
           "e2e_host_link_frac": round(max(e[f"{d}_per_sweep"] / (link[f"concurrent_{d}_GBps"] * 1e9)
                                           for d in ("h2d", "d2h")) / (e["s"] / steps), 4),
           "e2e_h2d_bytes_per_step": int(e["h2d_per_sweep"]), "e2e_d2h_bytes_per_step": int(e["d2h_per_sweep"]),
           "raw": {"value_hbm_resident": round(out["raw_dev"]["cups"], 1), "e2e": round(out["raw_host"]["cups"], 1)},
           "speedup_zfp_vs_raw": {"hbm_resident": round(v["cups"] / out["raw_dev"]["cups"], 3),
                                  "out_of_core": round(e["cups"] / out["raw_host"]["cups"], 3)},
           "max_rel_error": err,
           "in_core": in_core_c2(Z, fields, steps, warmup, out["raw_dev"]["u"], peak_gbs),
           "roofline_in_step": roof, "kernels_in_step": table, "lanes": lanes_summary(v["evs"]),
           "schedule": "HBM-resident: m_resident=1; out of core: serpentine=1, m_resident=1, slots=4"}
    if "pf_raw_host" in out:
        rep["paper_faithful"] = {"value_hbm_resident": round(out["pf_zfp_dev"]["cups"], 1),
                                 "e2e_out_of_core": round(out["pf_zfp_host"]["cups"], 1),
                                 "raw_e2e": round(out["pf_raw_host"]["cups"], 1),
                                 "speedup_out_of_core": round(out["pf_zfp_host"]["cups"] / out["pf_raw_host"]["cups"], 3)}
        ref = out["pf_raw_host"]
        pm = {"what": "PAPER.md:212-215 codes as rate vectors (u, u-, m); out of core; speedup vs code 1 "
                      "(the paper: 1.16x / 1.18x / 1.20x, fp64, V100-PCIe); the one read-write dataset is u- "
                      "(reading R25)", "1_original": {"rates": [0, 0, 0], "e2e": round(ref["cups"], 1)}}
        for key, lab, rates in (("2_rw_16", "pm2_host", [0, 16, 0]), ("3_ro_16", "pm3_host", [0, 0, 16]),
                                ("4_rw_ro_12", "pm4_host", [0, 12, 12])):
            er = rel_errors(out[lab]["u"], ref["u"])
            pm[key] = {"rates": rates, "e2e": round(out[lab]["cups"], 1),
                       "speedup": round(out[lab]["cups"] / ref["cups"], 3),
                       "normwise_max_rel_error": er["normwise_max"], "mean_pointwise_rel_error": er["mean_pointwise"]}
        rep["paper_modes"] = pm
        ref = out["f64raw_host"]
        pf64 = {"what": "the paper's precision and rates (fp64; PAPER.md:208, :212-215): codes 1-4 out of core and "
                        "every field at 32/64; speedup vs code 1 (the paper: 1.16x / 1.18x / 1.20x, V100-PCIe)",
                "1_original": {"rates": [0, 0, 0], "e2e": round(ref["cups"], 1),
                               "value": round(out["f64raw_dev"]["cups"], 1)}}
        for key, lab, rates in (("2_rw_32", "f64pm2_host", [0, 32, 0]), ("3_ro_32", "f64pm3_host", [0, 0, 32]),
                                ("4_rw_ro_24", "f64pm4_host", [0, 24, 24]), ("all_32", "f64all_host", [32, 32, 32])):
            er = rel_errors(out[lab]["u"], ref["u"])
            pf64[key] = {"rates": rates, "e2e": round(out[lab]["cups"], 1),
                         "speedup": round(out[lab]["cups"] / ref["cups"], 3),
                         "normwise_max_rel_error": er["normwise_max"], "mean_pointwise_rel_error": er["mean_pointwise"]}
        pf64["all_32"]["value"] = round(out["f64all_dev"]["cups"], 1)
        pf64["all_32_orchestrated"] = {"e2e": round(out["f64allo_host"]["cups"], 1),
                                       "value": round(out["f64allo_dev"]["cups"], 1)}
        rep["paper_precision_fp64"] = pf64
        rep["other_rates"] = {}
        for r in (8, 24):
            er = rel_errors(out[f"r{r}_dev"]["u"], out["raw_dev"]["u"])
            rep["other_rates"][str(r)] = {"value_hbm_resident": round(out[f"r{r}_dev"]["cups"], 1),
                                          "e2e": round(out[f"r{r}_host"]["cups"], 1),
                                          "normwise_max_rel_error": er["normwise_max"]}
        rep["temporal_blocking"] = {f"T={t}": {"value_hbm_resident": round(out[f"t{t}_dev"]["cups"], 1),
                                               "e2e": round(out[f"t{t}_host"]["cups"], 1)} for t in (8, 12)}
        rep["roofline_isolated"] = isolated_kernels(Z, fields, peak_gbs)
    return rep


# ---------------------------------------------------------------- GPU arm
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
    peak_gbs, peak_src = peaks()
    info = host_info()
    if dist:                     # all ranks probe their host links at the same time (shared PCIe / memory)
        dist.barrier()
    link = host_link_probe()
    if dist:
        for k in ("h2d_GBps", "d2h_GBps", "concurrent_h2d_GBps", "concurrent_d2h_GBps", "concurrent_per_direction_GBps"):
            link[k] = -D.max_over_ranks(dist, -link[k], device="cuda")      # the slowest rank's link
        link["ranks"] = world
        link["note"] = "all ranks probing at once; the minimum over ranks"
    with ClockSampler(local) as clk:
        c3 = c3_arm(args, Z, rank, world, local, dist, nccl_id, peak_gbs, peak_src, link, clk, info)
        c2 = c2_arm(args, Z, local, peak_gbs, peak_src, link, clk) if world == 1 and not args.no_c2 else None
        pp = None
        if world == 1 and not args.quick and not args.no_paper:
            try:
                pp = paper_problem(Z, local)
            except Exception as e:          # a context number: report, do not lose the headline
                pp = {"error": f"{type(e).__name__}: {e}"[:300]}
    clocks = clk.summary()
    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    rep = c3_report(c3, args, world, link, peak_gbs, peak_src, info)
    h = c3["headline"]
    line = {
        "metric": METRIC,
        "value": rep["value"],
        "unit": "cell-updates/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": rep["ms_per_step"],
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic, generated on the GPU (DENSE seed 2 wavefield, u- = u, LAYERED m; SURVEY 8(d))",
        "config": {"workload": f"C3{' (C4: z-split over %d GPUs)' % world if world > 1 else ''}: "
                               f"{C3N}x{C3N}x{C3Z} fp32 u, u-, m (309.2 GB raw) out of core, ZFP rate {RATE} on all "
                               f"three fields (154.6 GB pinned host store), T={T}, P={h['P']} ({h['D']} z-blocks"
                               f"{' per GPU' if world > 1 else ''})",
                   "grid": [C3N, C3N, C3Z], "tb": T, "block_planes": h["P"], "rate": RATE,
                   "schedule": f"serpentine sweeps + m {'compressed in HBM' if h['schedule'].get('m_hbm') else 'decoded once into HBM'}"
                               f" + {h['schedule'].get('slots')} output staging slots, kept blocks at the turns (the library's fastest "
                               "schedule of the same computation, bit-identical to the paper's; the paper's own: "
                               "c3_paper_faithful)",
                   "step": "one sweep = T leapfrog steps over the whole grid",
                   "l2": "inputs larger than L2 (the state is 154.6 GB; each sweep streams all of it)",
                   "parallelism": f"z-slabs x{world}, NCCL compressed halos" if world > 1 else "single GPU"},
        "e2e": rep["e2e"],
        "roofline": rep["roofline"],
        "roofline_stencil": rep["roofline_stencil"],
        "roofline_host_link": rep["roofline_host_link"],
        "gpu_launches": rep["gpu_launches"],
        "kernels_in_step": rep["kernels_in_step"],
        "roofline_codec": rep["codec_alu_roofline"],
        "lanes": rep["lanes"],
        "zfp_vs_raw": rep.get("zfp_vs_raw"),
        "c3_paper_faithful": rep.get("c3_paper_faithful"),
        "c3_paper_T12": rep.get("c3_paper_T12"),
        "c3_hbm_resident": rep.get("c3_hbm_resident"),
        "c3_rate24_resident_blocks": rep.get("c3_rate24_resident_blocks"),
        "c3_arena": c3["arena"],
        "headline_run": rep["headline_run"],
        "c2": c2,
        "paper_problem": pp,
        "host": info,
        "clocks": clocks,
    }
    if world == 1 and not args.no_cpu_baseline:
        log("cpu baseline")
        line["cpu_baseline"] = cpu_baseline(seconds=args.cpu_seconds, info=info)
    print(json.dumps(line))
    if dist:
        dist.destroy_process_group()


# ---------------------------------------------------------------- CPU oracle arm
def _oracle_sweep_sample(planes: int, nx: int = C3N, ny: int = 64, z0: int = 0):
    """One sweep (T steps + rate-16 round trips) of the oracle on an nx x ny x
    `planes` box of the C3 workload (DENSE(2), LAYERED); returns (cells*T, s)."""
    import oracle
    from paper_2109_05410_b200 import synth
    u = synth.dense(nx, ny, C3Z, seed=C3SEED, z0=z0, z1=z0 + planes, y0=0, y1=ny, x0=0, x1=nx)
    m = synth.layered(nx, ny, C3Z, z0=z0, z1=z0 + planes, y0=0, y1=ny, x0=0, x1=nx)
    t0 = time.perf_counter()
    oracle.advance(u, u, m, T, (RATE,) * 3, T)
    dt = time.perf_counter() - t0
    return nx * ny * planes * T, dt


def _oracle_timed(planes: int, seconds: float, max_sweeps: int = 16) -> dict:
    n_tot, s_tot, k = 0, 0.0, 0
    while s_tot < seconds and k < max_sweeps:
        n, dt = _oracle_sweep_sample(planes)
        n_tot += n
        s_tot += dt
        k += 1
    return {"n": n_tot, "s": s_tot, "sweeps": k}


def _oracle_c1_c2() -> dict:
    """C1 whole (64^3, PULSE(4) + LAYERED, P = 32, T = 2, rate 16, 10 steps: the
    oracle's reduced schedule) and one sweep of a 512 x 512 x 32 box of C2
    (DENSE(1) + LAYERED, T = 4, rate 16), timed in this process."""
    import oracle
    from paper_2109_05410_b200 import synth
    n = 64
    u, m = synth.pulse(n, n, n, sigma=4.0), synth.layered(n, n, n)
    t0 = time.perf_counter()
    oracle.advance(u, u, m, 2, (RATE,) * 3, 10)
    c1 = time.perf_counter() - t0
    u = synth.dense(512, 512, 512, seed=1, z0=0, z1=32)
    m = synth.layered(512, 512, 512, z0=0, z1=32)
    t0 = time.perf_counter()
    oracle.advance(u, u, m, T, (RATE,) * 3, T)
    c2 = time.perf_counter() - t0
    return {"c1": {"value": round(n ** 3 * 10 / c1, 1), "seconds": round(c1, 3)},
            "c2_sample": {"value": round(512 * 512 * 32 * T / c2, 1), "seconds": round(c2, 3)}}


def _oracle_subprocess(threads: int, seconds: float, planes: int) -> dict:
    """The oracle in a fresh process with OMP_NUM_THREADS = threads (its stencil
    loops are OpenMP; the codec round trips are serial C)."""
    env = dict(os.environ, OMP_NUM_THREADS=str(threads))
    out = subprocess.run([sys.executable, os.path.abspath(__file__), "--oracle-sample", str(seconds),
                          "--oracle-planes", str(planes)], capture_output=True, text=True, env=env,
                         timeout=600 + 4 * seconds)
    if out.returncode:
        raise RuntimeError(out.stderr[-500:])
    return json.loads(out.stdout.strip().splitlines()[-1])


def cpu_baseline(seconds: float = 16.0, info: dict | None = None):
    """The oracle, as it stands (C, OpenMP stencil loops, serial codec), timed
    on the host: whole sweeps of 4096 x 64 x 64 boxes of the C3 workload with
    all logical CPUs (OMP_NUM_THREADS = nproc) and with one thread, each for
    about seconds / 2."""
    import oracle
    oracle.build()
    info = info or host_info()
    planes = 64
    ncpu = os.cpu_count() or 1
    allc = _oracle_subprocess(ncpu, seconds / 2, planes)
    one = _oracle_subprocess(1, seconds / 2, planes)
    small = {}
    for th in (1, ncpu):        # C1 and C2 also at one thread
        r = subprocess.run([sys.executable, os.path.abspath(__file__), "--oracle-c1c2"], capture_output=True,
                           text=True, env=dict(os.environ, OMP_NUM_THREADS=str(th)), timeout=600)
        if r.returncode == 0:
            small[f"threads_{th}"] = json.loads(r.stdout.strip().splitlines()[-1])
    return {"value": round(allc["n"] / allc["s"], 1), "unit": "cell-updates/s", "cores": ncpu, "kind": "oracle",
            "sample": f"{allc['sweeps']} sweep(s) (T={T} steps + rate-{RATE} round trips each) of a "
                      f"4096x64x{planes} box of the C3 workload (DENSE(2) + LAYERED), {allc['s']:.1f} s, "
                      f"OMP_NUM_THREADS={ncpu}",
            "single_thread": {"value": round(one["n"] / one["s"], 1), "sweeps": one["sweeps"],
                              "seconds": round(one["s"], 1)},
            "c1_c2": dict(small, what="C1 whole (64^3, PULSE(4) + LAYERED, T = 2, rate 16, 10 steps) and one "
                                      "sweep of a 512x512x32 box of C2 (DENSE(1) + LAYERED, T = 4, rate 16), "
                                      "cell-updates/s at 1 thread and at all logical CPUs"),
            "host": {k: info.get(k) for k in ("model", "sockets", "physical_cores", "logical_cpus", "hypervisor")}}


def reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    oracle.build()
    info = host_info()
    planes = 16
    for _ in range(args.warmup):
        _oracle_sweep_sample(planes)
    tot_n, tot_s = 0, 0.0
    for _ in range(args.steps):
        n, dt = _oracle_sweep_sample(planes)
        tot_n += n
        tot_s += dt
    v = tot_n / tot_s
    sample = (f"each step: one sweep (T={T} steps + rate-{RATE} round trips) of a 4096x64x{planes} box of the C3 "
              f"workload (DENSE(2) + LAYERED), the oracle's OpenMP stencil on all logical CPUs")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(v, 1), "unit": "cell-updates/s",
        "n_gpus": int(os.environ.get("WORLD_SIZE", "1")), "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(tot_s * 1e3 / args.steps, 3), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"C3 sample: 4096x64x{planes} boxes of the {C3N}x{C3N}x{C3Z} grid, T={T}, rate {RATE}"},
        "cpu_baseline": {"value": round(v, 1), "unit": "cell-updates/s",
                         "cores": int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1)), "kind": "oracle",
                         "sample": sample, "host": {k: info.get(k) for k in ("model", "sockets", "physical_cores",
                                                                             "logical_cpus")}},
        "e2e": {"value": round(v, 1), "unit": "cell-updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10, help="timed sweeps of the C3 headline")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--sec-steps", type=int, default=3, help="timed sweeps of each secondary C3 run")
    ap.add_argument("--c2-steps", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=16.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-c2", action="store_true")
    ap.add_argument("--no-paper", action="store_true", help="skip the paper's own 1152^3 fp64 problem")
    ap.add_argument("--quick", action="store_true", help="the C3 headline and C2 rate 16 / raw only")
    ap.add_argument("--oracle-sample", type=float, default=None, help=argparse.SUPPRESS)
    ap.add_argument("--oracle-c1c2", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--oracle-planes", type=int, default=64, help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.oracle_c1c2:                         # cpu_baseline's child process (C1 / C2 sample)
        import oracle
        oracle.build()
        print(json.dumps(_oracle_c1_c2()))
        return
    if args.oracle_sample is not None:           # cpu_baseline's child process
        import oracle
        oracle.build()
        print(json.dumps(_oracle_timed(args.oracle_planes, args.oracle_sample)))
        return
    if args.warmup < 3:
        print("warning: --warmup < 3 is below the timing rules", file=sys.stderr)
    if args.impl == "reference":
        reference_arm(args)
    else:
        gpu_arm(args)


if __name__ == "__main__":
    main()
