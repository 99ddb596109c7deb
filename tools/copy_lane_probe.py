"""Per-copy rates and gaps of the C3 headline's H2D / D2H lanes (profile = 1
events): are the copies themselves slower than the link probe, or do they wait?

  python tools/copy_lane_probe.py
"""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2109_05410_b200 import oocz as Z  # noqa: E402
from paper_2109_05410_b200.oocz import STAGES  # noqa: E402

torch.cuda.set_device(0)
nx, nz = bench.C3N, bench.C3Z
cfg = Z.oocz_default_config(nx, nx, nz, tb=4, block_planes=64, rate=[16] * 3)
need = Z.oocz_host_store_bytes(cfg, 1)
arena = (Z.oocz_host_alloc(need), need)
opt = dict(P=64, serpentine=1, m_resident=1, slots=3)
r = bench.run_c3(Z, "probe", nx, nx, nz, (16,) * 3, opt, arena, 0, 1, None, 0, 3, 2, None, profile=1)
out = {"cups_G": round(r["cups"] / 1e9, 2)}
for lane in ("h2d", "d2h"):
    ev = sorted((e for e in r["evs"] if STAGES[e["stage"]] == lane), key=lambda e: e["start_ms"])
    rates = [e["bytes"] / ((e["end_ms"] - e["start_ms"]) / 1e3) / 1e9 for e in ev if e["end_ms"] > e["start_ms"]]
    gaps = [b["start_ms"] - a["end_ms"] for a, b in zip(ev, ev[1:])]
    span = ev[-1]["end_ms"] - ev[0]["start_ms"]
    out[lane] = {"events": len(ev), "GB_per_event_median": round(statistics.median(e["bytes"] for e in ev) / 1e9, 2),
                 "rate_GBps_median": round(statistics.median(rates), 2), "rate_GBps_min": round(min(rates), 2),
                 "rate_GBps_max": round(max(rates), 2), "gap_ms_total": round(sum(g for g in gaps if g > 0), 1),
                 "span_ms": round(span, 1), "bytes_over_span_GBps": round(sum(e["bytes"] for e in ev) / (span / 1e3) / 1e9, 2)}
Z.oocz_host_free(arena[0])
print(json.dumps(out))
