"""CPU checks of bench.py's host-side reporting (no GPU): the roofline of the
dominant kernel from per-launch events, the per-lane busy summary, the error
metrics of PAPER.md:247, and the codec ALU roofline read from the committed ncu
capture."""
import numpy as np
import pytest

import bench


def _ev(stage, lane, t0, t1, nbytes):
    return {"sweep": 0, "block": 0, "stage": stage, "lane": lane, "start_ms": t0, "end_ms": t1, "bytes": nbytes}


def test_roofline_picks_the_dominant_kernel_and_divides_bytes_by_time():
    # stages: 1 decode, 2 stencil, 3 encode, 6 copy (ignored)
    evs = [_ev(2, 1, 0.0, 1.0, 4_000_000_000), _ev(2, 1, 1.0, 2.0, 4_000_000_000),
           _ev(1, 4, 0.0, 0.5, 1_000_000_000), _ev(3, 5, 0.0, 0.25, 1_000_000_000),
           _ev(6, 1, 0.0, 10.0, 9_000_000_000)]
    r, table = bench.roofline(evs, 8000.0, "test")
    assert r["kernel"] == "stencil25_kernel" and r["bound"] == "hbm"
    assert r["achieved"] == pytest.approx(4000.0)            # 8e9 B over 2 ms
    assert r["frac"] == pytest.approx(0.5)
    assert r["avg_launch_ms"] == pytest.approx(1.0)
    assert r["algorithmic_bytes_per_launch"] == 4_000_000_000
    assert set(table) == {"stencil", "decode", "encode"}
    assert table["decode"]["GB/s"] == pytest.approx(2000.0)
    # traffic scales the committed ncu ratio by this run's bytes per launch
    assert r["traffic"] is None or 0.5 * 4e9 < r["traffic"] < 1.5 * 4e9


def test_lanes_summary_busy_fraction():
    evs = [_ev(2, 1, 0.0, 3.0, 0), _ev(2, 1, 5.0, 6.0, 0), _ev(1, 4, 1.0, 2.0, 0)]
    s = bench.lanes_summary(evs)
    assert s["span_ms"] == pytest.approx(6.0)
    assert s["compute"]["busy_ms"] == pytest.approx(4.0) and s["compute"]["busy_frac"] == pytest.approx(4 / 6, abs=1e-3)
    assert s["decode"]["busy_frac"] == pytest.approx(1 / 6, abs=1e-3)
    assert bench.lanes_summary([]) == {}


def test_rel_errors_metrics():
    b = np.full((4, 8, 8), 2.0, np.float32)
    a = b.copy()
    a[1, 2, 3] = 2.5                                        # one point off by 25 %
    r = bench.rel_errors(a, b, per_plane=10)
    assert r["normwise_max"] == pytest.approx(0.25)
    assert r["points"] == 40 and r["skipped"] == 0
    assert 0.0 <= r["mean_pointwise"] <= 0.25
    z = bench.rel_errors(b, b)
    assert z["normwise_max"] == 0.0 and z["mean_pointwise"] == 0.0
    # points where the reference is zero are skipped, not divided by
    c = np.zeros((2, 4, 4), np.float32)
    rc = bench.rel_errors(c, c, per_plane=5)
    assert rc["skipped"] == 10 and rc["mean_pointwise_significant"] == 0.0 and rc["significant_points"] == 0


def test_codec_alu_roofline_from_committed_capture():
    table = {"decode": {"ms": 2.0, "launches": 8, "avg_launch_ms": 0.25},
             "encode": {"ms": 1.0, "launches": 8, "avg_launch_ms": 0.125}}
    r = bench.codec_alu_roofline(table)
    assert r is not None
    for k in ("zfp_decode_kernel", "zfp_encode_kernel"):
        assert r[k]["bound"] == "alu" and 0.5 < r[k]["frac"] <= 1.0
        assert r[k]["peak"] == pytest.approx(148 * 4 * 0.5 * 1.965, rel=1e-3)
        assert r[k]["achieved"] == pytest.approx(r[k]["frac"] * r[k]["peak"], rel=1e-2)
    assert r["zfp_decode_kernel"]["in_step_avg_ms"] == pytest.approx(0.25)


def test_pick_P_and_host_info():
    assert bench.pick_P(1536, 64) == 64 and bench.pick_P(1536, 192) == 192
    assert bench.pick_P(192, 64) == 64 and bench.pick_P(768, 96) == 96
    assert bench.pick_P(40, 64) == 40          # nothing fits: the whole slab
    info = bench.host_info()
    assert info["logical_cpus"] >= 1 and info.get("mem_total_bytes", 1) > 0
