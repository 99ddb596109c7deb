"""profiles/<tag>_ncu_kernels.json from the two --set full captures of
tools/ncu_r02.sh (C3-wide slab and C2 slab, rate 16): per kernel launch its
duration, DRAM bytes against the algorithmic bytes, ALU-pipe and issue
utilisation, warp-instructions and registers.  Runs here on the .ncu-rep files
gpurun brings back (no GPU needed).

  python tools/ncu_kernels_json.py <tag>      # reads gpurun_out/<tag>_c{3,2}_kernels.ncu-rep
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import ncu_summary  # noqa: E402

RATE = 16
SLABS = {"c3_slab": (4096, 96, "4096 x 4096 x 96 planes of the C3 data (DENSE(2), LAYERED), stencil updates planes [4, 92)"),
         "c2_slab": (512, 160, "512 x 512 x 160 planes of the C2 data (DENSE(1), LAYERED), stencil updates planes [4, 156)")}


def main():
    tag = sys.argv[1]
    out = {"what": "ncu --set full --clock-control none of the three hot kernels (tools/ncu_r02.sh, "
                   "tools/prof_kernels.py), rate 16, 2 launches each",
           "reports": ", ".join(f"gpurun_out/{tag}_{c}_kernels.ncu-rep" for c in ("c3", "c2")) + " (scratch, not committed)"}
    for key, (n, planes, what) in SLABS.items():
        rep = f"gpurun_out/{tag}_{key[:2]}_kernels.ncu-rep"
        values = n * n * planes
        comp = values // 64 * 8 * RATE
        ks = []
        for d in ncu_summary.rows(rep):
            name = d["kernel"]
            alg = 16 * n * n * (planes - 8) if "stencil" in name else 4 * values + comp
            tr = d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]
            scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(
                d.get("gpu__time_duration.sum:unit"), 1.0)
            ks.append({"kernel": name, "us": d["gpu__time_duration.sum"] * scale,
                       "dram_read_B": d["dram__bytes_read.sum"], "dram_write_B": d["dram__bytes_write.sum"],
                       "traffic_B": tr, "algorithmic_B": alg, "traffic_over_algorithmic": round(tr / alg, 4),
                       "alu_pipe_pct": d["sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"],
                       "fma_pipe_pct": d["sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"],
                       "issue_active_pct": d["smsp__issue_active.avg.pct_of_peak_sustained_active"],
                       "warps_active_pct": d["sm__warps_active.avg.pct_of_peak_sustained_active"],
                       "warp_inst": d["smsp__inst_executed.sum"], "registers": d["launch__registers_per_thread"]})
        out[key] = {"slab": what, "kernels": ks}
    with open(f"profiles/{tag}_ncu_kernels.json", "w") as fh:
        json.dump(out, fh, indent=1)
    for key in SLABS:
        for k in out[key]["kernels"]:
            print(key, k["kernel"][:24], round(k["us"], 1), "us  alu", k["alu_pipe_pct"], " issue", k["issue_active_pct"],
                  " traffic/alg", k["traffic_over_algorithmic"])


if __name__ == "__main__":
    main()
