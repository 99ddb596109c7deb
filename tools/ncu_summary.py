"""Summaries of committed ncu captures (run here on the .ncu-rep files gpurun
brings back):

  python tools/ncu_summary.py instep <report> <out.json>
      per stencil launch inside the bench: duration, DRAM read / write bytes
      against the algorithmic 16 B per updated cell (profiles/*_instep_traffic.json)
  python tools/ncu_summary.py kernels <report> <out.json>
      per kernel: duration, issue / pipe utilisation, DRAM bytes, registers
"""
import csv
import io
import json
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "smsp__inst_executed.sum",
           "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
           "sm__warps_active.avg.pct_of_peak_sustained_active",
           "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
           "launch__grid_size", "launch__block_size", "smsp__thread_inst_executed_per_inst_executed.ratio"]


def rows(report):
    txt = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    r = list(csv.reader(io.StringIO(txt)))
    hdr, units = r[0], r[1]
    for row in r[2:]:
        d = {"kernel": row[hdr.index("Kernel Name")].split("(")[0].replace("(anonymous namespace)::", "")
             .replace("unnamed>::", "")}
        for m in METRICS:
            if m in hdr:
                v, u = row[hdr.index(m)], units[hdr.index(m)]
                try:
                    v = float(v.replace(",", ""))
                except ValueError:
                    pass
                if u == "Mbyte":
                    v, u = v * 1e6, "byte"
                if u == "Gbyte":
                    v, u = v * 1e9, "byte"
                d[m] = v
                d[m + ":unit"] = u
        yield d


def main():
    mode, rep, out = sys.argv[1:4]
    rs = list(rows(rep))
    if mode == "instep":
        # argv[4]: updated planes of each captured launch (comma list), nx*ny = argv[5]
        planes = [int(x) for x in sys.argv[4].split(",")]
        plane = int(sys.argv[5])
        st = [d for d in rs if "stencil25" in d["kernel"]]
        launches = []
        for d, pl in zip(st, planes):
            tr = d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]
            launches.append({"us": d["gpu__time_duration.sum"], "dram_read_B": d["dram__bytes_read.sum"],
                             "dram_write_B": d["dram__bytes_write.sum"], "traffic_B": tr,
                             "algorithmic_B": 16 * pl * plane})
        res = {"report": rep, "launches": launches,
               "traffic_over_algorithmic": round(sum(x["traffic_B"] for x in launches) /
                                                 sum(x["algorithmic_B"] for x in launches), 3)}
    else:
        res = {"report": rep, "kernels": rs}
    with open(out, "w") as fh:
        json.dump(res, fh, indent=1)
    print(json.dumps(res, indent=1)[:3000])


if __name__ == "__main__":
    main()
