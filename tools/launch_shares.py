"""Kernel shares of the sweeps in an ncu launch list (ncu --metrics
gpu__time_duration.sum --csv of a bench run): the launches after the last
set_field kernel (scan_field_kernel), i.e. the warm-up and timed sweeps.
Durations are serialised and cold-cache (ncu), so the SHARES are what compare
with the bench's in-step kernel times, not the absolute values.

  python tools/launch_shares.py <launches.csv>
"""
import collections
import csv
import json
import sys

SCALE = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, mi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    launches = []
    for r in rows[hi + 1:]:
        if len(r) <= mi:
            continue
        name = r[ki].split("(")[0].replace("(anonymous namespace)::", "").replace("oocz::<unnamed>::", "")
        launches.append((name, float(r[mi].replace(",", "")) * SCALE.get(r[ui], 1.0)))
    last = max(i for i, (n, _) in enumerate(launches) if "scan_field" in n)
    tot, cnt = collections.Counter(), collections.Counter()
    for n, us in launches[last + 1:]:
        tot[n] += us
        cnt[n] += 1
    s = sum(tot.values())
    out = {"source": sys.argv[1], "launches_in_sweeps": sum(cnt.values()),
           "kernels": {n: {"launches": cnt[n], "ms": round(v / 1e3, 2), "share": round(v / s, 4)}
                       for n, v in tot.most_common()}}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
