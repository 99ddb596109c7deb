#!/bin/bash
# A/B of the codec loops' additions on the FMA pipe (OOCZ_FMA_ADDS=1, IMAD with a
# constant-bank multiplier) against plain additions (-DOOCZ_FMA_ADDS=0), on the
# device paths and the isolated kernels (tools/ab_one.py), then C3 in HBM
# (tools/lane_probe.py c3hbm), alternating.  Variants:
#   python -m paper_2109_05410_b200.build -DOOCZ_FMA_ADDS=0 --out paper_2109_05410_b200/liboocz_ab_noadd.so
#   python -m paper_2109_05410_b200.build --force --out paper_2109_05410_b200/liboocz_ab_fmaadd.so
cd "$(dirname "$0")/.."
B=paper_2109_05410_b200
V=${VARIANTS:-"noadd fmaadd"}
for r in 1 2 3; do for v in $V; do OOCZ_LIB=$PWD/$B/liboocz_ab_$v.so python tools/ab_one.py; done; done
if [ -n "$C3" ]; then
  for v in $V; do echo "== $v"; OOCZ_LIB=$PWD/$B/liboocz_ab_$v.so python tools/lane_probe.py c3hbm | tail -1; done
fi
