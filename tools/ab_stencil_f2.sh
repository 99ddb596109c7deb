#!/bin/bash
# A/B of the stencil's packed fp32 arithmetic (FADD2/FFMA2, OOCZ_STENCIL_F2) and of
# a 2-plane z-march step (OOCZ_STENCIL_ZU=2: half the register-queue moves)
# on the device paths (tools/ab_one.py: C2 in HBM, C2 out of core, isolated
# kernels) and on C3 in HBM (tools/lane_probe.py c3hbm), alternating.  Variants:
#   python -m paper_2109_05410_b200.build -DOOCZ_STENCIL_F2=0 --out paper_2109_05410_b200/liboocz_ab_scalar.so
#   python -m paper_2109_05410_b200.build -DOOCZ_STENCIL_F2=0 -DOOCZ_STENCIL_ZU=2 --out .../liboocz_ab_zu2.so
#   python -m paper_2109_05410_b200.build -DOOCZ_STENCIL_ZU=1 --out .../liboocz_ab_f2.so
#   python -m paper_2109_05410_b200.build -DOOCZ_STENCIL_ZU=2 --out .../liboocz_ab_f2zu2.so
cd "$(dirname "$0")/.."
B=paper_2109_05410_b200
V=${VARIANTS:-"scalar zu2 f2 f2zu2"}
for r in 1 2; do for v in $V; do OOCZ_LIB=$PWD/$B/liboocz_ab_$v.so python tools/ab_one.py; done; done
if [ -n "$C3" ]; then
  for v in $V; do echo "== $v"; OOCZ_LIB=$PWD/$B/liboocz_ab_$v.so python tools/lane_probe.py c3hbm | head -1; done
fi
