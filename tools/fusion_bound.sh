#!/bin/bash
# Upper bound of what a fused decode->stencil / stencil->encode pass could save
# (SURVEY 8(f) row 3): the C2 HBM-resident pipeline with the decoder's output
# stores removed (OOCZ_DEC_NOSTORE: all its arithmetic, no float4 stores) and the
# encoder's input loads served from a 1 MB L2-resident range (OOCZ_ENC_L2IN), i.e.
# exactly the slab write + re-read a fused pass avoids.  Results are not the
# method's (timing only).  Alternating runs, two rounds.
set -e
cd "$(dirname "$0")/.."
B=paper_2109_05410_b200
[ -f $B/liboocz_ab_base.so ] || python -m paper_2109_05410_b200.build --out $B/liboocz_ab_base.so --force > /dev/null
[ -f $B/liboocz_ab_decnostore.so ] || python -m paper_2109_05410_b200.build -DOOCZ_DEC_NOSTORE --out $B/liboocz_ab_decnostore.so > /dev/null
[ -f $B/liboocz_ab_encl2.so ] || python -m paper_2109_05410_b200.build -DOOCZ_ENC_L2IN --out $B/liboocz_ab_encl2.so > /dev/null
[ -f $B/liboocz_ab_both.so ] || python -m paper_2109_05410_b200.build -DOOCZ_DEC_NOSTORE -DOOCZ_ENC_L2IN --out $B/liboocz_ab_both.so > /dev/null
for round in 1 2; do
  for v in base decnostore encl2 both; do
    OOCZ_LIB=$PWD/$B/liboocz_ab_$v.so python tools/ab_one.py
  done
done
