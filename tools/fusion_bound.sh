#!/bin/bash
# Upper bound of what a fused decode->stencil / stencil->encode pass could save
# (SURVEY 8(f) row 3): the C2 HBM-resident pipeline with the decoder's output
# stores removed after the warm-up (OOCZ_DEC_NOSTORE: all its arithmetic, no
# float4 stores once a context has made OOCZ_DEC_NOSTORE_AFTER decode launches,
# so the slabs keep real data from earlier blocks; removing them from the first
# launch left the slabs zero and the encoder coding all-zero blocks, which is
# what the first version of this bound measured) and the
# encoder's input loads served from a 1 MB L2-resident range (OOCZ_ENC_L2IN), i.e.
# exactly the slab write + re-read a fused pass avoids; and, for on-chip
# temporal blocking, every second stencil launch skipped (OOCZ_AB_HALF_STEPS:
# two steps for the price of one pass, no halo recompute).  Results are not the
# method's (timing only).  Alternating runs, two rounds.
set -e
cd "$(dirname "$0")/.."
B=paper_2109_05410_b200
# (the four libraries are built beforehand, e.g. here:
#  python -m paper_2109_05410_b200.build [-DOOCZ_DEC_NOSTORE] [-DOOCZ_ENC_L2IN] --out $B/liboocz_ab_<v>.so)
export OOCZ_DEC_NOSTORE_AFTER=${OOCZ_DEC_NOSTORE_AFTER:-30}
for round in 1 2; do
  for v in base decnostore encl2 both halfsteps; do
    OOCZ_LIB=$PWD/$B/liboocz_ab_$v.so python tools/ab_one.py
  done
done
# the same on C3 with the compressed store in HBM (P = 96: 16 blocks x 3 fields
# decoded per sweep, so the decoder stores stop after the 2 warm-up sweeps)
if [ "${C3:-1}" = 1 ]; then
  for v in base decnostore encl2 both halfsteps; do
    echo -n "liboocz_ab_$v.so C3 hbm:96 "
    OOCZ_DEC_NOSTORE_AFTER=100 OOCZ_LIB=$PWD/$B/liboocz_ab_$v.so python tools/c3_run.py --schedules hbm:96 \
        --warmup 2 --sweeps 3 --chunk 4 --no-parity | grep '^hbm'
  done
fi
