#!/bin/bash
# A/B of the codec rewrite on the device paths (tools/ab_one.py), alternating
cd "$(dirname "$0")/.."
B=paper_2109_05410_b200
for r in 1 2; do for v in old new; do OOCZ_LIB=$PWD/$B/liboocz_ab_$v.so python tools/ab_one.py; done; done
