#!/bin/bash
# A/B of cache policies on the slab traffic (device path, C2): streaming
# (evict-first) decoder stores, encoder loads, stencil stores; and the
# decoder-without-stores bound.  Alternating, two rounds.
cd "$(dirname "$0")/.."
B=paper_2109_05410_b200
for r in 1 2; do for v in base v1 v2 v3 decnostore; do OOCZ_LIB=$PWD/$B/liboocz_ab_$v.so python tools/ab_one.py; done; done
