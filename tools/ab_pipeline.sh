#!/bin/bash
# A/B the stencil ring depth inside the whole pipeline: value (device store) and e2e per build
for lib in liboocz.so liboocz_g128.so liboocz_g112.so liboocz_g96.so liboocz_g80.so; do
  OOCZ_LIB=$PWD/paper_2109_05410_b200/$lib python bench.py --quick --no-cpu-baseline > gpurun_out/ab_$lib.json 2>/dev/null
  OOCZ_LIB=$PWD/paper_2109_05410_b200/$lib python3 -c "
import json; d=json.load(open('gpurun_out/ab_$lib.json'))
print('$lib', 'value', round(d['value']/1e9,1), 'e2e', round(d['e2e']['value']/1e9,1), 'raw', round(d['raw']['value']/1e9,1), 'stencil_iso_ms', d['roofline_isolated']['stencil25_kernel']['ms'])"
done
