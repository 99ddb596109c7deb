#!/bin/bash
# A/B: stream priorities on / off, headline quick bench (value, e2e, in-step stencil)
for v in 0 1 0 1; do
  OOCZ_STREAM_PRIORITY=$v python bench.py --quick --no-cpu-baseline 2>/dev/null | tail -1 | python3 -c "
import json,sys; d=json.loads(sys.stdin.read())
print('prio=$v', 'value', round(d['value']/1e9,1), 'e2e', round(d['e2e']['value']/1e9,1), 'raw', round(d['raw']['value']/1e9,1), 'stencil_frac', d['roofline']['frac'], d['kernels_in_step'])"
done
