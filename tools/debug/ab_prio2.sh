#!/bin/bash
# A/B of stream priorities (compute stream high) through the whole bench: value,
# e2e and the in-step stencil roofline fraction, alternating runs
for i in 1 2; do
  for p in 0 1; do
    OOCZ_STREAM_PRIORITY=$p python bench.py --quick --no-cpu-baseline > gpurun_out/abp_$p_$i.json 2>/dev/null
    python3 -c "
import json; d=json.loads(open('gpurun_out/abp_$p_$i.json').read().strip().splitlines()[-1])
print('prio=$p run=$i', 'value', round(d['value']/1e9,1), 'e2e', round(d['e2e']['value']/1e9,1), 'raw', round(d['raw']['value']/1e9,1), 'stencil_frac', d['roofline']['frac'], 'kis', {k: v['ms'] for k, v in d['kernels_in_step'].items()})"
  done
done
