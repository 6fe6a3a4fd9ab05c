#!/bin/bash
cd "$(dirname "$0")/.."
for r in 1 2; do
for v in 8 4 2 1; do
  DFX_DENSE_SMAX=$v timeout 400 python bench.py --no-cpu-baseline --no-sweep > gpurun_out/ab.json 2>/dev/null
  python -c "
import json
d=[json.loads(l) for l in open('gpurun_out/ab.json') if l.startswith('{')][-1]; k=d['kernels']; print('smax=$v', 'value', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'conv', round(k['conv_mma']['ms_per_step']*1e3,1), d['clocks']['sm_mhz'])"
done
done
