#!/bin/bash
cd "$(dirname "$0")/.."
for r in 1 2; do
  for d in . ab/mb3 ab/mb4; do
    (cd $d && timeout 400 python bench.py --no-cpu-baseline --no-sweep 2>/dev/null) > gpurun_out/ab.json
    python -c "
import json
d=[json.loads(l) for l in open('gpurun_out/ab.json') if l.startswith('{')][-1]; k=d['kernels']; print('$d'.ljust(10), 'value', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'trunc', round(k['truncate']['ms_per_step']*1e3,1), d['clocks']['sm_mhz'])"
  done
done
