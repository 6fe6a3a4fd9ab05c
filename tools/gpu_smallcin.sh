#!/bin/bash
cd "$(dirname "$0")/.."
for r in 1 2; do
for v in 0 4; do
  for c in c2 c3; do
  DFX_SMALLCIN_EXACT=$v timeout 400 python bench.py --config $c --no-cpu-baseline --no-sweep > gpurun_out/ab.json 2>/dev/null
  python -c "
import json
d=[json.loads(l) for l in open('gpurun_out/ab.json') if l.startswith('{')][-1]; k=d['kernels']; print('$c smallcin=$v', 'value', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'conv', round(k['conv_mma']['ms_per_step']*1e3,1), 'tgt', round(k['conv_targets']['ms_per_step']*1e3,1), d['clocks']['sm_mhz'])"
  done
done
done
for n in 6 8; do
  DFX_BRANCH_SIDES=$n timeout 400 python bench.py --config c4 --no-cpu-baseline --no-sweep > gpurun_out/ab.json 2>/dev/null
  python -c "
import json
d=[json.loads(l) for l in open('gpurun_out/ab.json') if l.startswith('{')][-1]; print('c4 sides=$n', 'value', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), d['clocks']['sm_mhz'])"
done
