#!/bin/bash
cd "$(dirname "$0")/.."
for n in 1 2 3 4 6; do
  DFX_BRANCH_SIDES=$n timeout 400 python bench.py --config c4 --no-cpu-baseline --no-sweep > gpurun_out/ab.json 2>/dev/null
  python -c "
import json
d=[json.loads(l) for l in open('gpurun_out/ab.json') if l.startswith('{')][-1]; print('c4 sides=$n', 'value', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), d['clocks']['sm_mhz'])"
done
for b in 0 1; do
  DFX_BRANCH_STREAMS=$b timeout 900 python bench.py --config c5 --no-cpu-baseline --steps 10 > gpurun_out/ab.json 2>/dev/null
  python -c "
import json
d=[json.loads(l) for l in open('gpurun_out/ab.json') if l.startswith('{')][-1]; print('c5 branch=$b', 'value', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), d['clocks']['sm_mhz'])"
done
