#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 env DFX_GRID_HINT=1 python -m pytest tests/test_gpu_configs.py tests/test_gpu_fullwidth.py -m gpu -q -x -k "configs or crops_exact" 2>&1 | tail -2
for c in c2 c3 c4 c5; do
for r in 1 2; do
  for h in 0 1; do
    st=20; [ $c = c5 ] && st=10
    DFX_GRID_HINT=$h timeout 600 python bench.py --config $c --steps $st --no-cpu-baseline --no-sweep > gpurun_out/ab.json 2>/dev/null
    python -c "
import json
d=[json.loads(l) for l in open('gpurun_out/ab.json') if l.startswith('{')][-1]; print('$c hint=$h', 'value', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), d['clocks']['sm_mhz'])"
  done
done
done
