#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py tests/test_gpu_kats.py -m gpu -q -x -k "not c1" 2>&1 | tail -2
for c in c4 c5 c2; do
for r in 1 2; do
  for d in . ab/prev; do
    st=20; [ $c = c5 ] && st=10
    (cd $d && timeout 600 python bench.py --config $c --steps $st --no-cpu-baseline --no-sweep 2>/dev/null) > gpurun_out/ab.json
    python -c "
import json
d=[json.loads(l) for l in open('gpurun_out/ab.json') if l.startswith('{')][-1]; print('$c', '$d'.ljust(10), 'value', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), d['clocks']['sm_mhz'])"
  done
done
done
