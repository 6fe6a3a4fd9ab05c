#!/bin/bash
cd "$(dirname "$0")/.."
timeout 1200 python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py tests/test_gpu_tc.py -m gpu -q -x -k "not c1" 2>&1 | tail -2
for r in 1 2; do
  for f in 0 1; do
    DFX_FUSE_UPSAMPLE=$f timeout 600 python bench.py --config c4 --no-cpu-baseline --no-sweep > gpurun_out/ab.json 2>/dev/null
    python -c "
import json
d=[json.loads(l) for l in open('gpurun_out/ab.json') if l.startswith('{')][-1]; print('c4 up=$f', 'value', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), d['gpu_launches']//d['steps'], d['clocks']['sm_mhz'])"
  done
done
