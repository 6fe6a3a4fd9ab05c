#!/bin/bash
# GPU box: float4 add / upsample — C3 / C4 parity, then A/B vs ab/prev on C3 and C4
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py -m gpu -q -x -k "not c1" > gpurun_out/gpu_tests_lin.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gpu_tests_lin.log; tail -3 gpurun_out/gpu_tests_lin.log
for c in c3 c4; do
for r in 1 2; do
  for d in . ab/prev; do
    (cd $d && timeout 400 python bench.py --config $c --no-cpu-baseline --no-sweep 2>/dev/null) > gpurun_out/ab.json
    python -c "
import json
d=[json.loads(l) for l in open('gpurun_out/ab.json') if l.startswith('{')][-1]; print('$c', '$d'.ljust(10), 'value', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'linear', round(d['kernels']['linear_ops']['ms_per_step']*1e3,1), d['clocks']['sm_mhz'])"
  done
done
done
