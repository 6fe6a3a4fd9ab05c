#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_tc.py tests/test_gpu_configs.py tests/test_gpu_layers.py tests/test_gpu_parity.py -m gpu -q -x -k "not c1" > gpurun_out/gpu_tests_tpk.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gpu_tests_tpk.log; tail -3 gpurun_out/gpu_tests_tpk.log
for c in c3 c4; do
for r in 1 2; do
  for d in . ab/prev; do
    (cd $d && timeout 400 python bench.py --config $c --no-cpu-baseline --no-sweep 2>/dev/null) > gpurun_out/ab.json
    python -c "
import json
d=[json.loads(l) for l in open('gpurun_out/ab.json') if l.startswith('{')][-1]; print('$c', '$d'.ljust(10), 'value', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'conv', round(d['kernels']['conv_mma']['ms_per_step']*1e3,1), d['clocks']['sm_mhz'])"
  done
done
done
