#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kats.py tests/test_gpu_boundary.py -m gpu -q -x -k "not c1" > gpurun_out/gpu_tests_rb.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gpu_tests_rb.log; tail -3 gpurun_out/gpu_tests_rb.log
for c in c2 c4; do
for r in 1 2; do
  for d in . ab/prev; do
    (cd $d && timeout 400 python bench.py --config $c --no-cpu-baseline --no-sweep 2>/dev/null) > gpurun_out/ab.json
    python -c "
import json
d=[json.loads(l) for l in open('gpurun_out/ab.json') if l.startswith('{')][-1]; print('$c', '$d'.ljust(10), 'value', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'densify', round(d['kernels']['densify']['ms_per_step']*1e3,1), d['clocks']['sm_mhz'])"
  done
done
done
