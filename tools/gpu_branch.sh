#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_configs.py -m gpu -q -x > gpurun_out/gpu_tests_branch.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gpu_tests_branch.log; tail -3 gpurun_out/gpu_tests_branch.log
for c in c4 c3 c2; do
for r in 1 2; do
  for f in 0 1; do
    DFX_BRANCH_STREAMS=$f timeout 400 python bench.py --config $c --no-cpu-baseline --no-sweep > gpurun_out/ab.json 2>/dev/null
    python -c "
import json
d=[json.loads(l) for l in open('gpurun_out/ab.json') if l.startswith('{')][-1]; print('$c branch=$f', 'value', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), d['clocks']['sm_mhz'])"
  done
done
done
timeout 900 python bench.py --gpus 2 --no-cpu-baseline --no-sweep > gpurun_out/bench_c2_2ranks_1gpu.log 2>&1; echo "2ranks rc=$?"; grep '^{' gpurun_out/bench_c2_2ranks_1gpu.log | cut -c1-400
