#!/bin/bash
# GPU box: next conv's plan inside the activation commit launch — parity, then A/B (DFX_FUSE_PLAN) on C2 / C3
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_kats.py tests/test_gpu_tc.py tests/test_gpu_parity.py tests/test_gpu_fullwidth.py tests/test_gpu_configs.py -m gpu -q -x -k "not full_frame and not c1_16 and not exact_c1" > gpurun_out/gpu_tests_plan.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gpu_tests_plan.log; tail -4 gpurun_out/gpu_tests_plan.log
for c in c2 c3; do
for r in 1 2 3; do
  for f in 0 1; do
    DFX_FUSE_PLAN=$f timeout 600 python bench.py --config $c --no-cpu-baseline --no-sweep > gpurun_out/ab_plan$f.log 2>&1
    python - <<PY
import json
d=[json.loads(l) for l in open('gpurun_out/ab_plan$f.log') if l.startswith('{')][-1]
k=d['kernels']
print('$c fuse_plan=$f', round(d['value'],1), round(d['e2e']['value'],1), 'trunc', round(k['truncate']['ms_per_step']*1000,1), 'plan', round(k.get('conv_targets',{}).get('ms_per_step',0)*1000,1), d['gpu_launches']//d['steps'], d['clocks']['sm_mhz'])
PY
  done
done
done
DFX_KTRACE=1 timeout 300 python tools/ktrace.py > gpurun_out/ktrace2.log 2>&1; head -3 gpurun_out/ktrace2.log
