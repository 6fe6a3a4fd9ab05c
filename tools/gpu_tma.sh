#!/bin/bash
# GPU box: TMA patch staging — parity of every dense-path test, then an A/B (DFX_DENSE_TMA) of the bench
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kats.py tests/test_gpu_tc.py -m gpu -q -x > gpurun_out/gpu_tests_tma.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gpu_tests_tma.log; tail -5 gpurun_out/gpu_tests_tma.log
timeout 900 python -m pytest tests/test_gpu_fullwidth.py tests/test_gpu_parity.py -m gpu -q -x -k "not full_frame" >> gpurun_out/gpu_tests_tma.log 2>&1
echo "pytest2 rc=$?" >> gpurun_out/gpu_tests_tma.log; tail -3 gpurun_out/gpu_tests_tma.log
for r in 1 2 3; do
  for f in 0 1; do
    DFX_DENSE_TMA=$f timeout 600 python bench.py --no-cpu-baseline > gpurun_out/ab_tma$f.log 2>&1
    python - <<PY
import json
d=[json.loads(l) for l in open('gpurun_out/ab_tma$f.log') if l.startswith('{')][-1]
print('tma=$f', round(d['value'],1), round(d['e2e']['value'],1), 'conv', round(d['kernels']['conv_mma']['ms_per_step']*1000,1), d['clocks']['sm_mhz'])
PY
  done
done
