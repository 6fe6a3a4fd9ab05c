#!/bin/bash
# GPU box: the -m gpu suite with the parity report, then a default bench line.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
DFX_PARITY_REPORT=gpurun_out/parity_report.json timeout ${TEST_TIMEOUT:-1500} python -m pytest tests -m gpu -q -x ${PYTEST_ARGS} --durations=25 > gpurun_out/gpu_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
tail -40 gpurun_out/gpu_tests.log
if [ -z "$NO_BENCH" ]; then
  timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1
  tail -c 3000 gpurun_out/bench.log
fi
