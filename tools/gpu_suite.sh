#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
DFX_PARITY_REPORT=gpurun_out/parity_suite.json timeout 1800 python -m pytest tests -m gpu -q --durations=5 > gpurun_out/gpu_tests_suite.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gpu_tests_suite.log; tail -6 gpurun_out/gpu_tests_suite.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
