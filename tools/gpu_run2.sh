#!/bin/bash
# GPU box: new config / boundary parity tests, then bench lines for every config
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
DFX_PARITY_REPORT=gpurun_out/parity_report2.json timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_boundary.py -m gpu -q -x --durations=10 > gpurun_out/gpu_tests2.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gpu_tests2.log
tail -15 gpurun_out/gpu_tests2.log
for c in c2 c3 c4; do
  timeout 600 python bench.py --config $c --no-cpu-baseline $( [ $c = c2 ] && echo --sweep ) > gpurun_out/bench_$c.log 2>&1
  echo "== $c rc=$?"; tail -c 600 gpurun_out/bench_$c.log; echo
done
timeout 900 python bench.py --config c5 --no-cpu-baseline --steps 10 > gpurun_out/bench_c5.log 2>&1; echo "== c5 rc=$?"; tail -c 400 gpurun_out/bench_c5.log
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_c2.log 2>&1; echo "== ref rc=$?"; tail -c 1500 gpurun_out/bench_ref_c2.log
