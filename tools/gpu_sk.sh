#!/bin/bash
# stream-K dense conv: parity tests, per-launch timelines, same-box A/B
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "fullwidth or tc or parity or configs or layers" > gpurun_out/gpu_tests_sk.log 2>&1; tail -3 gpurun_out/gpu_tests_sk.log
for sk in 0 1; do
for i in 2 3 4 5 6; do
  echo "=== SK $sk dense launch $i"
  DFX_DENSE_SK=$sk DFX_CONV_DBG=64 DFX_CONV_TRACE_IDX=$i timeout 300 python tools/conv_trace2.py 2>&1 | tail -6 | grep -v "CTA start"
done
done > gpurun_out/conv_trace_sk.log 2>&1
cat gpurun_out/conv_trace_sk.log
VAR=DFX_DENSE_SK VALS="0 1" bash tools/gpu_env_ab.sh
