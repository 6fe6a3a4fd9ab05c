#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for i in 1 3 5; do
for cfg in "DFX_CONV_DBG=64" "DFX_CONV_DBG=66" "DFX_CONV_DBG=77" "DFX_CONV_DBG=79" "DFX_CONV_DBG=71"; do
  echo "=== dense launch $i $cfg"
  env $cfg DFX_CONV_TRACE_IDX=$i timeout 300 python tools/conv_trace2.py 2>&1 | tail -6 | grep -v "CTA start"
done
done > gpurun_out/conv_trace5.log 2>&1
cat gpurun_out/conv_trace5.log
