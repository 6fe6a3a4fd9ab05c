#!/bin/bash
# GPU box: per-kernel time in the real launch chain (DFX_KTRACE) and the dense
# conv pipeline stamps of every C2 conv layer (DFX_CONV_DBG=64)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
DFX_KTRACE=1 timeout 300 python tools/ktrace.py > gpurun_out/ktrace.log 2>&1; tail -50 gpurun_out/ktrace.log
for i in 0 1 2 3 4 5 6 7; do
  echo "=== dense launch $i"
  DFX_CONV_DBG=64 DFX_CONV_TRACE_IDX=$i timeout 300 python tools/conv_trace.py 2>&1 | grep -E "kernel \(CTA|median|CTAs|loader startup|epilogue items|segments" 
done > gpurun_out/conv_trace.log 2>&1
cat gpurun_out/conv_trace.log
