#!/bin/bash
# GPU box: per-CTA timelines of dense conv launches of a C2 frame; DBG 64 = trace,
# +4 = no weight copies (arrive only), +1 = no MMAs
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for d in 64 68 65 69; do
for i in ${IDX:-0 1 2 3 4 5 6 7}; do
  echo "=== dense launch $i dbg $d"
  DFX_CONV_DBG=$d DFX_CONV_TRACE_IDX=$i timeout 300 python tools/conv_trace2.py 2>&1 | tail -7
done
done > gpurun_out/conv_trace2.log 2>&1
cat gpurun_out/conv_trace2.log
