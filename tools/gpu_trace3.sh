#!/bin/bash
# dense conv launch i under debug bits (applied to that launch only): 64 trace,
# +1 no MMAs, +4 no weight copies, +8 no A stores
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for i in ${IDX:-1 3 5}; do
for d in 64 65 68 72 69 77; do
  echo "=== dense launch $i dbg $d"
  DFX_CONV_DBG=$d DFX_CONV_TRACE_IDX=$i timeout 300 python tools/conv_trace2.py 2>&1 | tail -6
done
done > gpurun_out/conv_trace3.log 2>&1
cat gpurun_out/conv_trace3.log
