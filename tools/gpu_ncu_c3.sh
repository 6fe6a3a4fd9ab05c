#!/bin/bash
# C3 (ResNet-18, 720p): launch list of one steady frame and ncu --set full of its strided (gathered) convs
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv \
  python tools/ncu_probe.py 4 c3 > /dev/null 2>&1; echo "list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_conv_tc -s 20 -c 6 -o gpurun_out/c3_conv_tc \
  python tools/ncu_probe.py 4 c3 > gpurun_out/ncu_c3.log 2>&1; echo "full rc=$?"
ncu -i gpurun_out/c3_conv_tc.ncu-rep --page raw --csv > gpurun_out/c3_conv_tc_raw.csv 2>/dev/null; rm -f gpurun_out/c3_conv_tc.ncu-rep
