ncu --set full --import-source on --clock-control none -k regex:"k_conv_plan" -s 32 -c 1 -o gpurun_out/plan16 python tools/ncu_probe.py 6 > gpurun_out/plan16.log 2>&1
tail -n 1 gpurun_out/plan16.log
