ncu --set full --clock-control none --import-source on -k regex:"k_conv_dense$|k_conv_dense\(" -s 32 -c 8 -o gpurun_out/dense python tools/ncu_probe.py 6 > gpurun_out/ncu_dense.log 2>&1
tail -2 gpurun_out/ncu_dense.log
