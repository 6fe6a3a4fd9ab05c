# full ncu capture (with source) of the conv8 dense launch of frame 5
ncu --set full --import-source on --clock-control none -k regex:k_conv_dense -s 37 -c 1 -o gpurun_out/dense8 python tools/ncu_probe.py 6 > gpurun_out/dense8.log 2>&1
tail -n 2 gpurun_out/dense8.log
