# full ncu capture (with source) of one truncation launch (layer 1, frame 5) and one conv_plan launch
ncu --set full --import-source on --clock-control none -k regex:k_trunc_coop -s 36 -c 2 -o gpurun_out/trunc python tools/ncu_probe.py 6 > gpurun_out/trunc.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_conv_plan -s 40 -c 1 -o gpurun_out/plan python tools/ncu_probe.py 6 > gpurun_out/plan.log 2>&1
tail -2 gpurun_out/trunc.log gpurun_out/plan.log
