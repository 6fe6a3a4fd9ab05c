ncu --set full --import-source on --clock-control none -k regex:"k_input_tile" -s 10 -c 2 -o gpurun_out/input python tools/ncu_probe.py 8 > gpurun_out/input.log 2>&1
tail -n 2 gpurun_out/input.log
