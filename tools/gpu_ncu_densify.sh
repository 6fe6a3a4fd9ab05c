ncu --set full --import-source on --clock-control none -k regex:"k_densify" -s 4 -c 1 -o gpurun_out/densify python tools/ncu_probe.py 6 > gpurun_out/densify.log 2>&1
tail -n 1 gpurun_out/densify.log
