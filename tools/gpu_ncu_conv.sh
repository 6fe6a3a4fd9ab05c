export BENCH_CFG=2 BENCH_FRAC=16
DFX_CONV_DBG=63 ncu --set full --import-source on --clock-control none -k regex:k_conv_dense -s 3 -c 1 -o gpurun_out/cd63 ./tools/bench_conv > gpurun_out/cd63.log 2>&1
DFX_CONV_DBG=0 ncu --set full --import-source on --clock-control none -k regex:k_conv_dense -s 3 -c 1 -o gpurun_out/cd0 ./tools/bench_conv > gpurun_out/cd0.log 2>&1
