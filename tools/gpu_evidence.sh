# Round evidence: smoke, gpu tests, bench, launch list, ncu full of the top kernels.
# The ncu captures skip the first 10 frames (ncu_probe runs 12) so they land on
# representative frames of the ~10 % workload: 16 conv launches (8 plan + 8 dense)
# and ~25 streaming launches per frame.
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -3 gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err  # the driver's default command
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/ncu_probe.py 12 > gpurun_out/ncu_probe.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_conv_dense|k_conv_plan|k_conv_tc" -s 160 -c 16 -o gpurun_out/conv_full python tools/ncu_probe.py 12 > gpurun_out/ncu_conv.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_trunc|k_maxpool|k_claims|k_input|k_densify|k_frame" -s 250 -c 25 -o gpurun_out/hbm_full python tools/ncu_probe.py 12 > gpurun_out/ncu_hbm.log 2>&1
ls -la gpurun_out
