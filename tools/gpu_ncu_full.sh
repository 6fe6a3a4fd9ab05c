set -x
python tools/tf32_peak.py gpurun_out/tf32_peak.json
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
ncu --set full --clock-control none --import-source on -k regex:k_conv_tc -s 24 -c 8 -o gpurun_out/conv_tc python tools/ncu_probe.py 5 > gpurun_out/ncu_conv.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_trunc_fused -s 27 -c 9 -o gpurun_out/trunc python tools/ncu_probe.py 5 > gpurun_out/ncu_trunc.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_maxpool_fused|k_conv_targets|k_claims|k_input_apply|k_densify|k_ring_add" -s 60 -c 20 -o gpurun_out/misc python tools/ncu_probe.py 5 > gpurun_out/ncu_misc.log 2>&1
tail -3 gpurun_out/ncu_*.log
ls -la gpurun_out
