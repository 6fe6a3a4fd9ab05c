DFX_CONV_DBG=0 timeout 120 ./tools/bench_conv | cut -c1-150
timeout 600 python -m pytest tests/test_gpu_tc.py -x -q 2>&1 | tail -2
bash tools/gpu_launch.sh
