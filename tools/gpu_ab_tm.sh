#!/bin/bash
# GPU box: parity subset with the fused activation pass 1, then an interleaved A/B
# of DFX_FUSE_TM (bench default config) and per-kernel launch lists of one frame
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_fullwidth.py -m gpu -q -x -k "not full_frame and not c1_16" > gpurun_out/gpu_tests_tm.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gpu_tests_tm.log; tail -3 gpurun_out/gpu_tests_tm.log
for r in 1 2 3; do
  for f in 0 1; do
    DFX_FUSE_TM=$f timeout 600 python bench.py --no-cpu-baseline > gpurun_out/ab_tm$f.log 2>&1
    python - <<PY
import json
d=[json.loads(l) for l in open('gpurun_out/ab_tm$f.log') if l.startswith('{')][-1]
print('fuse_tm=$f', round(d['value'],1), round(d['e2e']['value'],1), 'trunc', round(d['kernels']['truncate']['ms_per_step']*1000,1), 'conv', round(d['kernels']['conv_mma']['ms_per_step']*1000,1), 'plan', round(d['kernels']['conv_targets']['ms_per_step']*1000,1), d['clocks']['sm_mhz'])
PY
  done
done
for f in 0 1; do
  DFX_FUSE_TM=$f timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 250 -c 60 --csv --log-file gpurun_out/launches_tm$f.csv python tools/ncu_probe.py 8 > /dev/null 2>&1
done
ls gpurun_out
