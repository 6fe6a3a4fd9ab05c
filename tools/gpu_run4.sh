#!/bin/bash
# GPU box: full GPU suite, the reference's own python smoke test against the
# deltaflux surface (copied in .refsmoke/, not committed), A/B of DFX_FUSE_TM
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
DFX_PARITY_REPORT=gpurun_out/parity_report4.json timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/gpu_tests4.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gpu_tests4.log
tail -20 gpurun_out/gpu_tests4.log
if [ -f .refsmoke/test_smoke.py ]; then
  (cd .refsmoke && PYTHONPATH=$GRAFT_REPO_ROOT timeout 300 python -m pytest test_smoke.py -q -rA -p no:cacheprovider > ../gpurun_out/smoke_ref.log 2>&1; echo "smoke rc=$?" >> ../gpurun_out/smoke_ref.log)
  tail -15 gpurun_out/smoke_ref.log
fi
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
