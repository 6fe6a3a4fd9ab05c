#!/bin/bash
# GPU box: layer-level C-ABI tests, DFLX weights, reference smoke test; streams-per-GPU sweep
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_layers.py tests/test_weights_io.py -m gpu -q -x --durations=5 > gpurun_out/gpu_tests3.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gpu_tests3.log
tail -25 gpurun_out/gpu_tests3.log
if [ -f gpurun_out/test_smoke.py ]; then
  (cd gpurun_out && PYTHONPATH=$PWD/.. timeout 300 python -m pytest test_smoke.py -q -rA -p no:cacheprovider > smoke_ref.log 2>&1; echo "smoke rc=$?" >> smoke_ref.log; tail -15 smoke_ref.log)
fi
for s in 1 2 4 8; do
  timeout 600 python bench.py --streams $s --no-cpu-baseline --steps 30 > gpurun_out/bench_streams$s.log 2>&1
  echo "== streams $s rc=$?"; python - <<PY
import json
d=[json.loads(l) for l in open('gpurun_out/bench_streams$s.log') if l.startswith('{')][-1]
print($s, round(d['value'],1), round(d['e2e']['value'],1), d['clocks'])
PY
done
