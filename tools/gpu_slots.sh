#!/bin/bash
# GPU box: persistent device slot table (small per-frame block) — full GPU suite, then A/B vs ab/prev on C2 / C3
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests_slots.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gpu_tests_slots.log; tail -4 gpurun_out/gpu_tests_slots.log
for c in c2 c3; do
for r in 1 2; do
  for d in . ab/prev; do
    (cd $d && timeout 400 python bench.py --config $c --no-cpu-baseline --no-sweep 2>/dev/null) > gpurun_out/ab.json
    python -c "
import json
d=[json.loads(l) for l in open('gpurun_out/ab.json') if l.startswith('{')][-1]; print('$c', '$d'.ljust(10), 'value', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), d['clocks']['sm_mhz'])"
  done
done
done
KCONFIG=c2 DFX_KTRACE=1 timeout 300 python tools/ktrace.py 2>&1 | head -3
