#!/bin/bash
# same-box A/B of the current tree against ab/<dir> builds: DIRS="a b" CFGS="c2 c3" bash tools/gpu_ab_dirs.sh
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for cfg in ${CFGS:-c2}; do
for r in 1 2; do
  for v in cur $DIRS; do
    d=.; [ $v != cur ] && d=ab/$v
    (cd $d && timeout 400 python bench.py --config $cfg --steps 30 --warmup 3 --no-cpu-baseline --no-sweep 2>/dev/null) > gpurun_out/ab.json
    python -c "
import json
d=json.load(open('gpurun_out/ab.json')); print('$cfg $v'.ljust(12), 'value', round(d['value']), 'e2e', round(d['e2e']['value']), {k: round(v['ms_per_step']*1e3, 1) for k, v in d['kernels'].items()})" 2>/dev/null || echo "$cfg $v failed"
  done
done
done
