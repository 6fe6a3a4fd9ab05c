#!/bin/bash
# half-ring issuer ownership + producer tap pairs: full GPU suite, forced ring depths, same-box A/B
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_own.log 2>&1; tail -2 gpurun_out/gpu_tests_own.log
for n in 4 5 6 7; do
  echo "== NST $n"; DFX_CONV_NST=$n timeout 600 python -m pytest tests/test_gpu_fullwidth.py -q -x -k "crops_tf32x3 or single_conv" 2>&1 | tail -1
done
echo "== NMMA 1"; DFX_DENSE_NMMA=1 timeout 600 python -m pytest tests/test_gpu_fullwidth.py -q -x -k "crops_tf32x3" 2>&1 | tail -1
for cfg in c2 c3; do
for r in 1 2; do
  for v in cur ring8 prev; do
    d=.; e=""; [ $v = prev ] && d=ab/prev; [ $v = ring8 ] && e="DFX_DENSE_RING=8"
    (cd $d && env $e timeout 400 python bench.py --config $cfg --steps 30 --warmup 3 --no-cpu-baseline --no-sweep 2>/dev/null) > gpurun_out/ab.json
    python -c "
import json
d=json.load(open('gpurun_out/ab.json')); print('$cfg $v'.ljust(12), 'value', round(d['value']), 'e2e', round(d['e2e']['value']), {k: round(v['ms_per_step']*1e3, 1) for k, v in d['kernels'].items() if k.startswith('conv')})" 2>/dev/null || echo "$cfg $v failed"
  done
done
done
