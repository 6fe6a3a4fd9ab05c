#!/bin/bash
# producer tap pairs + issuer groups vs HEAD (ab/prev): parity subset, per-launch timelines, same-box A/B
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "fullwidth or tc or parity" > gpurun_out/gpu_tests_prod.log 2>&1; tail -2 gpurun_out/gpu_tests_prod.log
for i in 1 3 5; do
  for v in cur prev; do
    d=.; [ $v = prev ] && d=ab/prev
    echo "=== $v dense launch $i"
    (cd $d && DFX_CONV_DBG=64 DFX_CONV_TRACE_IDX=$i timeout 300 python tools/conv_trace2.py 2>&1) | grep -E "first|items done"
  done
done
for cfg in c2 c3; do
for r in 1 2; do
  for v in "cur" "cur2" "prev"; do
    d=.; e=""
    [ $v = prev ] && d=ab/prev
    [ $v = cur2 ] && e="DFX_DENSE_GK=2"
    (cd $d && env $e timeout 400 python bench.py --config $cfg --steps 30 --warmup 3 --no-cpu-baseline 2>/dev/null) > gpurun_out/ab.json
    python -c "
import json
d=json.load(open('gpurun_out/ab.json')); print('$cfg $v'.ljust(10), 'value', round(d['value']), 'e2e', round(d['e2e']['value']), {k: round(v['ms_per_step']*1e3, 1) for k, v in d['kernels'].items() if k.startswith('conv')})"
  done
done
done
