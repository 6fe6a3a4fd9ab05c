# same-box A/B: bench the current tree and ab/$AB (built by tools/ab_build.sh), interleaved
AB=${AB:-prev}; STEPS=${STEPS:-30}
for r in 1 2; do
  for d in . ab/$AB; do
    (cd $d && timeout 400 python bench.py --steps $STEPS --warmup 3 --no-cpu-baseline 2>/dev/null) > gpurun_out/ab.json
    python -c "
import json
d=json.load(open('gpurun_out/ab.json')); print('$d'.ljust(10), 'value', round(d['value']), 'e2e', round(d['e2e']['value']), {k: round(v['ms_per_step']*1e3, 1) for k, v in d['kernels'].items()})"
  done
done
