# A/B an environment knob on the same box: VAR=name VALS="a b" STEPS=30 bash tools/gpu_env_ab.sh
STEPS=${STEPS:-30}
for r in 1 2; do
  for v in $VALS; do
    env $VAR=$v timeout 400 python bench.py --steps $STEPS --warmup 3 --no-cpu-baseline > gpurun_out/ab_env.json 2> gpurun_out/ab_env.err || { echo "$VAR=$v failed"; tail -3 gpurun_out/ab_env.err; continue; }
    python -c "
import json
d=json.load(open('gpurun_out/ab_env.json')); print('$VAR=$v'.ljust(22), 'value', round(d['value']), 'e2e', round(d['e2e']['value']), {k: round(v['ms_per_step']*1e3, 1) for k, v in d['kernels'].items()})"
  done
done
