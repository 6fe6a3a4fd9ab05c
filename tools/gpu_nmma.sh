timeout 300 python -m pytest tests/test_gpu_kats.py -x -q 2>&1 | tail -2
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for r in 1 2; do for m in 1 2; do DFX_DENSE_NMMA=$m timeout 400 python bench.py --steps 30 --warmup 3 --no-cpu-baseline 2>/dev/null > gpurun_out/ab.json; python -c "
import json
d=json.load(open('gpurun_out/ab.json')); print('nmma $m value', round(d['value']), 'e2e', round(d['e2e']['value']), {k: round(v['ms_per_step']*1e3, 1) for k, v in d['kernels'].items() if k.startswith('conv')})"; done; done
(cd ab/base && timeout 400 python bench.py --steps 30 --warmup 3 --no-cpu-baseline 2>/dev/null) > gpurun_out/ab.json; python -c "
import json
d=json.load(open('gpurun_out/ab.json')); print('base value', round(d['value']), 'e2e', round(d['e2e']['value']), {k: round(v['ms_per_step']*1e3, 1) for k, v in d['kernels'].items() if k.startswith('conv')})"
