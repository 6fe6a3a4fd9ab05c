#!/bin/bash
cd "$(dirname "$0")/.."
for kb in 120 100; do
  DFX_DENSE_ALLOW_FEWST=1 DFX_DENSE_SMEM_KB=$kb timeout 600 python -m pytest tests/test_gpu_fullwidth.py tests/test_gpu_kats.py -m gpu -q -x -k "crops_tf32 or single_conv or pyramid" 2>&1 | tail -2
  DFX_DENSE_ALLOW_FEWST=1 DFX_DENSE_SMEM_KB=$kb DFX_PLAN_DUMP=1 timeout 300 python tools/fewst_probe.py 256 256 2 2>&1 | grep -E "^plan|OK|FAIL"
done
