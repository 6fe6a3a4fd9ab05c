#!/bin/bash
cd "$(dirname "$0")/.."
for shape in "64 128 8" "128 128 4" "128 256 4"; do
  DFX_DENSE_ALLOW_FEWST=1 DFX_DENSE_SMEM_KB=120 DFX_PLAN_DUMP=1 timeout 120 python tools/fewst_probe.py $shape 2>&1 | grep -E "^plan|OK|FAIL|rror" | head -5
done
