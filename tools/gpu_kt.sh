#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for c in c2 c4; do KCONFIG=$c DFX_KTRACE=1 timeout 300 python tools/ktrace.py 2>&1 | head -4; done
