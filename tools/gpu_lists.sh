#!/bin/bash
# launch lists (ncu gpu__time_duration) of one C3 and one C4 frame
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for c in c3 c4; do
  KCONFIG=$c timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$c.csv \
    python -c "
import os, sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import torch, bench, paper_2210_09887_b200 as dfx
spec, cfg, seq = bench.make_workload(6, seed=1000, config='$c')
e = dfx.DeltaEngine(spec, dfx.EngineConfig(**cfg, conv_mode='tf32x3'))
dev = [torch.from_numpy(f).cuda() for f, _ in seq]
for k in range(6):
    e.submit_frame(dev[k].data_ptr(), *dev[k].shape, seq[k][1]); e.sync()
" > /dev/null 2>&1; echo "$c rc=$?"
done
