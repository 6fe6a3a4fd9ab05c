import sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np
import bench, paper_2210_09887_b200 as dfx
spec, cfg, seq = bench.make_workload(45, seed=1000)
e = dfx.DeltaEngine(spec, dfx.EngineConfig(**cfg, conv_mode="tf32x3"))
for k, (f, H) in enumerate(seq):
    info, _ = e.run_frame_full(f, H)
    if k >= 20: print(k, {kk: (round(v, 3) if isinstance(v, float) else v) for kk, v in info.items() if kk in ("update_rate", "reset", "fresh", "evicted", "placement_rows", "placement_cols", "origin_tx", "origin_ty", "dropped")})
print(sorted(info.keys()))
