"""Run the bench workload (C2) for a few frames with nothing else: the target
command for ncu captures (python tools/ncu_probe.py [frames] [config])."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2210_09887_b200 as dfx  # noqa: E402

frames = int(sys.argv[1]) if len(sys.argv) > 1 else 8
config = sys.argv[2] if len(sys.argv) > 2 else "c2"
spec, cfg, seq = bench.make_workload(frames, seed=1000, config=config)
eng = dfx.DeltaEngine(spec, dfx.EngineConfig(**cfg, conv_mode="tf32x3"))
dev = [torch.from_numpy(f).cuda() for f, _ in seq]
for k in range(frames):
    eng.submit_frame(dev[k].data_ptr(), *dev[k].shape, seq[k][1])
    info = eng.sync()
print("update_rate", info["update_rate"], "conv_gflop", info["conv_flops"] / 1e9)
