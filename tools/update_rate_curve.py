"""Update rate per frame of the bench workload (dev tool): is it stationary?"""
import sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np
import bench, paper_2210_09887_b200 as dfx
N = int(sys.argv[1]) if len(sys.argv) > 1 else 120
thr = float(sys.argv[2]) if len(sys.argv) > 2 else bench.INPUT_THR
import netgen
if len(sys.argv) > 3:  # wobble: amp period
    spec, cfg, _ = bench.make_workload(2, seed=1000)
    seq = netgen.pan_wobble_sequence(np.random.default_rng(1000), 3, 512, 512, N, 2, 1, float(sys.argv[3]), float(sys.argv[4]))
else:
    spec, cfg, seq = bench.make_workload(N, seed=1000)
cfg = dict(cfg, input_threshold=thr)
e = dfx.DeltaEngine(spec, dfx.EngineConfig(**cfg, conv_mode="tf32x3"))
ur = []
for k, (f, H) in enumerate(seq):
    info, _ = e.run_frame_full(f, H)
    ur.append(info["update_rate"])
ur = np.array(ur)
for a in range(0, N, 10):
    print(f"frames {a:3d}-{a + 9:3d}: mean update rate {ur[a:a + 10].mean():.3f}")
