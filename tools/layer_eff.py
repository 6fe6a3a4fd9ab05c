"""Per-conv-layer conv FLOPs (the reference's FlopReport) of one steady-state
C2 frame, to pair with the launch list's per-launch times
(profiles/r02_frame_breakdown_c2.txt): python tools/layer_eff.py [frame]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import bench  # noqa: E402
import paper_2210_09887_b200 as dfx  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 10
spec, cfg, seq = bench.make_workload(k + 1, seed=1000)
e = dfx.DeltaEngine(spec, dfx.EngineConfig(**cfg, conv_mode="tf32x3"))
for f, H in seq:
    info, _ = e.run_frame_full(f, H)
print("frame", k, "update_rate", round(info["update_rate"], 3))
for l in spec.layers:
    if l.kind == "conv":
        fl, dfl = e.layer_flops(l.name)
        print(f"{l.name:8s} {l.conv.in_channels:4d}->{l.conv.out_channels:<4d} {fl / 1e9:7.3f} GFLOP (dense {dfl / 1e9:7.3f})")
