"""Long-run stability soak (serving-style): one C2 engine fed pinned host frames
through the pipelined submit path for DURATION seconds, cycling over a 24-frame
sequence (each wrap jumps the camera back: full resets, evictions and reclaims
on every cycle). Records frames/s and free device memory per window; fails on
any error, on memory growth, or if the output ever holds a non-finite value.

python tools/soak_long.py [seconds] [out.json]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2210_09887_b200 as dfx  # noqa: E402

dur = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
out_path = sys.argv[2] if len(sys.argv) > 2 else None
spec, cfg, seq = bench.make_workload(24, seed=1000)
eng = dfx.DeltaEngine(spec, dfx.EngineConfig(**cfg, conv_mode="tf32x3"))
frames = [torch.from_numpy(f).pin_memory() for f, _ in seq]
c, h, w = seq[0][0].shape
info0 = eng.run_frame_full(seq[0][0], seq[0][1])[1]
out = torch.empty(info0.size, dtype=torch.float32).pin_memory()
free0 = torch.cuda.mem_get_info()[0]
windows, n, t0 = [], 0, time.time()
tw, nw, resets = t0, 0, 0
while time.time() - t0 < dur:
    k = n % len(seq)
    eng.submit_host_frame(frames[k].data_ptr(), c, h, w, seq[k][1], out.data_ptr(), out.numel())
    n += 1
    nw += 1
    if nw == 2000:
        info = eng.sync()
        resets += int(info.get("reset", 0))
        o = out.numpy()
        assert np.isfinite(o).all(), "non-finite output"
        now = time.time()
        windows.append({"frames": n, "frames_per_s": nw / (now - tw), "free_mb": torch.cuda.mem_get_info()[0] / 2**20})
        tw, nw = now, 0
eng.sync()
free1 = torch.cuda.mem_get_info()[0]
rates = [x["frames_per_s"] for x in windows]
res = {"seconds": round(time.time() - t0, 1), "frames": n, "windows": len(windows),
       "frames_per_s_min": min(rates), "frames_per_s_median": float(np.median(rates)), "frames_per_s_max": max(rates),
       "free_mb_start": free0 / 2**20, "free_mb_end": free1 / 2**20,
       "note": "C2 engine, pinned host frames via dfx_engine_submit_host_frame (pipelined), 24-frame sequence "
               "cycled (camera jumps back on every wrap); windows of 2000 frames, host wall clock"}
print(json.dumps(res))
assert free1 >= free0 - (64 << 20), "device memory grew during the soak"
if out_path:
    json.dump({**res, "per_window": windows}, open(out_path, "w"), indent=1)
