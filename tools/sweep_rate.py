"""Update rate / frame time of the C2 sequence vs input threshold and dilation
(dev tool used to tune the C2 bench thresholds to the ~10% update rate that
SURVEY §8(d) names)."""
import sys, time
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np, torch
import netgen, paper_2210_09887_b200 as dfx

F = 16
spec = netgen.vgg8_net(np.random.default_rng(2210))
seq = netgen.pan_rotate_sequence(np.random.default_rng(1000), 3, 512, 512, F, 2, 1, 0.2, obj=True)
frames = [torch.from_numpy(f).cuda() for f, _ in seq]
for thr in (0.15, 0.2, 0.25, 0.3, 0.4, 0.5):
    for dil in (10, 4):
        e = dfx.DeltaEngine(spec, dfx.EngineConfig(tile_size=16, input_threshold=thr, mask_dilation=dil))
        ur, ms = [], []
        for k in range(F):
            t0 = time.time()
            e.submit_frame(frames[k].data_ptr(), *frames[k].shape, seq[k][1]); info = e.sync()
            if k >= 3:
                ur.append(info['update_rate']); ms.append((time.time() - t0) * 1e3)
        print(f"thr={thr} dil={dil}: update_rate mean={np.mean(ur):.3f} min={np.min(ur):.3f} max={np.max(ur):.3f} "
              f"ms/frame={np.mean(ms):.3f} conv_gflop={info['conv_flops']/1e9:.2f}", flush=True)
        e.close()
