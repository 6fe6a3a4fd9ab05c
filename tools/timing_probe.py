"""Quick per-frame timing of the workloads (dev tool; bench.py is the contract)."""
import sys
import time

sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
import numpy as np
import torch

import netgen
import paper_2210_09887_b200 as dfx


def workloads(which):
    if "c1" in which:
        yield ("C1", netgen.c1_net(np.random.default_rng(2210), 64),
               netgen.pan_sequence(np.random.default_rng(1), 64, 192, 192, 12, 5, 3), dict(tile_size=32, grid_rows=8, grid_cols=8))
    if "c2" in which:
        yield ("C2", netgen.vgg8_net(np.random.default_rng(2210)),
               netgen.pan_rotate_sequence(np.random.default_rng(1), 3, 512, 512, 12, 2, 1, 0.2), dict(tile_size=16))


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "c1c2"
    modes = sys.argv[2].split(",") if len(sys.argv) > 2 else ["exact", "tf32x3"]
    for name, spec, seq, cfg in workloads(which):
        for mode in modes:
            c = dfx.EngineConfig(**cfg)
            c.conv_mode = mode
            e = dfx.DeltaEngine(spec, c)
            frames = [torch.from_numpy(f).cuda() for f, _ in seq]
            for k in range(3):
                e.submit_frame(frames[k].data_ptr(), *frames[k].shape, seq[k][1])
                e.sync()
            torch.cuda.synchronize()
            t0 = time.time()
            ur = []
            for k in range(3, len(seq)):
                e.submit_frame(frames[k].data_ptr(), *frames[k].shape, seq[k][1])
                info = e.sync()
                ur.append(info['update_rate'])
            dt = (time.time() - t0) / (len(seq) - 3)
            print(f"{name} {mode}: {dt*1e3:.3f} ms/frame, update_rate {np.mean(ur):.3f}, "
                  f"conv GFLOP {info['conv_flops']/1e9:.2f}, kernels {e.kernel_count()}", flush=True)


if __name__ == "__main__":
    main()
