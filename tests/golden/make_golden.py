"""Generate the golden fixtures in tests/golden/ from the UNMODIFIED reference
engine (oracle/_ref/libdfxref.so, built from /root/reference by
oracle/Makefile). Run here, in the container that has /root/reference:

    python tests/golden/make_golden.py

Each fixture stores the network (schema-1 JSON, inline weights), the engine
config, the frames / homographies / ROI maps, and the reference's results per
frame: FrameResult scalars, output, gated input mask, ledger; plus every
layer's packet and state buffers after the last frame. tests/test_oracle.py
checks the C restatement (oracle/dfx_oracle.c) against them bit-for-bit, and
tests/test_gpu_parity.py checks the CUDA path against them.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, os.path.dirname(HERE))

import netgen  # noqa: E402
from oracle.oracle import RefEngine, build  # noqa: E402
from paper_2210_09887_b200.network import spec_to_json  # noqa: E402


def run_case(name, spec, cfg, seq, rois=None):
    eng = RefEngine(spec, cfg)
    rec = {"net": np.array(json.dumps(spec_to_json(spec))), "cfg": np.array(json.dumps(cfg))}
    frames = np.stack([f for f, _ in seq])
    hs = np.stack([h for _, h in seq])
    rec["frames"] = frames
    rec["homographies"] = hs
    if rois is not None:
        rec["rois"] = np.stack(rois)
    for k, (fr, H) in enumerate(seq):
        info, out = eng.run_frame(fr, H, None if rois is None else rois[k])
        rec[f"f{k}_info"] = np.array(json.dumps(info))
        rec[f"f{k}_out"] = out
        rec[f"f{k}_mask"] = eng.input_mask()
        used, ty, tx, cov = eng.read_ledger()
        rec[f"f{k}_ledger"] = np.stack([used.astype(np.int64), ty, tx, cov.astype(np.int64)])
    for l in ["input"] + [l.name for l in spec.layers]:
        d, halo, mask = eng.read_packet(l)
        rec[f"pkt_{l}"] = d
        rec[f"pkth_{l}"] = np.array(halo)
        rec[f"pktm_{l}"] = mask[:256]
        for which in (0, 1, 2):
            try:
                rec[f"st{which}_{l}"] = eng.read_state(l, which)
            except Exception:
                pass
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **rec)
    print(name, "frames", len(seq), "bytes", os.path.getsize(os.path.join(HERE, f"{name}.npz")))


def main():
    build(ref=True)
    rng = np.random.default_rng(2210)
    # 1. toy 3-layer net (netgen toy_net3 shape), static camera, zero thresholds
    spec = netgen.toy_net3(np.random.default_rng(43))
    seq = [(f, netgen.translation(0, 0)) for f in netgen.random_sequence(rng, 3, 32, 48, 4)]
    run_case("toy3_static", spec, dict(tile_size=16, input_threshold=0.0, default_threshold=0.0,
                                       override_net_thresholds=1, mask_dilation=0), seq)
    # 2. C1-shaped (8 ch), integer pan (+5,+3), reference defaults
    spec = netgen.c1_net(np.random.default_rng(2210), channels=8)
    seq = netgen.pan_sequence(rng, 8, 64, 64, 5, 5, 3)
    run_case("c1_small_pan", spec, dict(tile_size=16, grid_rows=6, grid_cols=6), seq)
    # 3. random DAGs (pools, adds, upsample, bn, stride 2), pan with reversal
    for i in range(3):
        spec = netgen.random_network(rng, max_channels=8)
        world = netgen.texture(rng, spec.in_channels, 48 + 120, 64 + 120)
        pos = [(0, 4), (9, 4), (30, 8), (62, 8), (40, 4), (5, 0)]
        seq = [(np.ascontiguousarray(world[:, y:y + 48, x:x + 64]), netgen.translation(x, y)) for x, y in pos]
        run_case(f"random_dag{i}", spec, dict(tile_size=16, input_threshold=0.05, default_threshold=0.02,
                                              mask_dilation=3, grid_rows=5, grid_cols=6), seq)
    # 4. pan + rotation (bilinear warp), ROI and noise suppression
    spec = netgen.random_network(rng, max_channels=6, in_channels=3)
    seq = netgen.pan_rotate_sequence(rng, 3, 48, 64, 4, 3, 2, 0.5, obj=True)
    rois = [(rng.random((1, 48, 64)) > 0.8).astype(np.float32) for _ in seq]
    run_case("rotate_roi_noise", spec, dict(tile_size=16, input_threshold=0.04, default_threshold=0.01,
                                            mask_dilation=2, roi_enabled=1, noise_suppression=1), seq, rois)


if __name__ == "__main__":
    main()
