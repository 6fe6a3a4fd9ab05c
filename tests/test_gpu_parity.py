"""Parity of the CUDA path (through the C-ABI) against the oracle.

conv_mode="exact": every output, gated mask, ledger slot, packet and
spherical-buffer word must be bit-identical (float ==) to the committed
golden fixtures (made from the unmodified reference) and to the C
restatement on random networks and sequences.
"""
import numpy as np
import pytest

import golden_util
import netgen
from engines import CudaEngine, OracleEngine, compare_engines

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("path", golden_util.golden_files(), ids=lambda p: p.split("/")[-1])
def test_exact_matches_golden(path):
    z, spec, cfg = golden_util.load(path)
    eng = CudaEngine(spec, cfg, "exact")

    def check(k, info, out, e_info, e_out, e_mask, e_ledger):
        assert info == e_info, (k, {x: (info[x], e_info[x]) for x in info if info[x] != e_info[x]})
        assert np.array_equal(out, e_out), (k, float(np.abs(out - e_out).max()))
        assert np.array_equal(eng.input_mask(), e_mask), k
        used, ty, tx, cov = eng.read_ledger()
        assert np.array_equal(np.stack([used, ty, tx, cov]).astype(np.int64), e_ledger), k

    last = {}

    def check_last(k, info, *a):
        last.update(info)
        check(k, info, *a)

    golden_util.replay(z, eng, check_last)
    ntiles = last["tiles_h"] * last["tiles_w"]
    for l in ["input"] + [l.name for l in spec.layers]:
        d, halo, mask = eng.read_packet(l)
        assert halo == int(z[f"pkth_{l}"]), l
        assert np.array_equal(d, z[f"pkt_{l}"]), (l, float(np.abs(d - z[f"pkt_{l}"]).max()))
        m = z[f"pktm_{l}"]
        assert np.array_equal(mask[:ntiles], m[:ntiles]), (l, mask[:ntiles], m[:ntiles])
        for which in (0, 1, 2):
            if f"st{which}_{l}" in z.files:
                s = eng.read_state(l, which)
                assert np.array_equal(s, z[f"st{which}_{l}"]), (l, which, float(np.abs(s - z[f"st{which}_{l}"]).max()))


@pytest.mark.parametrize("seed", range(10))
def test_exact_matches_oracle_random(seed):
    rng = np.random.default_rng(500 + seed)
    spec = netgen.random_network(rng, max_channels=12)
    h, w = 16 * int(rng.integers(2, 5)), 16 * int(rng.integers(2, 6))
    cfg = dict(tile_size=16, input_threshold=float(rng.choice([0.0, 0.05, 0.15])),
               default_threshold=float(rng.choice([0.0, 0.02])), mask_dilation=int(rng.integers(0, 8)),
               noise_suppression=int(seed % 3 == 0), roi_enabled=int(seed % 2),
               padded_convolutions=int(seed % 5 != 4))
    if seed % 3 == 1:
        cfg.update(grid_rows=h // 16 + 2, grid_cols=w // 16 + 2)
    if seed % 2 == 0:
        seq = netgen.pan_sequence(rng, spec.in_channels, h, w, 5, int(rng.integers(-9, 10)), int(rng.integers(-5, 6)))
    else:
        seq = netgen.pan_rotate_sequence(rng, spec.in_channels, h, w, 4, 3, -2, 0.6, obj=False)
    rois = [(rng.random((1, h, w)) > 0.75).astype(np.float32) for _ in seq] if cfg["roi_enabled"] else None
    compare_engines(OracleEngine(spec, cfg), CudaEngine(spec, cfg, "exact"), spec, seq, rois)


def test_exact_c1_config():
    """SURVEY §8(d) C1 at full width: 64 ch conv3x3 + relu, 192x192 frames in a
    8x8 grid of 32px tiles, pan (+5,+3), reference defaults, all 16 frames
    (the C checker needs ~5 s per 64-ch frame)."""
    rng = np.random.default_rng(2210)
    spec = netgen.c1_net(rng, channels=64)
    seq = netgen.pan_sequence(rng, 64, 192, 192, 16, 5, 3)
    cfg = dict(tile_size=32, grid_rows=8, grid_cols=8)
    compare_engines(OracleEngine(spec, cfg), CudaEngine(spec, cfg, "exact"), spec, seq, check_states=True)


def test_drop_in_surface():
    """tests/python/test_smoke.py semantics on the CUDA path: static camera
    dense equivalence is covered by golden toy3_static; here the pan events
    and zero-cost repeat (test_smoke.py:100-144)."""
    import paper_2210_09887_b200 as dfx
    rng = np.random.default_rng(7)
    spec = dfx.NetworkSpec(in_channels=1)
    spec.conv("conv1", "input", rng.uniform(-0.5, 0.5, (4, 1, 3, 3)).astype(np.float32),
              rng.uniform(-0.2, 0.2, 4).astype(np.float32))
    spec.relu("relu1", "conv1")
    spec.output("relu1")
    cfg = dfx.EngineConfig(tile_size=16)
    eng = dfx.DeltaEngine(spec, cfg)
    world = np.random.default_rng(4).uniform(0, 1, size=(1, 32, 48 + 16 * 3)).astype(np.float32)
    for k in range(4):
        r = eng.run_frame(world[:, :, 16 * k:16 * k + 48], dfx.translation_homography(16.0 * k, 0.0))
        if k == 0:
            assert r["fresh"] == 6 and r["update_rate"] == pytest.approx(1.0)
        else:
            assert r["fresh"] == 2 and not r["reset"]
    cfg = dfx.EngineConfig(tile_size=16, input_threshold=0.05)
    eng = dfx.DeltaEngine(spec, cfg)
    frame = np.random.default_rng(5).uniform(0, 1, size=(1, 32, 32)).astype(np.float32)
    eng.run_frame(frame, dfx.identity_homography())
    r2 = eng.run_frame(frame, dfx.identity_homography())
    assert r2["conv_flops"] == 0 and r2["update_rate"] == 0.0


def test_pipelined_host_frames_match_run_frame():
    """dfx_engine_submit_host_frame (copy stream, double-buffered device frame
    and output) produces, frame for frame, the outputs of the synchronous
    run_frame path (same arithmetic, exact mode)."""
    import torch
    import netgen
    import paper_2210_09887_b200 as dfx
    rng = np.random.default_rng(11)
    spec = netgen.c1_net(rng, channels=8)
    seq = netgen.pan_sequence(np.random.default_rng(12), 8, 64, 64, 6, 5, 3)
    cfg = dfx.EngineConfig(tile_size=16, conv_mode="exact")
    ref = dfx.DeltaEngine(spec, cfg)
    outs_ref = [ref.run_frame_full(f, H)[1] for f, H in seq]
    eng = dfx.DeltaEngine(spec, cfg)
    frames = [torch.from_numpy(f).pin_memory() for f, _ in seq]
    outs = [torch.empty(o.shape, dtype=torch.float32).pin_memory() for o in outs_ref]
    for k, (f, H) in enumerate(seq):
        eng.submit_host_frame(frames[k].data_ptr(), *f.shape, H, outs[k].data_ptr(), outs[k].numel())
    eng.sync()
    for k in range(len(seq)):
        assert np.array_equal(outs[k].numpy(), outs_ref[k]), k
