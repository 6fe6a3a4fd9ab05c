"""Parity at the benchmarked widths.

Every dense-conv plan variant the C2 benchmark runs (tools/plan_dump.cpp
prints them) is compared with the reference here:

    conv1   3->64   t16  KC=8,  one N block, two accumulator buffers
    conv2  64->64   t16  KC=16, one N block, two accumulator buffers
    conv3  64->128  t8   tile units (2 tiles / unit), NBD=128, ONE accumulator buffer
    conv4 128->128  t8   same
    conv5 128->256  t4   tile units (8 tiles / unit), TWO N blocks, one buffer
    conv6 256->256  t4   same
    conv7 256->256  t2   tile units (32 tiles / unit), two N blocks, 7 stages, split-K
    conv8 256->256  t2   same

Tolerance (stated): conv outputs, packets and states within
    |gpu - ref| <= 1e-4 * max(1, max|ref|)
(the reference's own 1e-4, acceptance.cpp:83, scaled to the value range);
FrameResult integers, input mask, every layer's packet mask and the ledger
bit-exact. `mask agreement` (fraction of identical per-layer tile decisions)
is recorded in the JSON written to $DFX_PARITY_REPORT when set.
"""
import json
import os

import numpy as np
import pytest

import netgen
from engines import CudaEngine, OracleEngine, RefEngine, compare_engines
from oracle import oracle

pytestmark = pytest.mark.gpu


def _tol(ref):
    return 1e-4 * max(1.0, float(np.abs(ref).max(initial=0.0)))


def _report(name, rec):
    path = os.environ.get("DFX_PARITY_REPORT")
    if not path:
        return
    data = {}
    if os.path.exists(path):
        try:
            data = json.load(open(path))
        except Exception:
            data = {}
    data[name] = rec
    json.dump(data, open(path, "w"), indent=1)


def run_tf32_parity(ref, gpu, spec, seq, name, check_states=True):
    """Frame-by-frame: infos, input mask, ledger, every packet's tile mask
    bit-exact; outputs / packets / states within _tol. Returns the record."""
    layers = ["input"] + [l.name for l in spec.layers]
    rec = {"frames": len(seq), "layers": len(layers), "mask_tiles": 0, "mask_equal": 0, "max_abs_out": 0.0,
           "max_rel_pkt": 0.0, "max_rel_state": 0.0, "update_rates": []}
    failures = []
    for k, (fr, H) in enumerate(seq):
        ia, oa = ref.run_frame(fr, H)
        ib, ob = gpu.run_frame(fr, H)
        rec["update_rates"].append(ia["update_rate"])
        if ia != ib:
            failures.append((k, "info", {x: (ia[x], ib[x]) for x in ia if ia[x] != ib[x]}))
        if not np.array_equal(ref.input_mask(), gpu.input_mask()):
            failures.append((k, "input_mask"))
        if not all(np.array_equal(x, y) for x, y in zip(ref.read_ledger(), gpu.read_ledger())):
            failures.append((k, "ledger"))
        d = float(np.abs(oa - ob).max(initial=0.0))
        rec["max_abs_out"] = max(rec["max_abs_out"], d)
        if d > _tol(oa):
            failures.append((k, "output", d))
        th, tw = ia["tiles_h"], ia["tiles_w"]
        for l in layers:
            pa, pb = ref.read_packet(l), gpu.read_packet(l)
            ma, mb = pa[2][:th * tw], pb[2][:th * tw]
            rec["mask_tiles"] += ma.size
            rec["mask_equal"] += int((ma == mb).sum())
            if pa[1] != pb[1] or not np.array_equal(ma, mb):
                failures.append((k, l, "packet mask", int((ma != mb).sum())))
                continue
            e = float(np.abs(pa[0] - pb[0]).max(initial=0.0))
            rec["max_rel_pkt"] = max(rec["max_rel_pkt"], e / max(1.0, float(np.abs(pa[0]).max(initial=0.0))))
            if e > _tol(pa[0]):
                failures.append((k, l, "packet", e))
        if check_states and (k == len(seq) - 1 or k % 4 == 3):
            for l in layers:
                for which in (0, 1, 2):
                    try:
                        sa = ref.read_state(l, which)
                    except Exception:
                        continue
                    sb = gpu.read_state(l, which)
                    e = float(np.abs(sa - sb).max(initial=0.0))
                    rec["max_rel_state"] = max(rec["max_rel_state"], e / max(1.0, float(np.abs(sa).max(initial=0.0))))
                    if e > _tol(sa):
                        failures.append((k, l, which, "state", e))
    rec["mask_agreement"] = rec["mask_equal"] / max(1, rec["mask_tiles"])
    rec["mean_update_rate_sparse"] = float(np.mean(rec["update_rates"][1:])) if len(seq) > 1 else None
    rec["failures"] = [str(f) for f in failures[:20]]
    _report(name, rec)
    assert not failures, failures[:10]
    return rec


def c2_crop_sequence(frames, size=128, seed=7000):
    return netgen.pan_rotate_sequence(np.random.default_rng(seed), 3, size, size, frames, 2, 1, 0.2, obj=True)


C2_CFG = dict(tile_size=16, input_threshold=0.3, default_threshold=0.02, mask_dilation=4)


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("thr", [0.3, 2.0])
def test_c2_vgg8_crops_tf32x3_vs_reference(thr):
    """The benchmarked network at its real widths (3->64->...->256) on 128x128
    crops of the bench's camera motion (pan + rotation + moving object),
    10 frames, against the UNMODIFIED reference engine."""
    spec = netgen.vgg8_net(np.random.default_rng(2210))
    cfg = dict(C2_CFG, input_threshold=thr)
    seq = c2_crop_sequence(10)
    run_tf32_parity(RefEngine(spec, cfg), CudaEngine(spec, cfg, "tf32x3"), spec, seq, f"c2_crops_thr{thr}")


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
def test_c2_vgg8_crops_exact_vs_reference():
    """Same network / crops in exact mode: every word bit-identical to the
    reference (plan, truncation, pooling and densify at 64-256 channels)."""
    spec = netgen.vgg8_net(np.random.default_rng(2210))
    seq = c2_crop_sequence(6)
    compare_engines(RefEngine(spec, C2_CFG), CudaEngine(spec, C2_CFG, "exact"), spec, seq, check_states=True)


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
def test_c2_vgg8_full_frame_tf32x3_vs_reference():
    """The bench configuration itself: 512x512 frames, dense first frame plus
    two sparse frames, against the reference (about 2 minutes of CPU)."""
    spec = netgen.vgg8_net(np.random.default_rng(2210))
    seq = netgen.pan_rotate_sequence(np.random.default_rng(1000), 3, 512, 512, 3, 2, 1, 0.2, obj=True)
    run_tf32_parity(RefEngine(spec, C2_CFG), CudaEngine(spec, C2_CFG, "tf32x3"), spec, seq, "c2_full_512",
                    check_states=True)


# single conv layers at every benchmarked dense plan shape (plus the tile-unit
# widths the C3 / C4 networks use, and their stride-32 stages' 1-px tiles, which
# take the gathered-target kernel); identity truncation at threshold 0 so the
# output IS the conv of the gated input and no tile decision sits at a threshold
@pytest.mark.parametrize("cin,cout,t", [(64, 128, 8), (128, 128, 8), (128, 256, 4), (256, 256, 4), (256, 256, 2),
                                        (128, 128, 4), (256, 256, 8), (32, 32, 8), (512, 512, 2), (64, 64, 8),
                                        (256, 256, 1), (512, 512, 1)])
def test_single_conv_dense_plans(cin, cout, t):
    rng = np.random.default_rng(100 + cin + cout + t)
    from paper_2210_09887_b200 import NetworkSpec
    spec = NetworkSpec(in_channels=cin)
    lim = float(np.sqrt(6.0 / (cin * 9)))
    spec.conv("conv1", "input", rng.uniform(-lim, lim, (cout, cin, 3, 3)).astype(np.float32), None)
    spec.truncate("t1", "conv1", threshold=0.0)
    spec.output("t1")
    cfg = dict(tile_size=t, input_threshold=0.0, default_threshold=0.0, override_net_thresholds=1, mask_dilation=0)
    side = max(8 * t, 24)
    seq = netgen.pan_sequence(rng, cin, side, side + t, 3, 3, 1)
    compare_engines(OracleEngine(spec, cfg), CudaEngine(spec, cfg, "tf32x3"), spec, seq, exact=False,
                    atol=1e-4 * 8 * np.sqrt(cin * 9 / 64.0))


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
def test_c1_16_frames_tf32x3_vs_reference():
    """SURVEY §8(d) C1 at full width for all 16 frames (tf32x3)."""
    rng = np.random.default_rng(2210)
    spec = netgen.c1_net(rng, channels=64)
    seq = netgen.pan_sequence(rng, 64, 192, 192, 16, 5, 3)
    cfg = dict(tile_size=32, grid_rows=8, grid_cols=8)
    run_tf32_parity(RefEngine(spec, cfg), CudaEngine(spec, cfg, "tf32x3"), spec, seq, "c1_16_frames",
                    check_states=True)
