"""Parity of the tensor-core (tcgen05 kind::tf32, 3-pass split) DeltaConv path.

Tolerance (stated): every output / packet / state value within
    |gpu - ref| <= 1e-4 * max(1, max|ref|)
of the reference's fp32 result (the reference's own acceptance convention is
1e-4 absolute, acceptance.cpp:83); update masks, active tiles, ledger and all
FrameResult integers bit-exact. A mask flip (a tile whose tile_max sits within
fp32 rounding of its threshold) would show up as an info/mask mismatch.
"""
import numpy as np
import pytest

import golden_util
import netgen
from engines import CudaEngine, OracleEngine, compare_engines

pytestmark = pytest.mark.gpu


def tol(ref):
    return 1e-4 * max(1.0, float(np.abs(ref).max(initial=0.0)))


@pytest.mark.parametrize("cin,cout,k,s", [(64, 64, 3, 1), (3, 64, 3, 1), (48, 80, 1, 1), (16, 272, 3, 2),
                                          (8, 16, 5, 1), (3, 32, 7, 2)])
def test_single_conv_layer_gemm(cin, cout, k, s):
    """One conv then identity truncation at threshold 0: the output is the conv
    of the gated input — checks the gathered implicit GEMM (tap offsets,
    K-blocks, N tiles, TMEM epilogue) value by value."""
    rng = np.random.default_rng(11 + cin + cout)
    from paper_2210_09887_b200 import NetworkSpec
    spec = NetworkSpec(in_channels=cin)
    spec.conv("conv1", "input", netgen.random_conv_weights(rng, cin, cout, k), None, stride=s)
    spec.truncate("t1", "conv1", threshold=0.0)
    spec.output("t1")
    cfg = dict(tile_size=16, input_threshold=0.0, default_threshold=0.0, override_net_thresholds=1, mask_dilation=0)
    seq = netgen.pan_sequence(rng, cin, 64, 80, 3, 7, 3)
    compare_engines(OracleEngine(spec, cfg), CudaEngine(spec, cfg, "tf32x3"), spec, seq, exact=False,
                    atol=1e-4 * 8 * np.sqrt(cin * k * k))


@pytest.mark.parametrize("path", golden_util.golden_files(), ids=lambda p: p.split("/")[-1])
def test_tf32x3_matches_golden(path):
    z, spec, cfg = golden_util.load(path)
    eng = CudaEngine(spec, cfg, "tf32x3")

    def check(k, info, out, e_info, e_out, e_mask, e_ledger):
        assert info == e_info, (k, {x: (info[x], e_info[x]) for x in info if info[x] != e_info[x]})
        assert float(np.abs(out - e_out).max(initial=0.0)) <= tol(e_out), k
        assert np.array_equal(eng.input_mask(), e_mask), k

    golden_util.replay(z, eng, check)


@pytest.mark.parametrize("seed", range(8))
def test_tf32x3_matches_oracle_random(seed):
    rng = np.random.default_rng(900 + seed)
    spec = netgen.random_network(rng, max_channels=24)
    h, w = 16 * int(rng.integers(2, 5)), 16 * int(rng.integers(2, 6))
    cfg = dict(tile_size=16, input_threshold=0.05, default_threshold=0.02, mask_dilation=int(rng.integers(0, 6)))
    seq = netgen.pan_sequence(rng, spec.in_channels, h, w, 5, int(rng.integers(-9, 10)), int(rng.integers(-5, 6)))
    a, b = OracleEngine(spec, cfg), CudaEngine(spec, cfg, "tf32x3")
    for fr, H in seq:
        ia, oa = a.run_frame(fr, H)
        ib, ob = b.run_frame(fr, H)
        assert ia == ib
        assert np.array_equal(a.input_mask(), b.input_mask())
        assert float(np.abs(oa - ob).max(initial=0.0)) <= tol(oa)


def test_tf32x3_c1_config():
    rng = np.random.default_rng(2210)
    spec = netgen.c1_net(rng, channels=64)
    seq = netgen.pan_sequence(rng, 64, 192, 192, 3, 5, 3)
    cfg = dict(tile_size=32, grid_rows=8, grid_cols=8)
    a, b = OracleEngine(spec, cfg), CudaEngine(spec, cfg, "tf32x3")
    for fr, H in seq:
        ia, oa = a.run_frame(fr, H)
        ib, ob = b.run_frame(fr, H)
        assert ia == ib
        assert np.array_equal(a.input_mask(), b.input_mask())
        assert float(np.abs(oa - ob).max()) <= tol(oa)


def test_fused_activation_pass1_matches_reference(monkeypatch):
    """DFX_FUSE_TM=1 (opt-in: the consuming activation's tile max folded into
    the dense conv and the plan's zero fill) keeps every mask / info / ledger
    bit-exact and values within tolerance on the C2 network at its widths."""
    monkeypatch.setenv("DFX_FUSE_TM", "1")
    from oracle import oracle
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built")
    from engines import RefEngine
    from test_gpu_fullwidth import C2_CFG, c2_crop_sequence, run_tf32_parity
    spec = netgen.vgg8_net(np.random.default_rng(2210))
    run_tf32_parity(RefEngine(spec, C2_CFG), CudaEngine(spec, C2_CFG, "tf32x3"), spec, c2_crop_sequence(6),
                    "c2_crops_fused_tm")


@pytest.mark.parametrize("kb", ["120", "64"])
def test_reduced_smem_budget_plans(monkeypatch, kb):
    """DFX_DENSE_SMEM_KB squeezes the dense plans: at 120 KB the 128 / 256-channel
    layers run 4-5 weight stages (conv_dense.cu dense_conv_plan), at 64 KB they
    no longer fit and fall back to the gathered-target kernel; results must be
    the same either way."""
    monkeypatch.setenv("DFX_DENSE_SMEM_KB", kb)
    from oracle import oracle
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built")
    from engines import RefEngine
    from test_gpu_fullwidth import C2_CFG, c2_crop_sequence, run_tf32_parity
    spec = netgen.vgg8_net(np.random.default_rng(2210))
    run_tf32_parity(RefEngine(spec, C2_CFG), CudaEngine(spec, C2_CFG, "tf32x3"), spec, c2_crop_sequence(5),
                    f"c2_crops_smem{kb}")
