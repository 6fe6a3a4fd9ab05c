"""The north_star configs beyond C1 / C2 on the CUDA path, against the
UNMODIFIED reference (oracle/_ref) at their real widths:

  C3  ResNet-18-style backbone: 7x7 stride-2 stem, 2x2 max pool, strided 3x3
      convs and 1x1 stride-2 projections on the gathered-target tensor-core
      kernel (k_conv_tc), residual adds, layer tiles 16 / 8 / 4 / 2 / 1 px
      (network.cpp:113-119); frames cropped from 720p to 192x256 so the CPU
      reference finishes in seconds (the layer shapes are the 720p ones);
  C4  HRNet-W32-style pose net at its named 256x192 crops: four branches,
      nearest upsample + add fusion, 1-px tiles on the stride-32 branch,
      patch-update sequences at 5 % and 35 % update rate.

Tolerance as in test_gpu_fullwidth.py (1e-4 x max(1, max|ref|); masks,
infos, ledger bit-exact); exact mode bit-exact.
"""
import numpy as np
import pytest

import netgen
from engines import CudaEngine, RefEngine, compare_engines
from oracle import oracle
from test_gpu_fullwidth import run_tf32_parity

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")]


def test_c3_resnet18_tf32x3_vs_reference():
    spec = netgen.resnet18_net(np.random.default_rng(2210))
    cfg = dict(tile_size=32)
    seq = netgen.pan_sequence(np.random.default_rng(1000), 3, 192, 256, 5, 4, 2)
    run_tf32_parity(RefEngine(spec, cfg), CudaEngine(spec, cfg, "tf32x3"), spec, seq, "c3_resnet18_192x256")


def test_c3_resnet18_exact_vs_reference():
    spec = netgen.resnet18_net(np.random.default_rng(2210))
    cfg = dict(tile_size=32)
    seq = netgen.pan_sequence(np.random.default_rng(1001), 3, 96, 128, 4, -5, 3)
    compare_engines(RefEngine(spec, cfg), CudaEngine(spec, cfg, "exact"), spec, seq, check_states=True)


@pytest.mark.parametrize("rate", [0.05, 0.35])
def test_c4_hrnet_tf32x3_vs_reference(rate):
    spec = netgen.hrnet_w32_net(np.random.default_rng(2210))
    cfg = dict(tile_size=32, mask_dilation=0)
    seq = netgen.patch_update_sequence(np.random.default_rng(77), 3, 256, 192, 5, rate, 32, 32, 0)
    rec = run_tf32_parity(RefEngine(spec, cfg), CudaEngine(spec, cfg, "tf32x3"), spec, seq, f"c4_hrnet_rate{rate}")
    assert rec["mean_update_rate_sparse"] > 0


def test_c4_hrnet_exact_vs_reference():
    spec = netgen.hrnet_w32_net(np.random.default_rng(2210))
    cfg = dict(tile_size=32, mask_dilation=0)
    seq = netgen.patch_update_sequence(np.random.default_rng(78), 3, 128, 96, 4, 0.2, 32, 0, 32)
    compare_engines(RefEngine(spec, cfg), CudaEngine(spec, cfg, "exact"), spec, seq, check_states=True)


@pytest.mark.parametrize("net", ["resnet18", "hrnet"])
def test_branch_streams_exact_vs_reference(monkeypatch, net):
    """DFX_BRANCH_STREAMS (default on): independent branches (HRNet branches and
    fusions, ResNet projection shortcuts) run on side streams joined by events;
    every word must stay bit-identical to the reference (exact mode)."""
    monkeypatch.setenv("DFX_BRANCH_STREAMS", "1")
    if net == "resnet18":
        spec = netgen.resnet18_net(np.random.default_rng(2210))
        cfg = dict(tile_size=32)
        seq = netgen.pan_sequence(np.random.default_rng(1001), 3, 96, 128, 4, -5, 3)
    else:
        spec = netgen.hrnet_w32_net(np.random.default_rng(2210))
        cfg = dict(tile_size=32, mask_dilation=0)
        seq = netgen.patch_update_sequence(np.random.default_rng(78), 3, 128, 96, 4, 0.2, 32, 0, 32)
    compare_engines(RefEngine(spec, cfg), CudaEngine(spec, cfg, "exact"), spec, seq, check_states=True)
