"""Randomised soak of the tf32x3 path against the UNMODIFIED reference engine.

Random valid DAGs (netgen.random_network, the reference's netgen.hpp:78-195
grammar) at realistic widths: convs of 2..96 or 2..160 channels, so the dense
tcgen05 kernel meets channel counts that are not multiples of 16 (8-channel
K-blocks, padded N blocks; two N blocks above 128), tile sizes 8 and 16
(tile units and 16x8-pixel block units), strided convs on the gathered kernel, pools, upsamples, adds and
batch norms, over pan sequences with a reversal. Every frame: FrameResult
integers, the input mask, every layer's packet tile mask and the ledger
bit-exact; outputs, packets and states within 1e-4 * max(1, max|ref|)
(test_gpu_fullwidth.run_tf32_parity).
"""
import numpy as np
import pytest

import netgen
from engines import CudaEngine, RefEngine, compare_engines
from oracle import oracle
from test_gpu_fullwidth import run_tf32_parity

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")]


@pytest.mark.parametrize("seed", range(40))
def test_random_wide_networks_vs_reference(seed):
    rng = np.random.default_rng(7100 + seed)
    spec = netgen.random_network(rng, max_channels=96 if seed % 2 else 160, in_channels=int(rng.integers(1, 4)))
    t = int(rng.choice([8, 16]))
    h, w = t * int(rng.integers(4, 9)), t * int(rng.integers(4, 9))
    cfg = dict(tile_size=t, input_threshold=float(rng.choice([0.05, 0.15])),
               default_threshold=float(rng.choice([0.01, 0.03])), mask_dilation=int(rng.integers(0, 5)),
               padded_convolutions=int(seed % 4 != 3))
    px, py = int(rng.integers(-7, 8)), int(rng.integers(-4, 5))
    seq = netgen.pan_sequence(rng, spec.in_channels, h, w, 5, px, py)
    seq = seq + seq[-2::-1][:2]  # pan back over the same world: evicted / re-claimed tiles
    run_tf32_parity(RefEngine(spec, cfg), CudaEngine(spec, cfg, "tf32x3"), spec, seq, f"soak_{seed}")


@pytest.mark.parametrize("seed", range(16))
def test_random_wide_networks_exact_vs_reference(seed):
    """The same kind of random DAGs in exact mode: every output, packet, mask,
    ledger slot and state word bit-identical to the reference."""
    rng = np.random.default_rng(7300 + seed)
    spec = netgen.random_network(rng, max_channels=64, in_channels=int(rng.integers(1, 4)))
    t = int(rng.choice([8, 16]))
    h, w = t * int(rng.integers(4, 8)), t * int(rng.integers(4, 8))
    cfg = dict(tile_size=t, input_threshold=float(rng.choice([0.05, 0.15])),
               default_threshold=float(rng.choice([0.01, 0.03])), mask_dilation=int(rng.integers(0, 5)))
    seq = netgen.pan_sequence(rng, spec.in_channels, h, w, 5, int(rng.integers(-7, 8)), int(rng.integers(-4, 5)))
    compare_engines(RefEngine(spec, cfg), CudaEngine(spec, cfg, "exact"), spec, seq + seq[-2::-1][:2])
