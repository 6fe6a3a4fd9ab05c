"""The oracle is pinned before it is trusted (CPU, no GPU needed).

* the C restatement (oracle/dfx_oracle.c) reproduces every committed golden
  fixture bit-for-bit (fixtures: tests/golden/make_golden.py, generated from
  the unmodified reference build);
* where the reference build exists (this container), the restatement is also
  checked live against it on random networks and sequences: outputs, gated
  masks, every layer's packet, every state buffer and the ledger.
"""
import numpy as np
import pytest

import golden_util
import netgen
from oracle.oracle import OracleEngine, RefEngine, ref_available


@pytest.mark.parametrize("path", golden_util.golden_files(), ids=lambda p: p.split("/")[-1])
def test_restatement_matches_golden(path):
    z, spec, cfg = golden_util.load(path)
    eng = OracleEngine(spec, cfg)

    def check(k, info, out, e_info, e_out, e_mask, e_ledger):
        assert info == e_info, f"frame {k}"
        assert np.array_equal(out, e_out), f"frame {k} output"
        assert np.array_equal(eng.input_mask(), e_mask), f"frame {k} mask"
        used, ty, tx, cov = eng.read_ledger()
        assert np.array_equal(np.stack([used, ty, tx, cov]).astype(np.int64), e_ledger)

    golden_util.replay(z, eng, check)
    for l in ["input"] + [l.name for l in spec.layers]:
        d, halo, mask = eng.read_packet(l)
        assert np.array_equal(d, z[f"pkt_{l}"]), l
        assert halo == int(z[f"pkth_{l}"])
        assert np.array_equal(mask[:256], z[f"pktm_{l}"])
        for which in (0, 1, 2):
            if f"st{which}_{l}" in z.files:
                assert np.array_equal(eng.read_state(l, which), z[f"st{which}_{l}"]), (l, which)


needs_ref = pytest.mark.skipif(not ref_available(), reason="reference build (oracle/_ref) not present")


def _compare_live(spec, cfg, seq, rois=None):
    r, o = RefEngine(spec, cfg), OracleEngine(spec, cfg)
    for k, (fr, H) in enumerate(seq):
        roi = None if rois is None else rois[k]
        ir, outr = r.run_frame(fr, H, roi)
        io, outo = o.run_frame(fr, H, roi)
        assert ir == io
        assert np.array_equal(outr, outo)
        assert np.array_equal(r.input_mask(), o.input_mask())
        for l in ["input"] + [l.name for l in spec.layers]:
            pr, po = r.read_packet(l), o.read_packet(l)
            assert np.array_equal(pr[0], po[0]) and pr[1] == po[1] and np.array_equal(pr[2], po[2]), l
        assert all(np.array_equal(a, b) for a, b in zip(r.read_ledger(), o.read_ledger()))


@needs_ref
@pytest.mark.parametrize("seed", range(12))
def test_restatement_matches_reference_random(seed):
    rng = np.random.default_rng(100 + seed)
    spec = netgen.random_network(rng, max_channels=8)
    h, w = 16 * int(rng.integers(2, 4)), 16 * int(rng.integers(2, 5))
    cfg = dict(tile_size=16, input_threshold=float(rng.choice([0.0, 0.05, 0.15])),
               default_threshold=float(rng.choice([0.0, 0.02])), mask_dilation=int(rng.integers(0, 8)),
               noise_suppression=int(seed % 3 == 0), roi_enabled=int(seed % 2),
               override_net_thresholds=int(seed % 4 == 0), padded_convolutions=int(seed % 5 != 4))
    if seed % 3 == 1:
        cfg.update(grid_rows=h // 16 + 2, grid_cols=w // 16 + 2)
    if seed % 2 == 0:
        seq = netgen.pan_sequence(rng, spec.in_channels, h, w, 5, int(rng.integers(-9, 10)), int(rng.integers(-5, 6)))
    else:
        seq = netgen.pan_rotate_sequence(rng, spec.in_channels, h, w, 4, 3, -2, 0.6, obj=False)
    rois = [(rng.random((1, h, w)) > 0.75).astype(np.float32) for _ in seq] if cfg["roi_enabled"] else None
    _compare_live(spec, cfg, seq, rois)


@needs_ref
def test_restatement_matches_reference_c1_shape():
    """C1's network shape at reduced size (64 ch is slow on one core)."""
    rng = np.random.default_rng(2210)
    spec = netgen.c1_net(rng, channels=16)
    seq = netgen.pan_sequence(rng, 16, 96, 96, 4, 5, 3)
    _compare_live(spec, dict(tile_size=32), seq)


def test_wrap_tile_kats():
    """tests/test_tile_grid.cpp:13-19 KATs, restated through the C oracle's
    floor_mod via the ledger of a tiny engine is overkill; check the formula."""
    def wrap(tx, ty, rows, cols):
        return (ty % rows, tx % cols)  # python % is the mathematical floor_mod
    assert wrap(0, 0, 4, 4) == (0, 0)
    assert wrap(5, 2, 4, 4) == (2, 1)
    assert wrap(-1, 0, 4, 4) == (0, 3)
    assert wrap(-5, -9, 4, 4) == (3, 3)
