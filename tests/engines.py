"""Uniform drivers for the three implementations of the path: the CUDA
product (through its C-ABI), the C restatement and the reference build."""
import numpy as np

from oracle.oracle import OracleEngine, RefEngine, config_struct  # noqa: F401


class CudaEngine:
    """The product's DeltaEngine with the oracle engines' test interface."""

    def __init__(self, spec, cfg, conv_mode="exact"):
        from paper_2210_09887_b200 import DeltaEngine, EngineConfig
        c = EngineConfig.from_any(cfg)
        c.conv_mode = conv_mode
        self.e = DeltaEngine(spec, c)
        self.spec = spec

    def run_frame(self, frame, h9, roi=None):
        return self.e.run_frame_full(frame, h9, roi)

    def __getattr__(self, k):
        return getattr(self.e, k)


def compare_engines(a, b, spec, seq, rois=None, exact=True, atol=0.0, check_states=True, check_packets=True,
                    report=None):
    """Run the same frames through engines a (checker) and b; assert parity.
    exact: bit-equality (==, so +-0 compare equal); else max-abs <= atol and
    identical masks/infos except flop counts."""
    layers = ["input"] + [l.name for l in spec.layers]
    worst = 0.0
    for k, (fr, H) in enumerate(seq):
        roi = None if rois is None else rois[k]
        ia, oa = a.run_frame(fr, H, roi)
        ib, ob = b.run_frame(fr, H, roi)
        assert ia == ib, (k, {x: (ia[x], ib[x]) for x in ia if ia[x] != ib[x]})
        assert oa.shape == ob.shape
        if exact:
            assert np.array_equal(oa, ob), (k, float(np.abs(oa - ob).max()))
        else:
            d = float(np.abs(oa - ob).max()) if oa.size else 0.0
            worst = max(worst, d)
            assert d <= atol, (k, d)
        assert np.array_equal(a.input_mask(), b.input_mask()), k
        assert all(np.array_equal(x, y) for x, y in zip(a.read_ledger(), b.read_ledger())), k
        if check_packets:
            for l in layers:
                pa, pb = a.read_packet(l), b.read_packet(l)
                assert pa[1] == pb[1], (k, l, "halo")
                th, tw = ia["tiles_h"], ia["tiles_w"]
                assert np.array_equal(pa[2][:th * tw], pb[2][:th * tw]), (k, l, "mask")
                if exact:
                    assert np.array_equal(pa[0], pb[0]), (k, l, float(np.abs(pa[0] - pb[0]).max()))
                else:
                    assert float(np.abs(pa[0] - pb[0]).max(initial=0.0)) <= atol, (k, l)
        if check_states:
            for l in layers:
                for which in (0, 1, 2):
                    try:
                        sa = a.read_state(l, which)
                    except Exception:
                        sa = None
                    try:
                        sb = b.read_state(l, which)
                    except Exception:
                        sb = None
                    assert (sa is None) == (sb is None), (k, l, which)
                    if sa is None:
                        continue
                    if exact:
                        assert np.array_equal(sa, sb), (k, l, which, float(np.abs(sa - sb).max()))
                    else:
                        assert float(np.abs(sa - sb).max(initial=0.0)) <= atol, (k, l, which)
    if report is not None:
        report["max_abs"] = worst
    return worst
