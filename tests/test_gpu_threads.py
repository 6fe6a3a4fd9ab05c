"""Engines driven from several host threads at once (one engine per camera
stream, each on its own CUDA stream; ctypes releases the GIL during the C-ABI
calls, so the engines' host code and kernels really overlap): every engine's
outputs, infos, masks and ledger equal the same engine run alone — bit for
bit in both modes (the tf32x3 kernels are deterministic: fixed-order split-K
and accumulator sums) — i.e. no host state (kernel attribute setup, TMA
descriptors, per-device caches, grid hints) leaks between engines."""
import threading

import numpy as np
import pytest

import netgen
from engines import CudaEngine

pytestmark = pytest.mark.gpu


def _run(spec, cfg, seq, out, slot, mode):
    eng = CudaEngine(spec, cfg, mode)
    res = []
    for fr, H in seq:
        info, o = eng.run_frame(fr, H)
        res.append((info, o, eng.input_mask().copy(), [x.copy() for x in eng.read_ledger()]))
    out[slot] = res


@pytest.mark.parametrize("mode", ["exact", "tf32x3"])
def test_four_threads_match_sequential(mode):
    spec = netgen.vgg8_net(np.random.default_rng(11), widths=(32, 64, "P", 128, 128))
    cfg = dict(tile_size=16, input_threshold=0.05, default_threshold=0.02, mask_dilation=2)
    seqs = [netgen.pan_rotate_sequence(np.random.default_rng(40 + i), 3, 256, 256, 6, 2 + i, 1, 0.3) for i in range(4)]
    alone = [None] * 4
    for i in range(4):
        _run(spec, cfg, seqs[i], alone, i, mode)
    together = [None] * 4
    ths = [threading.Thread(target=_run, args=(spec, cfg, seqs[i], together, i, mode)) for i in range(4)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    for i in range(4):
        assert together[i] is not None, i
        for k, (a, b) in enumerate(zip(alone[i], together[i])):
            assert a[0] == b[0], (i, k)
            assert np.array_equal(a[1], b[1]), (i, k, float(np.abs(a[1] - b[1]).max()))
            assert np.array_equal(a[2], b[2]), (i, k)
            assert all(np.array_equal(x, y) for x, y in zip(a[3], b[3])), (i, k)
