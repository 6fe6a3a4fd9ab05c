"""Network JSON + DFLX weight files (network.cpp:350-500,
io.cpp:32-65): networks WRITTEN by the reference's own save_network (one DFLX
file per conv weight / bias and batchnorm scale / shift, plus the manifest)
load through the product's loader to exactly the same parameters (CPU), and
drive the CUDA engine to the reference's results bit-for-bit (GPU, exact)."""
import ctypes as C
import os

import numpy as np
import pytest

import netgen
from oracle import oracle

pytestmark = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")


def save_with_reference(spec, path):
    lib = C.CDLL(oracle.REF_LIB)
    lib.dfr_last_error.restype = C.c_char_p
    desc, keep = spec.to_desc()
    rc = lib.dfr_save_network(C.byref(desc), path.encode())
    assert rc == 0, lib.dfr_last_error()


def nets():
    rng = np.random.default_rng(21)
    return [netgen.random_network(rng, max_channels=8) for _ in range(3)] + [netgen.resnet18_net(rng, widths=(8, 8, 16, 16))]


@pytest.mark.parametrize("i", range(4))
def test_reference_saved_network_loads_identically(tmp_path, i):
    import paper_2210_09887_b200 as dfx
    spec = nets()[i]
    path = str(tmp_path / "net.json")
    save_with_reference(spec, path)
    files = sorted(os.listdir(tmp_path))
    assert any(f.endswith(".dflx") for f in files), files
    got = dfx.load_network(path)
    assert got.in_channels == spec.in_channels and len(got.layers) == len(spec.layers)
    for a, b in zip(spec.layers, got.layers):
        assert (a.name, a.kind, list(a.inputs)) == (b.name, b.kind, list(b.inputs))
        if a.kind == "conv":
            assert np.array_equal(np.asarray(a.conv.weights, np.float32).ravel(), np.asarray(b.conv.weights).ravel())
            if a.conv.bias is not None and len(a.conv.bias):
                assert np.array_equal(np.asarray(a.conv.bias, np.float32), np.asarray(b.conv.bias))
        if a.kind == "batchnorm":
            assert np.array_equal(np.asarray(a.bn_scale, np.float32), np.asarray(b.bn_scale))
            assert np.array_equal(np.asarray(a.bn_shift, np.float32), np.asarray(b.bn_shift))


@pytest.mark.gpu
@pytest.mark.parametrize("i", range(4))
def test_dflx_weights_on_device_match_reference(tmp_path, i):
    import paper_2210_09887_b200 as dfx
    from engines import CudaEngine, RefEngine, compare_engines
    spec = nets()[i]
    path = str(tmp_path / "net.json")
    save_with_reference(spec, path)
    loaded = dfx.load_network(path)
    cfg = dict(tile_size=32, input_threshold=0.05, mask_dilation=2)
    seq = netgen.pan_sequence(np.random.default_rng(30 + i), spec.in_channels, 64, 96, 4, 5, -3)
    compare_engines(RefEngine(spec, cfg), CudaEngine(loaded, cfg, "exact"), spec, seq)
