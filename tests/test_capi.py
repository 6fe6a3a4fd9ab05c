"""The C-ABI library loads and exports every entry point include/dfx_b200.h
declares (CPU only: no compute calls), and the host-side API mirrors the
reference's Python surface."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "dfx_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)  # declarations only, not comments
    return sorted(set(re.findall(r"\b(dfx_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2210_09887_b200 import _capi
    lib = ctypes.CDLL(_capi.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 18
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_wrap_tile_kats_through_cabi():
    # tests/test_tile_grid.cpp:13-19 (input TileCoord{tx,ty} -> (row, col))
    from paper_2210_09887_b200 import wrap_tile
    assert wrap_tile(0, 0, 4, 4) == (0, 0)
    assert wrap_tile(5, 2, 4, 4) == (2, 1)
    assert wrap_tile(-1, 0, 4, 4) == (0, 3)
    assert wrap_tile(-5, -9, 4, 4) == (3, 3)


def test_default_config_matches_reference():
    from paper_2210_09887_b200 import EngineConfig, _capi
    lib, api = _capi.load_library()
    c = _capi.EngineConfigC()
    api["default_config"](ctypes.byref(c))
    py = EngineConfig().to_c()
    for k, _ in _capi.EngineConfigC._fields_:
        assert getattr(c, k) == pytest.approx(getattr(py, k)), k
    assert c.tile_size == 32 and c.mask_dilation == 10
    assert c.input_threshold == pytest.approx(0.15) and c.default_threshold == pytest.approx(0.02)


def test_network_json_roundtrip(tmp_path):
    import json
    import numpy as np
    import netgen
    from paper_2210_09887_b200 import load_network, spec_to_json
    spec = netgen.random_network(np.random.default_rng(3))
    p = tmp_path / "net.json"
    p.write_text(json.dumps(spec_to_json(spec)))
    back = load_network(str(p))
    assert [l.name for l in back.layers] == [l.name for l in spec.layers]
    for a, b in zip(spec.layers, back.layers):
        assert a.kind == b.kind and a.inputs == b.inputs
        if a.conv is not None:
            assert np.array_equal(np.asarray(a.conv.weights).ravel(), np.asarray(b.conv.weights).ravel())


def test_errors_surface_as_python_exceptions(tmp_path):
    import paper_2210_09887_b200 as dfx
    with pytest.raises(dfx.DeltafluxError):
        dfx.load_tensor(str(tmp_path / "missing.dflx"))
    with pytest.raises(dfx.DeltafluxError):
        dfx.load_network(str(tmp_path / "missing.json"))
