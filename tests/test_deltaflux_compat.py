"""The `deltaflux` import surface (deltaflux/_core.py) against the reference's
own Python smoke test (/root/reference/proj/tests/python/test_smoke.py, run
unmodified where the reference tree exists). Without a GPU the engine tests
must fail with the C-ABI's "no CUDA device" (no CPU fallback); on a GPU box
they pass (recorded in profiles/r02_test_smoke_gpu.log)."""
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SMOKE = "/root/reference/proj/tests/python/test_smoke.py"


def test_surface_names_match_reference_package():
    import deltaflux
    want = ["ConvParams", "DeltaEngine", "DeltafluxError", "EngineConfig", "NetworkSpec", "dense_avgpool",
            "dense_conv2d", "dense_maxpool", "dense_relu", "dense_upsample_nearest", "identity_homography",
            "load_frame", "load_network", "load_tensor", "run_dense", "save_ppm", "save_tensor",
            "translation_homography", "wrap_tile"]
    assert sorted(deltaflux.__all__) == sorted(want)
    for n in want:
        assert hasattr(deltaflux, n), n


def test_run_dense_validates_natively():
    import deltaflux as dfx
    spec = dfx.NetworkSpec(in_channels=2)
    spec.conv("c", "input", np.ones((3, 1, 3, 3), np.float32))  # expects 1 channel, gets 2
    spec.output("c")
    with pytest.raises(dfx.DeltafluxError, match="expects 1 channels, gets 2"):
        dfx.run_dense(spec, 16, np.zeros((2, 16, 16), np.float32))


def test_ppm_roundtrip(tmp_path):
    import deltaflux as dfx
    x = np.random.default_rng(1).uniform(0, 1, (3, 5, 7)).astype(np.float32)
    p = str(tmp_path / "a.ppm")
    dfx.save_ppm(x, p)
    y = dfx.load_frame(p)
    assert y.shape == x.shape and float(np.abs(y - x).max()) <= 0.5 / 255 + 1e-6


@pytest.mark.skipif(not os.path.exists(SMOKE), reason="reference tree absent")
def test_reference_test_smoke_runs_against_the_mirror(tmp_path):
    env = dict(os.environ, PYTHONPATH=ROOT + os.pathsep + os.environ.get("PYTHONPATH", ""))
    r = subprocess.run([sys.executable, "-m", "pytest", SMOKE, "-q", "-p", "no:cacheprovider", "-rA"],
                       capture_output=True, text=True, cwd=str(tmp_path), env=env, timeout=600)
    out = r.stdout
    engine_tests = ["test_engine_matches_dense_when_static", "test_engine_pan_reports_fresh_tiles",
                    "test_identical_frames_cost_nothing"]
    for t in ["test_wrap_tile_modulo", "test_dense_conv_box_filter", "test_dense_ops", "test_tensor_file_roundtrip",
              "test_errors_surface_as_python_exceptions"]:
        assert f"PASSED {SMOKE}::{t}" in out or f"PASSED ../{SMOKE.lstrip('/')}::{t}" in out or \
            any(l.startswith("PASSED") and l.endswith(t) for l in out.splitlines()), out[-3000:]
    try:
        import torch
        gpu = torch.cuda.is_available()
    except Exception:
        gpu = False
    for t in engine_tests:
        line = [l for l in out.splitlines() if l.endswith(t) or (t in l and l.startswith(("PASSED", "FAILED")))]
        assert line, out[-3000:]
        if gpu:
            assert line[0].startswith("PASSED"), out[-3000:]
        else:
            assert line[0].startswith("FAILED") and "no CUDA device" in out, out[-3000:]
