"""INTEGRATION.md's reference-side wrapper (include/dfx_deltaflux.hpp) is real
code: it is compiled here against the reference's own headers
(/root/reference/proj/include/deltaflux/*.hpp) and linked with
libdfx_b200.so. Without a GPU the engine must surface the C-ABI's "no CUDA
device" as dflx::Error (no CPU fallback); an invalid network must be a
dflx::ValidationError either way."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_INC = "/root/reference/proj/include"
LIB_DIR = os.path.join(ROOT, "paper_2210_09887_b200")


@pytest.mark.skipif(not os.path.isdir(REF_INC), reason="reference headers absent (GPU box)")
def test_wrapper_compiles_against_reference_and_maps_errors(tmp_path):
    exe = tmp_path / "integration_main"
    cmd = ["g++", "-std=c++20", "-O1", "-Wall", "-Werror", "-I", REF_INC, "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", "integration_main.cpp"), "-L", LIB_DIR, "-ldfx_b200",
           f"-Wl,-rpath,{LIB_DIR}", "-o", str(exe)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "validation: ValidationError" in out.stdout
    try:
        import torch
        gpu = torch.cuda.is_available()
    except Exception:
        gpu = False
    if gpu:
        assert "engine: ok" in out.stdout, out.stdout
    else:
        assert "engine: Error:" in out.stdout and "no CUDA device" in out.stdout, out.stdout
