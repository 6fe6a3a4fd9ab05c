"""K-block pipeline stamps of the last dense conv of a real bench frame (dev tool).
Run with DFX_CONV_DBG=64."""
import sys, ctypes as C
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np
import bench, paper_2210_09887_b200 as dfx
from paper_2210_09887_b200 import _capi
spec, cfg, seq = bench.make_workload(8, seed=1000)
e = dfx.DeltaEngine(spec, dfx.EngineConfig(**cfg, conv_mode="tf32x3"))
for f, H in seq: e.run_frame_full(f, H)
lib, _ = _capi.load_library()
tr = (C.c_longlong * 1024)()
assert lib.dfx_debug_conv_trace(tr, 1024) == 0
t0 = tr[3]
print("kernel start", tr[500] - t0, "end", tr[501] - t0, "epi item0", tr[504] - t0, tr[505] - t0)
base = tr[500]
for q in range(24):
    print(f"mma pair {q:2d}: wait {tr[600+3*q]-base:7d} full_ok {tr[601+3*q]-base:7d} issued {tr[602+3*q]-base:7d}")
for k in range(40):
    print(f"kb {k:2d} prod start {tr[k*8]-t0:7d} empty_ok {tr[k*8+1]-t0:7d} arrive {tr[k*8+2]-t0:7d}")
