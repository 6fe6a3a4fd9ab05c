"""Per-conv-layer FLOPs (reference FlopReport) of the bench workload, averaged
over frames 3..N (dev tool)."""
import sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np, torch
import bench, paper_2210_09887_b200 as dfx
N = 10
spec, cfg, seq = bench.make_workload(N, seed=1000)
e = dfx.DeltaEngine(spec, dfx.EngineConfig(**cfg, conv_mode="tf32x3"))
names = [l.name for l in spec.layers if l.conv is not None]
acc = {n: [] for n in names}
for k, (f, H) in enumerate(seq):
    e.run_frame_full(f, H)
    if k >= 3:
        for n in names:
            acc[n].append(e.layer_flops(n))
for n in names:
    f = np.mean([a[0] for a in acc[n]]) / 1e9
    d = np.mean([a[1] for a in acc[n]]) / 1e9
    print(f"{n}: {f:.3f} GFLOP (dense {d:.2f}, ratio {f / d:.3f})")
import ctypes as C
from paper_2210_09887_b200 import _capi
lib, _ = _capi.load_library()
nl = len(spec.layers)
g = (C.c_int * nl)(); u = (C.c_int * nl)()
lib.dfx_engine_debug_counts(e._h if isinstance(e._h, C.c_void_p) else C.c_void_p(e._h.value if hasattr(e._h, "value") else e._h), g, u, nl)
for i, l in enumerate(spec.layers):
    if l.conv is not None:
        print(f"{l.name}: gathered targets {g[i]}, dense units {u[i]} (= {u[i] * 128} px computed)")
