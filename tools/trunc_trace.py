"""Phase durations of the truncation kernel (DFX_TRUNC_TRACE=1) over the last
frame of the bench workload: per layer, median/max over CTAs of each phase."""
import ctypes
import os
import sys

os.environ["DFX_TRUNC_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2210_09887_b200 as dfx  # noqa: E402
from paper_2210_09887_b200 import _capi  # noqa: E402

frames = int(sys.argv[1]) if len(sys.argv) > 1 else 6
spec, cfg, seq = bench.make_workload(frames, seed=1000)
eng = dfx.DeltaEngine(spec, dfx.EngineConfig(**cfg, conv_mode="tf32x3"))
dev = [torch.from_numpy(f).cuda() for f, _ in seq]
for k in range(frames):
    eng.submit_frame(dev[k].data_ptr(), *dev[k].shape, seq[k][1])
    eng.sync()
lib, _ = _capi.load_library()
buf = np.zeros(64 * 1024 * 16, dtype=np.uint64)
fn = lib.dfx_debug_trunc_trace
fn.argtypes = [ctypes.c_void_p, ctypes.c_longlong]
assert fn(buf.ctypes.data, buf.size) == 0
tr = buf.reshape(64, 1024, 16).astype(np.int64)
per_frame = 9
total = frames * per_frame
names = ["pdl_wait", "list", "tilemax", "ring", "bar_wait", "commit"]
print("layer  " + " ".join(f"{n:>14s}" for n in names) + "   span(us)")
for L in range(per_frame):
    s = (total - per_frame + L) % 64
    t = tr[s]
    t = t[t[:, 0] > 0]
    t0 = t[:, 0].min()
    d = np.diff(t[:, :7], axis=1) / 1e3
    cells = " ".join(f"{np.median(d[:, j]):6.2f}/{d[:, j].max():6.2f}" for j in range(6))
    print(f"{L:5d}  {cells}   {(t[:, 6].max() - t0) / 1e3:7.2f}  (first start->last start {(t[:, 0].max() - t0) / 1e3:.2f})")
print("list detail (median/max us): preload, ext loads done, prefix, syncthreads")
for L in range(per_frame):
    s = (total - per_frame + L) % 64
    t = tr[s]
    t = t[t[:, 0] > 0]
    seg = [(0, 7), (1, 8), (8, 9), (9, 10)]
    print(f"{L:5d}  " + " ".join(f"{np.median((t[:, b] - t[:, a]) / 1e3):6.2f}/{((t[:, b] - t[:, a]) / 1e3).max():6.2f}" for a, b in seg))
print("tilemax detail, CTAs with an item (n, median/max us): phase start->addr, addr->loads, loads->reduced")
for L in range(per_frame):
    s = (total - per_frame + L) % 64
    t = tr[s]
    t = t[(t[:, 0] > 0) & (t[:, 11] > 0) & (t[:, 11] >= t[:, 2])]
    seg = [(2, 11), (11, 12), (12, 13), (13, 3)]
    print(f"{L:5d} n={len(t):4d} " + " ".join(f"{np.median((t[:, b] - t[:, a]) / 1e3):6.2f}/{((t[:, b] - t[:, a]) / 1e3).max():6.2f}" for a, b in seg))
